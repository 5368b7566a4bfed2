"""Constraint sharding on one GPU: the partial sweeps / checks of ranks 0..W-1 (fsmt_shard mode 1)
sum to the unsharded result, through caller-bound device buffers (fsmt_bind_buffers)."""
import numpy as np
import pytest

import fsmt_gen
from fsmt_gen.points import random_points

pytestmark = pytest.mark.gpu


@pytest.mark.parametrize("name,world", [("cfg4s", 2), ("cfg3s", 3), ("cfg2s", 2), ("cfg2", 2)])
def test_constraint_shards_sum_to_full(name, world):
    import torch
    import paper_2603_22877_b200 as P
    inst = fsmt_gen.config(name)
    R = 40
    full = P.Solver(0)
    full.load_formula(inst.text)
    full.build_xbdd()
    d = full.get_dims()
    a, b = random_points(d["n_bool"], d["n_real"], R, seed=3, b_lo=0.0, b_hi=1.0)
    full.begin(R, 9)
    full.set_state(a, b)
    full.sweep(1.2, 1)
    obj_f, ga_f, gb_f = full.get_sweep()
    unsat_f = full.stage_end(1)
    sums = [np.zeros_like(obj_f), np.zeros_like(ga_f), np.zeros_like(gb_f), np.zeros(R, dtype=np.int64)]
    for rank in range(world):
        s = P.Solver(0)
        s.load_formula(inst.text)
        s.build_xbdd()
        s.shard(rank, world, 1)
        s.begin(R, 9)
        s.set_state(a, b)
        ga = torch.zeros((d["n_bool"], R), dtype=torch.float64, device="cuda")
        gb = torch.zeros((d["n_real"], R), dtype=torch.float64, device="cuda")
        obj = torch.zeros(R, dtype=torch.float64, device="cuda")
        un = torch.zeros(R, dtype=torch.int32, device="cuda")
        s.bind_buffers(ga, gb, obj, un)
        s.sweep(1.2, 1)
        s.stage_end(1, copy=False)
        torch.cuda.synchronize()
        sums[0] += obj.cpu().numpy()
        sums[1] += ga.cpu().numpy()
        sums[2] += gb.cpu().numpy()
        sums[3] += un.cpu().numpy()
    assert np.allclose(sums[0], obj_f, rtol=1e-9, atol=1e-9)
    assert np.allclose(sums[1], ga_f, rtol=1e-6, atol=1e-7) and np.allclose(sums[2], gb_f, rtol=1e-6, atol=1e-7)
    assert np.array_equal(sums[3], unsat_f.astype(np.int64))
