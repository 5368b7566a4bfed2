"""Constraint sharding on one GPU: the partial sweeps / checks of ranks 0..W-1 (fsmt_shard mode 1)
sum to the unsharded result BIT FOR BIT (the sweep's fp64 sums are exact, DESIGN.md
§7 item 14), through caller-bound device buffers (fsmt_bind_buffers)."""
import numpy as np
import pytest

import fsmt_gen
from fsmt_gen.points import random_points, random_counters

pytestmark = pytest.mark.gpu


def _solver(P, text):
    s = P.Solver(0)
    s.load_formula(text)
    s.build_xbdd()
    return s


@pytest.mark.parametrize("name,world", [("cfg4s", 2), ("cfg3s", 3), ("cfg2s", 2), ("cfg2", 2), ("cfg4m", 3)])
def test_constraint_shards_sum_to_full(name, world):
    import torch
    import paper_2603_22877_b200 as P
    inst = fsmt_gen.config(name)
    R = 40
    full = _solver(P, inst.text)
    d = full.get_dims()
    a, b = random_points(d["n_bool"], d["n_real"], R, seed=3, b_lo=0.0, b_hi=1.0)
    U = random_counters(d["n_cons"], R, seed=4, max_u=6)
    full.begin(R, 9)
    full.set_state(a, b)
    full.set_counters(U)
    full.sweep(1.2, 5)
    obj_f, ga_f, gb_f = full.get_sweep()
    unsat_f = full.stage_end(5)
    U_f = full.get_counters()
    # each rank sweeps its share into one flat bound buffer [grad_a | grad_b | obj | slot rows] (grid
    # units, as the multi-GPU driver all-reduces it); the exact sum, chained on one rank
    # (fsmt_sweep_finish), must be the unsharded sweep bit for bit
    rows = d["n_slot_rows"]
    nb, nr = d["n_bool"], d["n_real"]
    flat_sum = None
    unsat_sum = np.zeros(R, dtype=np.int64)
    U_sh = U.copy()
    ranks = []
    for rank in range(world):
        s = _solver(P, inst.text)
        s.shard(rank, world, 1)
        s.begin(R, 9)
        s.set_state(a, b)
        s.set_counters(U)
        flat = torch.zeros((nb + nr + 1 + rows) * R, dtype=torch.float64, device="cuda")
        un = torch.zeros(R, dtype=torch.int32, device="cuda")
        umax = torch.zeros(R, dtype=torch.int32, device="cuda")
        s.bind_buffers(flat[:nb * R].view(nb, R), flat[nb * R:(nb + nr) * R].view(nr, R),
                       flat[(nb + nr) * R:(nb + nr + 1) * R], un, umax)
        if rows:
            s.bind_slot_grads(flat[(nb + nr + 1) * R:].view(rows, R))
        s.sweep(1.2, 5)
        torch.cuda.synchronize()
        part = flat.cpu().numpy().copy()
        flat_sum = part if flat_sum is None else flat_sum + part      # exact: on-grid values
        s.stage_end(5, copy=False)
        torch.cuda.synchronize()
        unsat_sum += un.cpu().numpy()
        Ur = s.get_counters()                       # each shard updates only its own constraints' rows
        U_sh = np.where(Ur != U, Ur, U_sh)
        ranks.append((s, flat))
    s0, flat0 = ranks[0]
    flat0.copy_(torch.from_numpy(flat_sum))
    s0.sweep_finish()
    obj, ga, gb = s0.get_sweep()
    assert np.array_equal(obj, obj_f)
    assert np.array_equal(ga, ga_f) and np.array_equal(gb, gb_f)
    assert np.array_equal(unsat_sum, unsat_f.astype(np.int64))
    assert np.array_equal(U_sh, U_f)


def test_bind_buffers_rejects_host_memory():
    import torch
    import paper_2603_22877_b200 as P
    s = _solver(P, fsmt_gen.config("cfg4s").text)
    s.begin(8, 1)
    d = s.get_dims()
    with pytest.raises(P.FsmtError):
        s.bind_buffers(torch.zeros((d["n_bool"], 8), dtype=torch.float64))
