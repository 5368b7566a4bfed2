"""The multi-GPU drivers with the REAL engine at world size 2 (two processes, one Solver each, on the
one visible GPU, over gloo with the drivers' host staging): restart-sharded and constraint-sharded
solves must reproduce the world-size-1 solve bit for bit (every restart's sums are
exact, DESIGN.md §7 item 14, and Philox is keyed by the global restart id)."""
import os
import socket

import numpy as np
import pytest

pytestmark = pytest.mark.gpu

KAPPAS = [0.5, 1.0, 2.0, 4.0, 8.0, 16.0]


def _port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    p = s.getsockname()[1]
    s.close()
    return p


def _worker(rank, world, port, mode, out):
    import torch
    import torch.distributed as dist
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    dist.init_process_group("gloo", rank=rank, world_size=world)
    torch.cuda.set_device(0)
    import fsmt_gen
    import paper_2603_22877_b200 as P
    from paper_2603_22877_b200 import dist as D
    inst = fsmt_gen.config("cfg4s")
    s = P.Solver(0)
    s.load_formula(inst.text)
    s.build_xbdd()
    s.set_params(kappas=KAPPAS, eta=0.05)
    d = s.get_dims()
    R = 64
    if mode == "restart":
        res = D.solve_restart_sharded(s, d["n_bool"], d["n_real"], R // world, 6, 21, KAPPAS)
        a, b = s.get_state()
        state = (a.tolist(), b.tolist())
    else:
        res = D.solve_constraint_sharded(s, d["n_bool"], d["n_real"], R, 6, 21, KAPPAS, 1e-2)
        a, b = s.get_state()
        state = (a.tolist(), b.tolist())
    out[(mode, world, rank)] = ((res.verdict, res.winner_restart, res.winner_stage, res.best_unsat, res.stages_run,
                                 res.x.tolist(), res.y.tolist()), state)
    dist.destroy_process_group()


@pytest.mark.parametrize("mode", ["restart", "constraint"])
def test_world2_real_engine_matches_world1(mode):
    import torch.multiprocessing as mp
    out = mp.Manager().dict()
    mp.spawn(_worker, args=(1, _port(), mode, out), nprocs=1, join=True)
    mp.spawn(_worker, args=(2, _port(), mode, out), nprocs=2, join=True)
    ref, ref_state = out[(mode, 1, 0)]
    for rank in (0, 1):
        got, st = out[(mode, 2, rank)]
        assert got == ref, (rank, got[:5], ref[:5])
        if mode == "constraint":                  # every rank holds the full state, bit for bit
            assert st == ref_state
        else:                                     # rank k holds global restarts [32k, 32k + 32)
            a1, b1 = np.array(ref_state[0]), np.array(ref_state[1])
            a2, b2 = np.array(st[0]), np.array(st[1])
            if got[4] == ref[4]:                  # same number of stages run
                assert np.array_equal(a2, a1[:, 32 * rank:32 * rank + 32])
                assert np.array_equal(b2, b1[:, 32 * rank:32 * rank + 32])
