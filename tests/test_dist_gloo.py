"""Host-side logic of the restart-sharded multi-GPU driver, world_size 2 over gloo on CPU.

A deterministic fake engine stands in for the GPU Solver (the driver only sees the step
API); the sharded result must equal the single-process result over all restarts.
"""
import os
import socket

import numpy as np
import pytest
import torch.distributed as dist
import torch.multiprocessing as mp

N_BOOL, N_REAL = 5, 3


class FakeEngine:
    """unsat[r, t] and the model are pure functions of (global restart, stage)."""

    def __init__(self, sat_at=None):
        self.sat_at = sat_at      # (global restart, stage) that reaches unsat 0, or None

    def begin(self, R, seed, restart_offset=0):
        self.R, self.seed, self.off = R, seed, restart_offset

    def _unsat(self, g, t):
        if self.sat_at is not None and (g, t) == self.sat_at:
            return 0
        return 1 + (g * 7919 + t * 104729 + self.seed) % 13

    def run_stage(self, t, kappa, steps):
        self.t = t
        u = np.array([self._unsat(self.off + r, t) for r in range(self.R)], dtype=np.uint32)
        return u, int(u.min())

    def get_model(self, r):
        g = self.off + r
        x = np.array([1 if (g >> i) & 1 else -1 for i in range(N_BOOL)], dtype=np.int8)
        y = np.array([g + 0.25 * self.t, -g, 0.5], dtype=np.float32)
        return x, y


def reference(R_total, seed, kappas, sat_at):
    eng = FakeEngine(sat_at)
    eng.begin(R_total, seed, 0)
    best = None
    for t, _ in enumerate(kappas, start=1):
        u, _ = eng.run_stage(t, 1.0, 1)
        r = int(np.argmin(u))
        if best is None or u[r] < best[0]:
            best = (int(u[r]), t, r, eng.get_model(r))
        if best[0] == 0:
            break
    return best


def _worker(rank, world, port, R, seed, kappas, sat_at, out):
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    dist.init_process_group("gloo", rank=rank, world_size=world)
    from paper_2603_22877_b200.dist import solve_restart_sharded
    res = solve_restart_sharded(FakeEngine(sat_at), N_BOOL, N_REAL, R, 1, seed, kappas)
    out[rank] = (res.verdict, res.winner_restart, res.winner_stage, res.best_unsat, res.x.tolist(), res.y.tolist())
    dist.destroy_process_group()


def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    p = s.getsockname()[1]
    s.close()
    return p


@pytest.mark.parametrize("sat_at", [None, (11, 3), (2, 5)])
def test_restart_sharded_matches_single_process(sat_at):
    world, R, seed, kappas = 2, 8, 17, [0.5, 1.0, 1.5, 2.0, 2.5, 3.0]
    mgr = mp.Manager()
    out = mgr.dict()
    mp.spawn(_worker, args=(world, _free_port(), R, seed, kappas, sat_at, out), nprocs=world, join=True)
    ref = reference(world * R, seed, kappas, sat_at)
    for rank in range(world):
        verdict, g, t, u, x, y = out[rank]
        assert (u, t, g) == (ref[0], ref[1], ref[2])
        assert verdict == (10 if ref[0] == 0 else 0)
        assert x == ref[3][0].tolist() and np.allclose(y, ref[3][1])
