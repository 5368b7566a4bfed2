"""Constraint-sharded driver over gloo on CPU: world_size 2 must give the
same trajectory, verdict and model as world_size 1 (a deterministic fake engine whose partial
gradients / violation counts are exact dyadic sums stands in for the GPU Solver)."""
import os
import socket

import numpy as np
import pytest
import torch
import torch.distributed as dist
import torch.multiprocessing as mp

NB, NR, C = 6, 4, 23


class FakeConstraintEngine:
    def shard(self, rank, world, mode):
        assert mode == 1
        self.c0, self.c1 = C * rank // world, C * (rank + 1) // world

    def begin(self, R, seed, off):
        self.R = R
        g = torch.Generator().manual_seed(seed)
        self.a = torch.randint(-8, 8, (NB, R), generator=g).double()
        self.b = torch.randint(-8, 8, (NR, R), generator=g).double()

    def bind_buffers(self, ga, gb, obj, unsat, umax):
        self.ga, self.gb, self.obj, self.unsat, self.umax = ga, gb, obj, unsat, umax

    def step_sizes(self, kappa):
        return 0.5, 0.25

    def sweep(self, kappa, t):
        self.ga.zero_()
        self.gb.zero_()
        self.obj.zero_()
        for c in range(self.c0, self.c1):
            self.ga[c % NB] += (c + 1) * torch.sign(self.a[c % NB] + 0.5)
            self.gb[c % NR] += (c % 3) - 1.0
            self.obj += torch.floor(self.a[c % NB] / 4)

    def update(self, eta, eps, eta_b=0.0):
        self.a -= eta * self.ga
        self.b -= eta_b * self.gb

    def stage_end(self, t, copy=False):
        self.unsat.zero_()
        for c in range(self.c0, self.c1):
            v = (c + t + torch.arange(self.R) + torch.floor(self.a[c % NB]).long()) % 5 != 0
            self.unsat += v.int()
            self.umax.copy_(torch.maximum(self.umax, self.unsat))     # a local max the driver all-reduces

    def get_model(self, r):
        return np.sign(self.a[:, r].numpy() + 0.5).astype(np.int8), self.b[:, r].numpy().astype(np.float32)


def _worker(rank, world, port, out):
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    dist.init_process_group("gloo", rank=rank, world_size=world)
    from paper_2603_22877_b200.dist import solve_constraint_sharded
    res = solve_constraint_sharded(FakeConstraintEngine(), NB, NR, 16, 2, 5, [1.0, 2.0, 3.0, 4.0], 0.0)
    out[(world, rank)] = (res.verdict, res.winner_restart, res.winner_stage, res.best_unsat, res.x.tolist(),
                          res.y.tolist())
    dist.destroy_process_group()


def _port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    p = s.getsockname()[1]
    s.close()
    return p


def test_constraint_sharded_matches_single_rank():
    out = mp.Manager().dict()
    mp.spawn(_worker, args=(1, _port(), out), nprocs=1, join=True)
    mp.spawn(_worker, args=(2, _port(), out), nprocs=2, join=True)
    ref = out[(1, 0)]
    assert out[(2, 0)] == ref and out[(2, 1)] == ref
