"""Restart-sharded multi-GPU solve: one process per GPU over torch.distributed.

The paper runs 8 independent seeded replicas, one per GPU.  Here the
restarts of one solve are sharded instead: rank k owns global restarts
[k*R, (k+1)*R) (Philox counters use the global id, so every restart's trajectory is the
same whatever the sharding).  There is no data-path collective; per stage the ranks
exchange one int64 (C1/C2: all-reduce MIN of (unsat << 32 | global restart)) and, when the
best model improves, the owning rank broadcasts it (C3: x int8[n_bool] + y f32[n_real]).
The winner is the lexicographically smallest (stage, restart) with unsat = 0, else the
smallest (unsat, stage, restart) -- identical to a single process running all restarts.

`engine` is anything with the Solver step API: begin(R, seed, restart_offset),
run_stage(t, kappa, steps) -> (unsat[R], min), get_model(r) -> (x, y), and dims
(n_bool, n_real).  On GPU ranks it is a paper_2603_22877_b200.Solver.
"""
from __future__ import annotations

from dataclasses import dataclass

import numpy as np
import torch
import torch.distributed as dist

SAT, UNKNOWN = 10, 0


@dataclass
class DistResult:
    verdict: int
    x: np.ndarray
    y: np.ndarray
    winner_restart: int
    winner_stage: int
    best_unsat: int
    stages_run: int


def _device_for_backend():
    return torch.device("cuda", torch.cuda.current_device()) if dist.get_backend() == "nccl" else torch.device("cpu")


def solve_restart_sharded(engine, n_bool: int, n_real: int, restarts_per_rank: int, steps: int, seed: int,
                          kappas, group=None) -> DistResult:
    rank = dist.get_rank(group)
    world = dist.get_world_size(group)
    R = int(restarts_per_rank)
    dev = _device_for_backend()
    engine.begin(R, seed, restart_offset=rank * R)
    best_key = None           # (unsat, stage, global restart)
    x_best = torch.zeros(n_bool, dtype=torch.int8, device=dev)
    y_best = torch.zeros(n_real, dtype=torch.float32, device=dev)
    key_t = torch.zeros(1, dtype=torch.int64, device=dev)
    stages = 0
    for t, kappa in enumerate(kappas, start=1):
        unsat, _ = engine.run_stage(t, float(kappa), steps)
        stages = t
        r_loc = int(np.argmin(unsat))                      # first minimum = lowest restart id
        key_t.fill_((int(unsat[r_loc]) << 32) | (rank * R + r_loc))
        dist.all_reduce(key_t, op=dist.ReduceOp.MIN, group=group)      # C1 + C2
        k = int(key_t.item())
        u_min, g_min = k >> 32, k & 0xFFFFFFFF
        if best_key is None or u_min < best_key[0]:
            best_key = (u_min, t, g_min)
            owner = g_min // R
            if owner == rank:
                x, y = engine.get_model(g_min - rank * R)
                x_best.copy_(torch.as_tensor(np.asarray(x, dtype=np.int8)))
                y_best.copy_(torch.as_tensor(np.asarray(y, dtype=np.float32)))
            dist.broadcast(x_best, src=owner, group=group)                 # C3
            dist.broadcast(y_best, src=owner, group=group)
        if u_min == 0:
            break
    return DistResult(SAT if best_key[0] == 0 else UNKNOWN, x_best.cpu().numpy(), y_best.cpu().numpy(),
                      best_key[2], best_key[1], best_key[0], stages)
