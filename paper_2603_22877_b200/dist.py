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


def solve_constraint_sharded(engine, n_bool: int, n_real: int, restarts: int, steps: int, seed: int, kappas,
                             eta: float, eps: float, group=None) -> DistResult:
    """Constraint-sharded solve (BASELINE config 5): every rank holds all R
    restarts and sweeps only its share of the constraints (engine.shard(rank, world, 1)).
    Per PGD step the partial gradients and objectives are all-reduced (C4: SUM over
    R*(n_bool+n_real) f64 + R f64), then every rank applies the identical K3 update; per
    stage the partial violation counts are all-reduced (C5: SUM over R u32).  All ranks
    therefore keep bit-identical states and reach the same verdict.

    engine: shard, begin, bind_buffers(ga, gb, obj, unsat), sweep(kappa, t), update(eta, eps),
    stage_end(t, copy=False), get_model(r).
    """
    rank = dist.get_rank(group)
    world = dist.get_world_size(group)
    dev = _device_for_backend()
    R = int(restarts)
    engine.shard(rank, world, 1)
    engine.begin(R, seed, 0)
    ga = torch.zeros((n_bool, R), dtype=torch.float64, device=dev)
    gb = torch.zeros((n_real, R), dtype=torch.float64, device=dev)
    obj = torch.zeros(R, dtype=torch.float64, device=dev)
    unsat = torch.zeros(R, dtype=torch.int32, device=dev)
    engine.bind_buffers(ga, gb, obj, unsat)
    best = None
    stages = 0
    for t, kappa in enumerate(kappas, start=1):
        for _ in range(steps):
            engine.sweep(float(kappa), t)
            for buf in (ga, gb, obj):                                    # C4
                dist.all_reduce(buf, op=dist.ReduceOp.SUM, group=group)
            engine.update(eta, eps)
        engine.stage_end(t, copy=False)
        dist.all_reduce(unsat, op=dist.ReduceOp.SUM, group=group)          # C5
        stages = t
        u = unsat.cpu().numpy()
        r = int(np.argmin(u))
        if best is None or int(u[r]) < best[0]:
            x, y = engine.get_model(r)
            best = (int(u[r]), t, r, np.asarray(x, dtype=np.int8).copy(), np.asarray(y, dtype=np.float32).copy())
        if best[0] == 0:
            break
    return DistResult(SAT if best[0] == 0 else UNKNOWN, best[3], best[4], best[2], best[1], best[0], stages)
