"""Multi-GPU drivers: one process per GPU over torch.distributed.

Restart-sharded (the default, `solve_restart_sharded`).  The paper runs 8 independent seeded
replicas, one per GPU.  Here the restarts of one solve are sharded instead:
rank k owns global restarts [k*R, (k+1)*R) (Philox counters use the global id, and every
restart's sums are exact (fsmt_sweep's on-grid accumulation), so each restart's trajectory is
bit-identical whatever the sharding).  There is no data-path collective; per stage the ranks
exchange one int64 (C1/C2: all-reduce MIN of (unsat << 32 | global restart)) and, when the best
model improves, the owning rank broadcasts it (C3: x int8[n_bool] + y f32[n_real]).  The winner
is the lexicographically smallest (stage, restart) with unsat = 0, else the smallest (unsat,
stage, restart) -- identical to a single process running all restarts.

Constraint-sharded (`solve_constraint_sharded`, BASELINE config 5): every rank holds all R
restarts and sweeps / checks only its share of the constraints (fsmt_shard mode 1).  Per PGD
step ONE all-reduce SUM of a flat f64 buffer [grad_a | grad_b | obj] (C4); per stage unsat
(SUM) and umax (MAX, the ERWA weight shift) (C5).  The gradient partial sums are integers in
grid units and the objective partials multiples of one power of two (kernels.hpp FxScale), so
the all-reduced sums are exact in any reduction order: every rank holds the single-GPU values
bit for bit and applies the identical K3 update.

`engine` is anything with the Solver step API (on GPU ranks a paper_2603_22877_b200.Solver):
restart-sharded: begin(R, seed, restart_offset), run_stage(t, kappa, steps) -> (unsat[R], min),
get_model(r) -> (x, y); constraint-sharded additionally shard, bind_buffers, sweep, step_sizes,
update, stage_end.  A GPU engine runs its kernels on torch's current stream (bound here), so
NCCL collectives on that stream are ordered after them without a host synchronisation.
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


def _comm_device():
    return torch.device("cuda", torch.cuda.current_device()) if dist.get_backend() == "nccl" else torch.device("cpu")


def _is_gpu_engine(engine) -> bool:
    return hasattr(engine, "device_buffers")     # paper_2603_22877_b200.Solver


def _bind_torch_stream(engine):
    if _is_gpu_engine(engine) and torch.cuda.is_available():
        engine.bind_stream(torch.cuda.current_stream().cuda_stream)


class RestartShardedStage:
    """Per-stage exchange of the restart-sharded solve (C1-C3), shared by solve_restart_sharded
    and bench.py's multi-rank step: after a stage, `exchange(t, unsat)` all-reduces the best
    (unsat, global restart), broadcasts an improved model from its owner, and returns the global
    minimum unsat."""

    def __init__(self, engine, n_bool: int, n_real: int, restarts_per_rank: int, group=None, keep_model=True):
        self.engine, self.group, self.keep_model = engine, group, keep_model
        self.rank = dist.get_rank(group)
        self.R = int(restarts_per_rank)
        dev = _comm_device()
        self.best_key = None            # (unsat, stage, global restart)
        self.x_best = torch.zeros(n_bool, dtype=torch.int8, device=dev)
        self.y_best = torch.zeros(n_real, dtype=torch.float32, device=dev)
        self.key_t = torch.zeros(1, dtype=torch.int64, device=dev)

    def exchange(self, t: int, unsat) -> int:
        r_loc = int(np.argmin(unsat))                              # first minimum = lowest restart id
        self.key_t.fill_((int(unsat[r_loc]) << 32) | (self.rank * self.R + r_loc))
        dist.all_reduce(self.key_t, op=dist.ReduceOp.MIN, group=self.group)      # C1 + C2
        k = int(self.key_t.item())
        u_min, g_min = k >> 32, k & 0xFFFFFFFF
        if self.best_key is None or u_min < self.best_key[0]:
            self.best_key = (u_min, t, g_min)
            if self.keep_model:
                owner = g_min // self.R
                if owner == self.rank:
                    x, y = self.engine.get_model(g_min - self.rank * self.R)
                    self.x_best.copy_(torch.as_tensor(np.asarray(x, dtype=np.int8)))
                    self.y_best.copy_(torch.as_tensor(np.asarray(y, dtype=np.float32)))
                dist.broadcast(self.x_best, src=owner, group=self.group)          # C3
                dist.broadcast(self.y_best, src=owner, group=self.group)
        return u_min


def solve_restart_sharded(engine, n_bool: int, n_real: int, restarts_per_rank: int, steps: int, seed: int,
                          kappas, group=None) -> DistResult:
    rank = dist.get_rank(group)
    R = int(restarts_per_rank)
    _bind_torch_stream(engine)
    engine.begin(R, seed, restart_offset=rank * R)
    ex = RestartShardedStage(engine, n_bool, n_real, R, group)
    stages = 0
    for t, kappa in enumerate(kappas, start=1):
        unsat, _ = engine.run_stage(t, float(kappa), steps)
        stages = t
        if ex.exchange(t, unsat) == 0:
            break
    bk = ex.best_key
    return DistResult(SAT if bk[0] == 0 else UNKNOWN, ex.x_best.cpu().numpy(), ex.y_best.cpu().numpy(),
                      bk[2], bk[1], bk[0], stages)


class ConstraintShardedBuffers:
    """The bound buffers of a constraint-sharded engine and their collectives (C4, C5).

    grads = one flat f64 [n_bool*R | n_real*R | R | slot_rows*R] (grad_a, grad_b, obj and the
    symmetric classes' slot-table rows) all-reduced with ONE call per PGD step, after which the engine
    chains the rows (sweep_finish); unsat / umax int32 [R] per stage.  A GPU engine under a CPU backend (gloo)
    keeps device buffers and stages each collective through host memory (the library rejects host
    buffers); a CPU engine (tests) binds the communication tensors directly."""

    def __init__(self, engine, n_bool: int, n_real: int, R: int, group=None, nvls: bool = False):
        self.group = group
        self.engine = engine
        comm = _comm_device()
        gpu = _is_gpu_engine(engine)
        bind = torch.device("cuda", torch.cuda.current_device()) if gpu else comm
        rows = engine.get_dims().get("n_slot_rows", 0) if gpu else 0
        n = (n_bool + n_real + 1 + rows) * R
        self.n = n
        # nvls: the flat buffer is symmetric memory with a multicast address and C4 is the library's
        # in-switch all-reduce (fsmt_mc_allreduce_f64) between two device barriers instead of NCCL
        self.symm = None
        if nvls:
            if not (gpu and dist.get_backend(group) == "nccl"):
                raise RuntimeError("nvls needs a GPU engine under the NCCL backend")
            import torch.distributed._symmetric_memory as symm_mem
            self.flat = symm_mem.empty(n, dtype=torch.float64, device=bind)
            self.flat.zero_()
            gname = (group or dist.group.WORLD).group_name
            self.symm = symm_mem.rendezvous(self.flat, gname)
            if not self.symm.multicast_ptr:
                raise RuntimeError("nvls: no multicast support on this group (needs >= 2 GPUs behind NVSwitch)")
        else:
            self.flat = torch.zeros(n, dtype=torch.float64, device=bind)
        self.unsat = torch.zeros(R, dtype=torch.int32, device=bind)
        self.umax = torch.zeros(R, dtype=torch.int32, device=bind)
        self.stage = bind != comm
        if self.stage:
            self.flat_c = torch.zeros(n, dtype=torch.float64, device=comm)
            self.unsat_c = torch.zeros(R, dtype=torch.int32, device=comm)
            self.umax_c = torch.zeros(R, dtype=torch.int32, device=comm)
        ga = self.flat[: n_bool * R].view(n_bool, R)
        gb = self.flat[n_bool * R:(n_bool + n_real) * R].view(n_real, R)
        obj = self.flat[(n_bool + n_real) * R:(n_bool + n_real + 1) * R]
        engine.bind_buffers(ga, gb, obj, self.unsat, self.umax)
        if rows:
            engine.bind_slot_grads(self.flat[(n_bool + n_real + 1) * R:].view(rows, R))
        self.chain = rows > 0

    def _reduce(self, dev_t, comm_t, op):
        if self.stage:
            comm_t.copy_(dev_t)                    # synchronising D2H on torch's (= the engine's) stream
            dist.all_reduce(comm_t, op=op, group=self.group)
            dev_t.copy_(comm_t)
        else:
            dist.all_reduce(dev_t, op=op, group=self.group)

    def reduce_grads(self):                                                       # C4
        if self.symm is not None:
            self.symm.barrier(channel=0)           # every rank's sweep has written its copy
            self.engine.mc_allreduce_f64(self.symm.multicast_ptr, self.n, dist.get_rank(self.group),
                                         dist.get_world_size(self.group))
            self.symm.barrier(channel=1)           # every rank's multicast stores have landed
        else:
            self._reduce(self.flat, self.flat_c if self.stage else None, dist.ReduceOp.SUM)
        if self.chain:
            self.engine.sweep_finish()

    def reduce_stage(self):                                                       # C5
        self._reduce(self.unsat, self.unsat_c if self.stage else None, dist.ReduceOp.SUM)
        self._reduce(self.umax, self.umax_c if self.stage else None, dist.ReduceOp.MAX)


def solve_constraint_sharded(engine, n_bool: int, n_real: int, restarts: int, steps: int, seed: int, kappas,
                             eps: float, group=None, nvls: bool = False) -> DistResult:
    """Constraint-sharded Alg.2 (BASELINE config 5); step sizes per stage from the
    engine's params (engine.step_sizes(kappa): eta and eta_mode, as fsmt_run_stage uses them)."""
    rank = dist.get_rank(group)
    world = dist.get_world_size(group)
    R = int(restarts)
    _bind_torch_stream(engine)
    engine.shard(rank, world, 1)
    engine.begin(R, seed, 0)
    bufs = ConstraintShardedBuffers(engine, n_bool, n_real, R, group, nvls=nvls)
    best = None
    stages = 0
    for t, kappa in enumerate(kappas, start=1):
        eta_a, eta_b = engine.step_sizes(float(kappa))
        for _ in range(steps):
            engine.sweep(float(kappa), t)
            bufs.reduce_grads()
            engine.update(eta_a, eps, eta_b=eta_b)
        engine.stage_end(t, copy=False)
        bufs.reduce_stage()
        stages = t
        u = bufs.unsat.cpu().numpy()
        r = int(np.argmin(u))
        if best is None or int(u[r]) < best[0]:
            x, y = engine.get_model(r)
            best = (int(u[r]), t, r, np.asarray(x, dtype=np.int8).copy(), np.asarray(y, dtype=np.float32).copy())
        if best[0] == 0:
            break
    return DistResult(SAT if best[0] == 0 else UNKNOWN, best[3], best[4], best[2], best[1], best[0], stages)
