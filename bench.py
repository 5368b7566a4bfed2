#!/usr/bin/env python
"""FourierSMT hot-path benchmark (BASELINE.json metric: xBDD COP+grad evals/s).

A bench *step* is one pass of the whole hot path over the synthetic workload: one
annealing stage of Alg.2 for all restarts = S PGD steps (each: K1 sweep
= slot probabilities + smoothing + forward/backward xBDD pass + gradient accumulation,
then K3 projected update with the eps test) followed by K4 rounding and K5 exact
verification + ERWA counter update, ending in the per-stage exchange of the multi-GPU
driver (restart-sharded: C1/C2 best-(unsat, restart) all-reduce + C3 model broadcast,
paper_2603_22877_b200.dist.RestartShardedStage; constraint-sharded: C4 one flat gradient
all-reduce per PGD step + C5 per stage).
value = constraints x restarts x S x K / time, whole job (all ranks).

Workload (N=1): cfg4 "placement-10k" = 10,656 vars / 705,072 constraints, R = 1,024
restarts per GPU (restart mode: weak scaling, global restart ids rank*R + r; constraint mode,
BASELINE config 5: R restarts in total, constraints split over the ranks, strong scaling).

  python bench.py [--gpus N] [--steps K] [--warmup W] [--config cfg4] [--restarts R]
                  [--pgd-steps S] [--mode restart|constraint] [--impl reference]

--gpus N > 1 without torchrun re-launches itself under torch.distributed.run with N ranks
(one per GPU, NCCL, 127.0.0.1); under torchrun WORLD_SIZE must equal N.
"""
from __future__ import annotations

import argparse
import json
import math
import os
import platform
import socket
import statistics
import subprocess
import sys
import threading
import time

ROOT = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, ROOT)

SURVEY_BYTES_PER_EVAL = {"cfg4": 194.0, "cfg3": 98.9, "cfg2": 194.0}    # SURVEY §8(d) + 1 B (U is u16), per (c, r)
FMA_PER_EVAL = {"cfg4": 264.0, "cfg3": 142.0, "cfg2": 480.0,            # SURVEY §8(d) model
                "place9856": 296.0}   # the same model for 9 bit pairs + 4 atoms: 31 nodes x 6 + 22 slots + 4 x 22
KAPPA = 1.0                                                              # fixed kappa, t = 1
METRIC = "xBDD COP+grad evals/s (constraints x restarts)"
TTS_KAPPAS = [300.0 ** (i / 19) for i in range(20)] + [300.0] * 200     # DESIGN.md §9 recipe


def parse_args():
    p = argparse.ArgumentParser()
    p.add_argument("--gpus", type=int, default=1)
    p.add_argument("--steps", type=int, default=5)
    p.add_argument("--warmup", type=int, default=3)
    p.add_argument("--config", default="cfg4")
    p.add_argument("--restarts", type=int, default=1024)
    p.add_argument("--pgd-steps", type=int, default=8)
    p.add_argument("--mode", default="restart", choices=["restart", "constraint"])
    p.add_argument("--nvls", action="store_true", help="constraint mode: C4 as the in-switch multicast all-reduce "
                   "(fsmt_mc_allreduce_f64 on symmetric memory) instead of NCCL")
    p.add_argument("--impl", default="ours", choices=["ours", "reference"])
    p.add_argument("--no-e2e", action="store_true")
    p.add_argument("--no-cpu-baseline", action="store_true")
    p.add_argument("--no-prepare", action="store_true", help="generic kernels (no fsmt_prepare(R))")
    p.add_argument("--no-tts", action="store_true", help="skip the time-to-SAT fields (cfg4, N=1)")
    return p.parse_args()


def _free_port() -> int:
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    p = s.getsockname()[1]
    s.close()
    return p


def maybe_relaunch(args) -> bool:
    """--gpus N > 1 outside torchrun: re-exec under torch.distributed.run (N ranks).  Returns True
    when this process only launched the ranks (their rank 0 printed the line)."""
    world = os.environ.get("WORLD_SIZE")
    if world is not None:
        if int(world) != args.gpus:
            sys.exit(f"bench.py: --gpus {args.gpus} but WORLD_SIZE={world}")
        return False
    if args.gpus <= 1:
        return False
    cmd = [sys.executable, "-m", "torch.distributed.run", "--nnodes=1", f"--nproc-per-node={args.gpus}",
           "--master-addr", "127.0.0.1", "--master-port", str(_free_port()), os.path.abspath(__file__)] + sys.argv[1:]
    rc = subprocess.call(cmd)
    if rc:
        sys.exit(rc)
    return True


def peaks():
    try:
        with open(os.path.join(ROOT, "MEASURED_PEAKS.json")) as fh:
            d = json.load(fh)
        return float(d["hbm_gbs"]), "measured (MEASURED_PEAKS.json)", float(d.get("sm_max_mhz", 1965.0))
    except Exception:
        return 6650.0, "fallback (B200_PROFILING.md)", 1965.0


class ClockSampler:
    """nvidia-smi clocks + throttle reasons sampled during the timed region."""
    Q = ("index,clocks.sm,clocks.max.sm,power.draw,clocks_event_reasons.active,clocks_event_reasons.hw_slowdown,"
         "clocks_event_reasons.hw_thermal_slowdown,clocks_event_reasons.sw_thermal_slowdown,"
         "clocks_event_reasons.sw_power_cap")

    def __init__(self, device_index: int):
        self.dev = device_index
        self.rows = []
        self.proc = None

    def __enter__(self):
        try:
            self.proc = subprocess.Popen(["nvidia-smi", f"--id={self.dev}", f"--query-gpu={self.Q}",
                                          "--format=csv,noheader,nounits", "-lms", "200"],
                                         stdout=subprocess.PIPE, stderr=subprocess.DEVNULL, text=True)
            self.th = threading.Thread(target=self._read, daemon=True)
            self.th.start()
        except Exception:
            self.proc = None
        return self

    def _read(self):
        for line in self.proc.stdout:
            self.rows.append([x.strip() for x in line.split(",")])

    def __exit__(self, *a):
        if self.proc is not None:
            self.proc.terminate()
            try:
                self.proc.wait(timeout=5)
            except Exception:
                self.proc.kill()

    def summary(self):
        sm = []
        smax = None
        reasons = set()
        names = ["hw_slowdown", "hw_thermal_slowdown", "sw_thermal_slowdown", "sw_power_cap"]
        for r in self.rows:
            try:
                sm.append(float(r[1]))
                smax = float(r[2])
                for n, v in zip(names, r[5:9]):
                    if v.strip().lower() == "active":
                        reasons.add(n)
            except (ValueError, IndexError):
                continue
        if not sm:
            return {"sm_mhz": None, "sm_max_mhz": None, "reasons": ["unsampled"], "samples": 0}
        return {"sm_mhz": statistics.median(sm), "sm_max_mhz": smax, "reasons": sorted(reasons), "samples": len(sm)}


# ----------------------------------------------------------------------------------- CPU oracle

_OS = {}      # the oracle sample, inherited by forked workers


def _oracle_chunk(args):
    from oracle import objective
    lo, hi = args
    f, pts, kappa = _OS["f"], _OS["pts"], _OS["kappa"]
    for a, b in pts:
        objective.objective_and_gradient_grouped(f, a, b, kappa, subset=range(lo, hi))
    return (hi - lo) * len(pts)


def cpu_model() -> str:
    try:
        with open("/proc/cpuinfo") as fh:
            for ln in fh:
                if ln.startswith("model name"):
                    return ln.split(":", 1)[1].strip()
    except OSError:
        pass
    return platform.processor() or "unknown"


class OracleSample:
    """A bounded sample of the workload for the fp64 CPU oracle (test infrastructure; the
    bench's cpu_baseline and --impl reference legs only): the first n constraints of the config,
    SURVEY §8(d)'s 4 sampled restarts (seeded points), objective + gradient per restart with the
    oracle's grouped sparse-WFE path, split into constraint chunks over all host cores."""

    def __init__(self, inst, n_cons: int, restarts: int = 4, kappa: float = KAPPA):
        import numpy as np
        from tests.helpers import subformula
        from oracle import hsmt
        sub, keep = subformula(inst.text, extra_constraints=range(min(n_cons, inst.n_cons)))
        f = hsmt.parse(sub)
        rng = np.random.default_rng(0)
        lo = 0.0 if inst.name.startswith("cfg4") else -1.0
        pts = [(rng.uniform(-1, 1, f.n_bool), rng.uniform(lo, 1, f.n_real)) for _ in range(restarts)]
        _OS.update(f=f, pts=pts, kappa=kappa)
        self.n = len(keep)
        self.restarts = restarts
        self.cores = os.cpu_count() or 1

    def run(self, cores: int | None = None) -> tuple[float, int]:
        """(wall seconds, evals) of one pass over the sample on `cores` processes (fork)."""
        import multiprocessing as mp
        cores = cores or self.cores
        edges = [self.n * k // (cores * 4) for k in range(cores * 4 + 1)]
        chunks = [(lo, hi) for lo, hi in zip(edges[:-1], edges[1:]) if hi > lo]
        t0 = time.perf_counter()
        if cores == 1:
            evals = sum(_oracle_chunk(c) for c in chunks)
        else:
            with mp.get_context("fork").Pool(cores) as pool:
                evals = sum(pool.map(_oracle_chunk, chunks))
        return time.perf_counter() - t0, evals


def oracle_sample_size(cores: int) -> int:
    """~6,000 constraints x 4 restarts per core: about 15 s of oracle work per pass."""
    return 6000 * max(1, cores)


def cpu_baseline(inst, config: str) -> dict:
    cores = os.cpu_count() or 1
    smp = OracleSample(inst, oracle_sample_size(cores))
    smp.run()                                               # warm (page-in, imports)
    wall, evals = smp.run()
    one = OracleSample(inst, 1500, restarts=1)
    w1, e1 = one.run(cores=1)
    return {"value": evals / wall, "unit": "evals/s", "cores": cores, "kind": "oracle",
            "cpu_model": cpu_model(), "one_thread_value": e1 / w1,
            "sample": f"first {smp.n} constraints of {config} x {smp.restarts} seeded restarts, fp64 oracle "
                      f"(grouped sparse xWFE) objective+gradient, constraint chunks over {cores} processes "
                      f"({wall:.1f} s); one_thread_value: first {one.n} constraints x 1 restart on 1 process"}


def time_to_sat(P, inst, device: int, R: int, seeds=range(8)) -> dict:
    """BASELINE metric, second half: fsmt_solve wall time from call to verified return on this
    instance (load/build/prepare excluded), median over 8 seeds, with the DESIGN.md §9
    recipe; one untimed warm-up solve first (module loading)."""
    s = P.Solver(device)
    s.load_formula(inst.text)
    s.build_xbdd()
    s.prepare(R)
    s.set_params(kappas=TTS_KAPPAS, eta=0.4, eta_mode=3, erwa_mode=1, time_limit_s=1000.0)
    s.solve(R, 2, 10_000)
    times, solved = [], 0
    for seed in seeds:
        res = s.solve(R, 2, seed)
        ok = res.verdict == P.SAT and s.verify(res.x, res.y) == 0
        solved += ok
        times.append(res.stats["solve_ms"] / 1e3 if ok else float("inf"))
    med = statistics.median(times)
    return {"median_s": med if math.isfinite(med) else None, "max_s": max(times) if solved == len(times) else None,
            "solved": solved, "seeds": len(times), "restarts": R, "steps_per_stage": 2,
            "recipe": "eta 0.4 (eta_mode 3), ERWA reset-to-0, kappa 1->300 over 20 stages then held 200"}


def workload_config(args, n_vars: int, n_cons: int, world: int = 1) -> dict:
    """The workload both arms name in `config` (same keys, so the driver compares like with like)."""
    names = {"cfg4": "placement-10k", "cfg3": "scheduling-2k", "cfg2": "random-200",
             "place9856": "paper placement n_m=64 n_l=8 with routing"}
    g = args.restarts * world if args.mode == "restart" else args.restarts
    return {"workload": f"{args.config}: {names.get(args.config, args.config)}, {n_vars} vars / {n_cons} constraints",
            "restarts_per_gpu": args.restarts if args.mode == "restart" else None, "global_restarts": g,
            "pgd_steps_per_stage": args.pgd_steps, "kappa": KAPPA, "mode": args.mode}


def run_reference(args):
    """--impl reference: the fp64 oracle as it stands, on all host cores, same metric/config."""
    if int(os.environ.get("RANK", "0")) != 0:
        return
    import fsmt_gen
    inst = fsmt_gen.config(args.config)
    cores = os.cpu_count() or 1
    smp = OracleSample(inst, oracle_sample_size(cores) // 3)
    for _ in range(args.warmup):
        smp.run()
    ts, ev = [], 0
    for _ in range(args.steps):
        w, e = smp.run()
        ts.append(w)
        ev += e
    total = sum(ts)
    value = ev / total
    sample = (f"first {smp.n} constraints of {args.config} x {smp.restarts} seeded restarts per step, fp64 oracle "
              f"objective+gradient over {cores} processes")
    line = {
        "impl": "reference", "metric": METRIC, "value": value, "unit": "evals/s", "n_gpus": args.gpus,
        "steps": args.steps, "warmup": args.warmup, "ms_per_step": 1e3 * total / len(ts), "higher_is_better": True,
        "scaling": "weak" if args.mode == "restart" else "strong", "vs_baseline": None, "dtype": "f64",
        "data": "synthetic",
        "config": {**workload_config(args, inst.n_bool + inst.n_real, inst.n_cons, args.gpus), "oracle_sample": sample},
        "cpu_baseline": {"value": value, "unit": "evals/s", "cores": cores, "kind": "oracle", "cpu_model": cpu_model(),
                         "sample": sample},
        "e2e": {"value": value, "unit": "evals/s", "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0},
    }
    print(json.dumps(line), flush=True)


# ----------------------------------------------------------------------------------- GPU arm


def main():
    args = parse_args()
    if args.impl == "reference":
        return run_reference(args)
    if maybe_relaunch(args):
        return
    import numpy as np
    import torch
    import torch.distributed as dist

    world = int(os.environ.get("WORLD_SIZE", "1"))
    rank = int(os.environ.get("RANK", "0"))
    local = int(os.environ.get("LOCAL_RANK", "0"))
    if world > 1:
        # communicator init lines (NCCL INFO) on stderr, so the driver can check comm_nranks
        os.environ.setdefault("NCCL_DEBUG", "INFO")
        os.environ.setdefault("NCCL_DEBUG_SUBSYS", "INIT")
        os.environ.setdefault("NCCL_DEBUG_FILE", "/dev/stderr")
        torch.cuda.set_device(local)
        dist.init_process_group("nccl", device_id=torch.device("cuda", local))
    torch.cuda.set_device(local)
    import paper_2603_22877_b200 as P
    from paper_2603_22877_b200 import dist as D
    import fsmt_gen

    inst = fsmt_gen.config(args.config)
    s = P.Solver(local)
    t0 = time.perf_counter()
    s.load_formula(inst.text)
    s.build_xbdd()
    R = args.restarts
    if not args.no_prepare:
        s.prepare(R)                  # kernels specialised for R restarts (part of the build)
    build_s = time.perf_counter() - t0
    jit_status = s.jit_info()["status"]    # e.g. "active; prepared R=1024 k1 cap=28" (register cap chosen)
    dims = s.get_dims()
    S = args.pgd_steps
    s.set_params(eta=0.01, eps=1e-2)
    stream = torch.cuda.current_stream()
    s.bind_stream(stream.cuda_stream)
    constraint_mode = args.mode == "constraint" and world > 1
    if constraint_mode:
        s.shard(rank, world, 1)
        s.begin(R, seed=12345, restart_offset=0)
        bufs = D.ConstraintShardedBuffers(s, dims["n_bool"], dims["n_real"], R, nvls=args.nvls)
        eta_a, eta_b = s.step_sizes(KAPPA)

        def step(t):
            for _ in range(S):                              # K1 (shard) + C4 + K3
                s.sweep(KAPPA, t)
                bufs.reduce_grads()
                s.update(eta_a, 1e-2, eta_b=eta_b)
            s.stage_end(t, copy=False)                      # K4 + K5 (shard) + C5
            bufs.reduce_stage()
    else:
        s.begin(R, seed=12345, restart_offset=rank * R)
        ex = D.RestartShardedStage(s, dims["n_bool"], dims["n_real"], R) if world > 1 else None

        def step(t):
            unsat, mn = s.run_stage(t, KAPPA, S)           # S x (K1 + K3), K4 + K5; unsat[R] to host
            if ex is not None:
                ex.exchange(t, unsat)                       # C1/C2 (+ C3 when the best model improves)

    for w in range(args.warmup):
        step(1)
    s.set_timing(True)
    s.get_timing(reset=True)
    if world > 1:
        dist.barrier()
    torch.cuda.synchronize()
    launches0 = s.kernel_launches()
    ev0 = torch.cuda.Event(enable_timing=True)
    ev1 = torch.cuda.Event(enable_timing=True)
    with ClockSampler(local) as clk:
        ev0.record(stream)
        for k in range(args.steps):
            step(1)
        ev1.record(stream)
        torch.cuda.synchronize()
    if world > 1:
        dist.barrier()
    ms = ev0.elapsed_time(ev1)
    launches = s.kernel_launches() - launches0
    timing = s.get_timing(reset=True)
    s.set_timing(False)
    t_max = torch.tensor([ms], dtype=torch.float64, device="cuda")
    if world > 1:
        dist.all_reduce(t_max, op=dist.ReduceOp.MAX)
    ms_max = float(t_max.item())
    units = dims["n_cons"] * R * S * args.steps * (1 if constraint_mode else world)   # whole job
    value = units / (ms_max / 1e3)

    # e2e: through the C ABI with HOST buffers: H2D of the step's state, stage, D2H of the result
    e2e = None
    if not args.no_e2e and not constraint_mode:
        a_h = torch.empty((dims["n_bool"], R), dtype=torch.float32).pin_memory()
        b_h = torch.empty((dims["n_real"], R), dtype=torch.float32).pin_memory()
        a_np, b_np = a_h.numpy(), b_h.numpy()
        s.bind_stream(None)
        st_a, st_b = s.get_state()
        a_np[...] = st_a
        b_np[...] = st_b
        if world > 1:
            dist.barrier()
        torch.cuda.synchronize()
        te0 = time.perf_counter()
        for k in range(args.steps):
            s.set_state(a_np, b_np)                    # H2D from pinned host memory
            unsat, mn = s.run_stage(1, KAPPA, S)       # D2H of unsat[R] inside run_stage
        te = time.perf_counter() - te0
        te_t = torch.tensor([te], dtype=torch.float64, device="cuda")
        if world > 1:
            dist.all_reduce(te_t, op=dist.ReduceOp.MAX)
        h2d = (dims["n_bool"] + dims["n_real"]) * R * 4
        e2e = {"value": units / float(te_t.item()), "unit": "evals/s",
               "h2d_bytes_per_step": h2d, "d2h_bytes_per_step": R * 4}

    # roofline for the dominant kernel (K1) from live per-launch CUDA-event timing
    k1_ms, k1_n = timing["k1_sweep"]
    hbm, peak_src, sm_max = peaks()
    k1_avg_s = (k1_ms / max(k1_n, 1)) / 1e3
    evals_per_launch = dims["n_cons"] * R / (world if constraint_mode else 1)
    bpe = SURVEY_BYTES_PER_EVAL.get(args.config, 194.0)
    achieved = bpe * evals_per_launch / k1_avg_s / 1e9
    traffic = None
    prof = os.path.join(ROOT, "profiles", f"k1_traffic_{args.config}.json")
    if os.path.exists(prof) and not constraint_mode and R == 1024:
        try:
            traffic = json.load(open(prof)).get("dram_bytes_per_launch")
        except Exception:
            traffic = None
    fma_pe = FMA_PER_EVAL.get(args.config, 264.0)
    alu_achieved = 2.0 * fma_pe * evals_per_launch / k1_avg_s / 1e12
    alu_peak = 148 * 128 * 2 * sm_max * 1e6 / 1e12
    clocks = clk.summary()
    if rank == 0:
        line = {
            "metric": METRIC, "value": value, "unit": "evals/s", "n_gpus": world, "steps": args.steps,
            "warmup": args.warmup, "ms_per_step": ms_max / args.steps, "higher_is_better": True,
            "scaling": "strong" if constraint_mode else "weak",
            "vs_baseline": None, "dtype": "f32", "data": "synthetic",
            "config": {**workload_config(args, dims["n_bool"] + dims["n_real"], dims["n_cons"], world),
                       "kernels": "generic" if args.no_prepare else "specialised for R (fsmt_prepare)",
                       "parallelism": (f"constraint-sharded x{world} (one flat {'NVLS multicast' if args.nvls else 'NCCL'} all-reduce per PGD step)" if constraint_mode
                                       else f"restart-sharded x{world}"),
                       "l2": "inputs exceed L2 (u16 U counters %.0f MB + structure + state per step)" % (dims["n_cons"] * R * 2 / 1e6),
                       "accumulation": "fp64, exact on-grid sums (deterministic)", "build_s": round(build_s, 2),
                       "jit": jit_status},
            "roofline": {"bound": "alu", "achieved": alu_achieved, "peak": alu_peak, "unit": "TFLOP/s",
                         "frac": alu_achieved / alu_peak, "traffic": traffic, "kernel": ("fsmt_k1_jit (the JIT sweep; cfg4's 1-slot bound class runs as fsmt_k1_c1 on an auxiliary stream)"
                                    if args.config == "cfg4" else "fsmt_k1_jit / fsmt_k1_c<k> (JIT sweep kernels)"),
                         "basis": f"SURVEY 8(d) model {fma_pe:.0f} FMA-eq (x2 flop) per (constraint,restart) eval x "
                                  f"{evals_per_launch:.0f} evals per launch / live CUDA-event launch time; peak = 148 SMs x "
                                  f"128 FP32 lanes x 2 x {sm_max:.0f} MHz (DESIGN.md §7)",
                         "k1_ms_per_launch": k1_ms / max(k1_n, 1),
                         "k1_share_of_step": k1_ms / ms if ms > 0 else None,
                         "hbm": {"algorithmic_gbs": achieved, "algorithmic_bytes_per_eval": bpe,
                                 "actual_gbs": (traffic / k1_avg_s / 1e9) if traffic else None, "peak_gbs": hbm,
                                 "peak_src": peak_src, "note": "SURVEY 8(d) effective-bandwidth gate; restart tiles "
                                 "share each structure fetch, so actual DRAM traffic is far below the algorithmic bytes"}},
            "kernel_ms": {k: {"total_ms": v[0], "groups": v[1]} for k, v in timing.items()},
            "clocks": clocks,
            "e2e": e2e,
            "gpu_launches": int(launches),
        }
        if not args.no_cpu_baseline and world == 1:
            try:
                line["cpu_baseline"] = cpu_baseline(inst, args.config)
            except Exception as e:  # the baseline must never kill the bench line
                line["cpu_baseline"] = {"value": None, "unit": "evals/s", "cores": os.cpu_count(), "kind": "oracle",
                                        "sample": f"failed: {e}"}
        if not args.no_tts and world == 1 and args.config == "cfg4":
            for key, Rt in (("time_to_sat", 32), ("time_to_sat_r1024", 1024)):
                try:
                    line[key] = time_to_sat(P, inst, local, Rt)
                except Exception as e:  # never kill the bench line
                    line[key] = {"median_s": None, "note": f"failed: {e}"}
        print(json.dumps(line), flush=True)
    if world > 1:
        dist.destroy_process_group()


if __name__ == "__main__":
    main()
