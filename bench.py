#!/usr/bin/env python
"""FourierSMT hot-path benchmark (BASELINE.json metric: xBDD COP+grad evals/s).

A bench *step* is one pass of the whole hot path over the synthetic workload: one
annealing stage of Alg.2 for all restarts = S PGD steps (each: K1 sweep
= slot probabilities + smoothing + forward/backward xBDD pass + gradient accumulation,
then K3 projected update with the eps test) followed by K4 rounding and K5 exact
verification + ERWA counter update, ending in the 4-byte found-flag exchange (C1).
value = constraints x restarts x S x K / time, whole job (all ranks).

Workload (N=1): cfg4 "placement-10k" = 10,656 vars / 705,072 constraints, R = 1,024
restarts per GPU (weak scaling: restart-sharded, global restart ids rank*R + r).

  python bench.py [--gpus N] [--steps K] [--warmup W] [--config cfg4] [--restarts R]
                  [--pgd-steps S] [--impl reference]
"""
from __future__ import annotations

import argparse
import json
import math
import os
import statistics
import subprocess
import sys
import threading
import time

ROOT = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, ROOT)

SURVEY_BYTES_PER_EVAL = {"cfg4": 193.0, "cfg3": 97.9, "cfg2": 193.0}    # SURVEY §8(d), per (c, r)
FMA_PER_EVAL = {"cfg4": 264.0, "cfg3": 142.0, "cfg2": 480.0}            # SURVEY §8(d) model
KAPPA = 1.0                                                              # fixed kappa, t = 1
METRIC = "xBDD COP+grad evals/s (constraints x restarts)"


def parse_args():
    p = argparse.ArgumentParser()
    p.add_argument("--gpus", type=int, default=1)
    p.add_argument("--steps", type=int, default=5)
    p.add_argument("--warmup", type=int, default=3)
    p.add_argument("--config", default="cfg4")
    p.add_argument("--restarts", type=int, default=1024)
    p.add_argument("--pgd-steps", type=int, default=8)
    p.add_argument("--impl", default="ours", choices=["ours", "reference"])
    p.add_argument("--no-e2e", action="store_true")
    p.add_argument("--no-cpu-baseline", action="store_true")
    p.add_argument("--no-prepare", action="store_true", help="generic kernels (no fsmt_prepare(R))")
    p.add_argument("--no-tts", action="store_true", help="skip the time-to-SAT field (cfg4, N=1)")
    return p.parse_args()


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


def oracle_sample(inst, n_cons_sample: int, seed: int = 0):
    """Bounded sample of the workload for the oracle: the first n constraints, one restart."""
    import numpy as np
    from tests.helpers import subformula
    from oracle import hsmt
    text = inst.text
    lines = text.splitlines()
    n_atoms_lines = sum(1 for ln in lines if ln.startswith("a "))
    # constraints are after the atoms; take the first n_cons_sample constraints
    sub, keep = subformula(text, extra_constraints=range(n_cons_sample))
    f = hsmt.parse(sub)
    rng = np.random.default_rng(seed)
    a = rng.uniform(-1, 1, f.n_bool)
    b = rng.uniform(0, 1, f.n_real)
    return f, a, b, len(keep)


def time_oracle(f, a, b, kappa=KAPPA):
    from oracle import objective
    t0 = time.perf_counter()
    objective.objective_and_gradient_grouped(f, a, b, kappa)
    return time.perf_counter() - t0


def time_to_sat(P, inst, device: int, seeds=range(8), R: int = 32) -> dict:
    """BASELINE metric, second half: fsmt_solve wall time from call to verified return on this
    instance (load/build/prepare excluded), median over 8 seeds, with the DESIGN.md §9
    recipe; one untimed warm-up solve first (module loading)."""
    s = P.Solver(device)
    s.load_formula(inst.text)
    s.build_xbdd()
    s.prepare(R)
    kappas = [300.0 ** (i / 19) for i in range(20)] + [300.0] * 200
    s.set_params(kappas=kappas, eta=0.4, eta_mode=3, erwa_mode=1, time_limit_s=1000.0)
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
    names = {"cfg4": "placement-10k", "cfg3": "scheduling-2k", "cfg2": "random-200"}
    return {"workload": f"{args.config}: {names.get(args.config, args.config)}, {n_vars} vars / {n_cons} constraints",
            "restarts_per_gpu": args.restarts, "global_restarts": args.restarts * world,
            "pgd_steps_per_stage": args.pgd_steps, "kappa": KAPPA}


def run_reference(args):
    """--impl reference: the fp64 oracle as it stands, on the host cores, same metric/config."""
    rank = int(os.environ.get("RANK", "0"))
    if rank != 0:
        return
    import fsmt_gen
    inst = fsmt_gen.config(args.config)
    n_sample = 1500 if args.config in ("cfg4", "cfg3") else min(inst.n_cons, 500)
    f, a, b, n = oracle_sample(inst, n_sample)
    for _ in range(args.warmup):
        time_oracle(f, a, b)
    ts = [time_oracle(f, a, b) for _ in range(args.steps)]
    total = sum(ts)
    value = n * len(ts) / total
    line = {
        "impl": "reference", "metric": METRIC, "value": value, "unit": "evals/s", "n_gpus": args.gpus,
        "steps": args.steps, "warmup": args.warmup, "ms_per_step": 1e3 * total / len(ts), "higher_is_better": True,
        "scaling": "weak", "vs_baseline": None, "dtype": "f64", "data": "synthetic",
        "config": {**workload_config(args, inst.n_bool + inst.n_real, inst.n_cons),
                   "oracle_sample": f"first {n} constraints, 1 restart, one objective+gradient evaluation per step"},
        "cpu_baseline": {"value": value, "unit": "evals/s", "cores": 1, "kind": "oracle",
                         "sample": f"first {n} constraints of {args.config}, 1 restart, objective+gradient per step"},
        "e2e": {"value": value, "unit": "evals/s", "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0},
    }
    print(json.dumps(line))


# ----------------------------------------------------------------------------------- GPU arm


def main():
    args = parse_args()
    if args.impl == "reference":
        return run_reference(args)
    import numpy as np
    import torch
    import torch.distributed as dist

    world = int(os.environ.get("WORLD_SIZE", "1"))
    rank = int(os.environ.get("RANK", "0"))
    local = int(os.environ.get("LOCAL_RANK", "0"))
    if world > 1:
        dist.init_process_group("nccl", device_id=torch.device("cuda", local))
    torch.cuda.set_device(local)
    import paper_2603_22877_b200 as P
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
    dims = s.get_dims()
    S = args.pgd_steps
    s.set_params(eta=0.01, eps=1e-2)
    stream = torch.cuda.current_stream()
    s.bind_stream(stream.cuda_stream)
    s.begin(R, seed=12345, restart_offset=rank * R)
    found = torch.zeros(1, dtype=torch.int32, device="cuda")

    def step(t):
        _, mn = s.run_stage(t, KAPPA, S, want_unsat=False)
        if world > 1:                                   # C1: early-exit flag, 4 bytes
            found.fill_(1 if mn == 0 else 0)
            dist.all_reduce(found, op=dist.ReduceOp.MAX)
        return mn

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
    evals_per_rank = dims["n_cons"] * R * S * args.steps
    value = evals_per_rank * world / (ms_max / 1e3)

    # e2e: through the C ABI with HOST buffers: H2D of the step's state, stage, D2H of the result
    e2e = None
    if not args.no_e2e:
        a_h = torch.empty((dims["n_bool"], R), dtype=torch.float32).pin_memory()
        b_h = torch.empty((dims["n_real"], R), dtype=torch.float32).pin_memory()
        a_np, b_np = a_h.numpy(), b_h.numpy()
        s.bind_stream(None)
        st_a, st_b = s.get_state()
        a_np[...] = st_a
        b_np[...] = st_b
        unsat = np.empty(R, dtype=np.uint32)
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
        e2e = {"value": evals_per_rank * world / float(te_t.item()), "unit": "evals/s",
               "h2d_bytes_per_step": h2d, "d2h_bytes_per_step": R * 4}

    # roofline for the dominant kernel (K1) from live per-launch CUDA-event timing
    k1_ms, k1_n = timing["k1_sweep"]
    hbm, peak_src, sm_max = peaks()
    k1_avg_s = (k1_ms / max(k1_n, 1)) / 1e3
    evals_per_launch = dims["n_cons"] * R
    bpe = SURVEY_BYTES_PER_EVAL.get(args.config, 193.0)
    achieved = bpe * evals_per_launch / k1_avg_s / 1e9
    traffic = None
    prof = os.path.join(ROOT, "profiles", f"k1_traffic_{args.config}.json")
    if os.path.exists(prof):
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
            "warmup": args.warmup, "ms_per_step": ms_max / args.steps, "higher_is_better": True, "scaling": "weak",
            "vs_baseline": None, "dtype": "f32", "data": "synthetic",
            "config": {**workload_config(args, dims["n_bool"] + dims["n_real"], dims["n_cons"], world),
                       "kernels": "generic" if args.no_prepare else "specialised for R (fsmt_prepare)",
                       "parallelism": f"restart-sharded x{world}",
                       "l2": "inputs exceed L2 (U counters %.0f MB + structure + state per step)" % (dims["n_cons"] * R / 1e6),
                       "accumulation": "fp64", "build_s": round(build_s, 2)},
            "roofline": {"bound": "alu", "achieved": alu_achieved, "peak": alu_peak, "unit": "TFLOP/s",
                         "frac": alu_achieved / alu_peak, "traffic": traffic, "kernel": "fsmt_k1_jit",
                         "basis": f"SURVEY 8(d) model {fma_pe:.0f} FMA-eq (x2 flop) per (constraint,restart) eval x "
                                  f"{evals_per_launch} evals per launch / live CUDA-event launch time; peak = 148 SMs x "
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
                n_sample = 1500 if args.config in ("cfg4", "cfg3") else min(inst.n_cons, 500)
                f, a, b, n = oracle_sample(inst, n_sample)
                time_oracle(f, a, b)
                reps, tot = 0, 0.0
                while tot < 10.0 and reps < 50:
                    tot += time_oracle(f, a, b)
                    reps += 1
                line["cpu_baseline"] = {"value": n * reps / tot, "unit": "evals/s", "cores": 1, "kind": "oracle",
                                        "sample": f"first {n} constraints of {args.config}, 1 restart, "
                                                  f"objective+gradient x{reps} ({tot:.1f} s)"}
            except Exception as e:  # the baseline must never kill the bench line
                line["cpu_baseline"] = {"value": None, "unit": "evals/s", "cores": 1, "kind": "oracle",
                                        "sample": f"failed: {e}"}
        if not args.no_tts and world == 1 and args.config == "cfg4":
            try:
                line["time_to_sat"] = time_to_sat(P, inst, local)
            except Exception as e:  # never kill the bench line
                line["time_to_sat"] = {"median_s": None, "note": f"failed: {e}"}
        print(json.dumps(line))
    if world > 1:
        dist.destroy_process_group()


if __name__ == "__main__":
    main()
