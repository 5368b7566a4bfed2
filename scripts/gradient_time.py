#!/usr/bin/env python
"""B200 analog of the paper's gradient-time study (Fig.3b; Supp. Note 12):
for the random hybrid family at n = 100..1000, the objective + gradient at 10,000 points
in 100 groups of 100 points, group g at 1/sigma = g/100, timed with CUDA events around the
sweep launches (slot tables, K1, chain); also the 10,000 points as ONE sweep (R = 10,000, one kappa),
and the A/B of the CARD form (FSMT_JIT_COUNT: 1 = count-distribution class, 0 = xBDD class when it fits
the register budget, else the generic interpreter).  One JSON line per (n, variant).

  python scripts/gradient_time.py [--n 100 200 ...] [--oracle]
"""
from __future__ import annotations

import argparse
import json
import os
import sys
import time

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

# the paper's per-instance averages of the gradient time (Supp. Table "gradient-time"; ms,
# means over the 9-10 instances of each n): GPU = one L40S, CPU = 64 EPYC threads -- context only
# (another machine, another implementation; the table does not say per how many points)
PAPER_L40S_MS = {100: 12.68, 200: 13.64, 300: 12.77, 400: 12.80, 500: 12.60, 600: 12.79, 700: 12.76, 800: 12.84,
                 900: 12.87, 1000: 12.65}
PAPER_CPU64_MS = {100: 5.00, 200: 21.78, 300: 34.15, 400: 43.14, 500: 48.40, 600: 56.27, 700: 62.40, 800: 69.08,
                  900: 77.37, 1000: 84.36}


def build(P, text, env):
    old = {k: os.environ.get(k) for k in env}
    os.environ.update(env)
    try:
        s = P.Solver(0)
        s.load_formula(text)
        s.build_xbdd()
    finally:
        for k, v in old.items():
            if v is None:
                os.environ.pop(k, None)
            else:
                os.environ[k] = v
    return s


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--n", type=int, nargs="+", default=list(range(100, 1001, 100)))
    ap.add_argument("--oracle", action="store_true", help="also time the fp64 CPU oracle at one point per n")
    args = ap.parse_args()
    import numpy as np
    import torch
    import fsmt_gen
    import paper_2603_22877_b200 as P
    from fsmt_gen.points import random_points
    for n in args.n:
        inst = fsmt_gen.config(f"rand{n}")
        for variant, env in (("default", {}), ("count", {"FSMT_JIT_COUNT": "1"}), ("no-count", {"FSMT_JIT_COUNT": "0"})):
            s = build(P, inst.text, env)
            info = s.jit_info()
            d = s.get_dims()
            G, R = 100, 100
            s.prepare(R)
            s.begin(R, 1)
            pts = [random_points(d["n_bool"], d["n_real"], R, seed=1000 + g) for g in range(G)]
            for g in range(3):                                    # warm-up
                s.set_state(*pts[g])
                s.sweep(g / 100.0, 1)
            s.set_timing(True)
            s.get_timing(reset=True)
            for g in range(G):                                     # 100 groups x 100 points, 1/sigma = g/100
                s.set_state(*pts[g])
                s.sweep(g / 100.0, 1)
            ms, cnt = s.get_timing(reset=True)["k1_sweep"]
            s.set_timing(False)
            # the same 10,000 points as one sweep (one kappa), with the module prepared for it
            RB = G * R
            s.prepare(RB)
            a = np.concatenate([p[0] for p in pts], axis=1)
            b = np.concatenate([p[1] for p in pts], axis=1)
            s.begin(RB, 1)
            s.set_state(a, b)
            s.sweep(0.5, 1)
            one_ms = s.time_sweep(0.5, 1, 20)
            line = {"n": n, "variant": variant, "constraints": d["n_cons"], "jit": info["status"],
                    "jit_classes": info["jit_classes"], "jit_cons": info["jit_cons"],
                    "groups_ms_total": ms, "groups": cnt, "ms_per_group_of_100": ms / max(cnt, 1),
                    "us_per_point": 1e3 * ms / (G * R),
                    "batched_10000_ms": one_ms, "batched_us_per_point": 1e3 * one_ms / RB,
                    "batched_evals_per_s": d["n_cons"] * RB / (one_ms / 1e3),
                    "paper_l40s_ms_context": PAPER_L40S_MS.get(n), "paper_cpu64_ms_context": PAPER_CPU64_MS.get(n)}
            if args.oracle and variant == "default":
                from oracle import hsmt, objective
                f = hsmt.parse(inst.text)
                t0 = time.perf_counter()
                objective.objective_and_gradient_grouped(f, a[:, 0].astype(np.float64), b[:, 0].astype(np.float64), 0.5)
                line["oracle_cpu_ms_per_point_1proc"] = 1e3 * (time.perf_counter() - t0)
            print(json.dumps(line), flush=True)
            del s
            torch.cuda.synchronize()


if __name__ == "__main__":
    main()
