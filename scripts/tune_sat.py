#!/usr/bin/env python
"""Sweep solver hyper-parameters the paper leaves open (R12 schedule, R13 eta, steps, ERWA
reading, rounding) for time-to-SAT on one config.  Prints one JSON line per setting.

  python scripts/tune_sat.py --config cfg3s --restarts 1024 --seeds 0 1 2
"""
from __future__ import annotations

import argparse
import itertools
import json
import os
import sys
import time

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)


def schedules(kmax_list, n_stages, holds=(1,)):
    out = {"default": [round(0.1 * i, 4) for i in range(1, 21)]}
    for kmax in kmax_list:
        g = [kmax ** (i / (n_stages - 1)) for i in range(n_stages)]          # geometric 1 .. kmax
        out[f"geo1-{kmax}"] = g
        out[f"geo0.1-{kmax}"] = [0.1 * (kmax / 0.1) ** (i / (n_stages - 1)) for i in range(n_stages)]
        for m in holds:                                                      # then hold kmax m times as long
            out[f"geo1-{kmax}-hold" + ("" if m == 1 else str(m))] = g + [kmax] * (m * n_stages)
    return out


def main():
    p = argparse.ArgumentParser()
    p.add_argument("--config", default="cfg3s")
    p.add_argument("--restarts", type=int, default=1024)
    p.add_argument("--seeds", type=int, nargs="+", default=[0, 1, 2])
    p.add_argument("--steps", type=int, nargs="+", default=[40])
    p.add_argument("--etas", type=float, nargs="+", default=[0.01, 0.05])
    p.add_argument("--kmax", type=float, nargs="+", default=[20.0, 100.0])
    p.add_argument("--stages", type=int, default=20)
    p.add_argument("--holds", type=int, nargs="+", default=[1])
    p.add_argument("--erwa", type=int, nargs="+", default=[0, 1])
    p.add_argument("--rounding", type=int, nargs="+", default=[0])
    p.add_argument("--eta-modes", type=int, nargs="+", default=[0])
    p.add_argument("--proj-iters", type=int, nargs="+", default=[0])
    p.add_argument("--n-roundings", type=int, nargs="+", default=[1])
    p.add_argument("--time-limit", type=float, default=120.0)
    p.add_argument("--only", default="")
    a = p.parse_args()
    import paper_2603_22877_b200 as P
    import fsmt_gen
    from paper_2603_22877_b200 import native as N
    inst = fsmt_gen.config(a.config)
    s = P.Solver(0)
    s.load_formula(inst.text)
    s.build_xbdd()
    sch = schedules(a.kmax, a.stages, a.holds)
    if a.only:
        sch = {k: v for k, v in sch.items() if k in a.only.split(",")}
    for (name, ks), steps, eta, erwa, rnd, em, pi, nr in itertools.product(sch.items(), a.steps, a.etas, a.erwa,
                                                                            a.rounding, a.eta_modes, a.proj_iters,
                                                                            a.n_roundings):
        if nr > 1 and rnd == 0:
            continue
        s.set_params(kappas=ks, eta=eta, erwa_mode=erwa, rounding=rnd, time_limit_s=a.time_limit, eta_mode=em,
                     proj_iters=pi, n_roundings=nr)
        solved, times, best = 0, [], []
        t0 = time.perf_counter()
        for seed in a.seeds:
            res = s.solve(a.restarts, steps, seed)
            ok = res.verdict == N.SAT and s.verify(res.x, res.y) == 0
            solved += ok
            times.append(res.stats["solve_ms"] / 1e3)
            best.append(res.stats["best_unsat"])
        print(json.dumps({"config": a.config, "schedule": name, "steps": steps, "eta": eta, "erwa": erwa,
                          "rounding": rnd, "eta_mode": em, "proj_iters": pi, "n_roundings": nr, "solved": solved, "runs": len(a.seeds), "best_unsat": best,
                          "solve_s": [round(x, 3) for x in times], "wall_s": round(time.perf_counter() - t0, 2)}),
              flush=True)


if __name__ == "__main__":
    main()
