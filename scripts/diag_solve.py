#!/usr/bin/env python
"""Diagnose a solve on a placement/scheduling config: per-stage unsat statistics over the
restarts, and for the best model the kind of violated constraints (placement: same-bin overlaps).

  python scripts/diag_solve.py --config cfg4 --kmax 50 --eta 0.2 --eta-mode 1 --steps 40
"""
from __future__ import annotations

import argparse
import json
import os
import sys
import time

import numpy as np

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)


def main():
    p = argparse.ArgumentParser()
    p.add_argument("--config", default="cfg4")
    p.add_argument("--restarts", type=int, default=1024)
    p.add_argument("--steps", type=int, default=40)
    p.add_argument("--stages", type=int, default=20)
    p.add_argument("--kmin", type=float, default=1.0)
    p.add_argument("--kmax", type=float, default=50.0)
    p.add_argument("--eta", type=float, default=0.2)
    p.add_argument("--eta-mode", type=int, default=1)
    p.add_argument("--erwa", type=int, default=1)
    p.add_argument("--seed", type=int, default=0)
    a = p.parse_args()
    import paper_2603_22877_b200 as P
    import fsmt_gen
    inst = fsmt_gen.config(a.config)
    s = P.Solver(0)
    s.load_formula(inst.text)
    s.build_xbdd()
    kap = [a.kmin * (a.kmax / a.kmin) ** (i / max(a.stages - 1, 1)) for i in range(a.stages)]
    s.set_params(kappas=kap, eta=a.eta, eta_mode=a.eta_mode, erwa_mode=a.erwa)
    s.begin(a.restarts, a.seed)
    best = None
    t0 = time.perf_counter()
    for t, k in enumerate(kap, start=1):
        u, m = s.run_stage(t, k, a.steps)
        A, B = s.get_state()
        sat_a = float(np.mean(np.abs(A) > 0.99))
        print(json.dumps({"stage": t, "kappa": round(k, 3), "unsat_min": int(u.min()), "unsat_med": float(np.median(u)),
                          "a_saturated": round(sat_a, 3), "b_std": float(B.std()), "t": round(time.perf_counter() - t0, 2)}),
              flush=True)
        r = int(np.argmin(u))
        if best is None or u[r] < best[0]:
            best = (int(u[r]), t, r, *s.get_model(r))
        if u[r] == 0:
            break
    n, per = s.verify(best[3], best[4], per_con=True)
    viol = np.nonzero(per)[0]
    out = {"best_unsat": best[0], "stage": best[1], "restart": best[2], "host_unsat": n}
    if a.config.startswith("cfg4"):
        K = inst.meta["bits_per_module"]
        nm, nl = inst.meta["n_m"], inst.meta["n_l"]
        M = inst.meta["modules"]
        x = best[3]
        bits = (x.reshape(M, K) == -1).astype(int)
        bins = (bits * (1 << np.arange(K))).sum(1)
        occ = np.bincount(bins, minlength=nm * nl)
        area = np.zeros(nm * nl)
        for j in range(M):
            w, h = inst.meta["sizes"][j]
            area[bins[j]] += float(w) * float(h)
        out.update({"bin_occupancy_max": int(occ.max()), "bin_area_max": float(area.max()),
                    "bins_over_area_1": int((area > 1.0).sum()),
                    "violated_nonoverlap": int((viol < M * (M - 1) // 2).sum()),
                    "violated_bounds": int((viol >= M * (M - 1) // 2).sum())})
    cons_lines = [ln for ln in inst.text.splitlines() if ln[:2] in ("c ", "e ")]
    out["violated_lines"] = [cons_lines[i][:120] for i in viol[:12]]
    print(json.dumps(out))


if __name__ == "__main__":
    main()
