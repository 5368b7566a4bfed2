#!/usr/bin/env python
"""Time one K1 sweep of a config at R restarts (CUDA events inside the library, 20 launches after warm-up):
the per-class A/B driver for small formulas (python scripts/one_sweep.py rand1000 10000)."""
import json
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))


def main():
    import fsmt_gen
    import paper_2603_22877_b200 as P
    from fsmt_gen.points import random_points
    name, R = sys.argv[1], int(sys.argv[2])
    s = P.Solver(0)
    s.load_formula(fsmt_gen.config(name).text)
    s.build_xbdd()
    if len(sys.argv) > 3 and sys.argv[3] == "prepare":
        s.prepare(R)                       # the R-specialised module with its register caps
    d = s.get_dims()
    a, b = random_points(d["n_bool"], d["n_real"], R, seed=5)
    s.begin(R, 1)
    s.set_state(a, b)
    s.sweep(0.5, 1)
    ms = s.time_sweep(0.5, 1, 20)
    print(json.dumps({"config": name, "R": R, "sweep_ms": ms, "evals_per_s": d["n_cons"] * R / (ms / 1e3), "jit": s.jit_info()["status"],
                      "env": {k: v for k, v in os.environ.items() if k.startswith("FSMT_")}}), flush=True)


if __name__ == "__main__":
    main()
