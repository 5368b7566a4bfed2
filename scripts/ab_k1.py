#!/usr/bin/env python
"""A/B of the JIT sweep's build-time knobs (env vars read at fsmt_build_xbdd): runs bench.py once
per variant in a fresh process and prints K1 ms/launch and the bench value.

  python scripts/ab_k1.py "" "FSMT_JIT_SVAL=1" "FSMT_JIT_SVAL=1 FSMT_TILE_VMAX=64"
"""
import json
import os
import subprocess
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def main():
    variants = sys.argv[1:] or [""]
    extra = os.environ.get("AB_ARGS", "--steps 5 --warmup 3 --no-e2e --no-cpu-baseline --no-tts").split()
    for v in variants:
        env = dict(os.environ)
        for kv in v.split():
            k, val = kv.split("=", 1)
            env[k] = val
        p = subprocess.run([sys.executable, os.path.join(ROOT, "bench.py")] + extra, env=env, capture_output=True,
                           text=True, timeout=900)
        line = next((l for l in p.stdout.splitlines() if l.startswith("{")), None)
        if line is None:
            print(json.dumps({"variant": v, "error": (p.stderr or p.stdout)[-400:]}), flush=True)
            continue
        d = json.loads(line)
        print(json.dumps({"variant": v or "default", "k1_ms": round(d["roofline"]["k1_ms_per_launch"], 3),
                          "value": d["value"], "frac": round(d["roofline"]["frac"], 4),
                          "sm_mhz": d["clocks"].get("sm_mhz"), "jit": d["config"].get("jit")}), flush=True)


if __name__ == "__main__":
    main()
