#!/bin/bash
# SURVEY §8(d) config 5 on one GPU: the bench step (cfg4, 8 PGD steps + stage end) at R = 1k..64k
# restarts, kernels prepared for each R.  One JSON line per R in gpurun_out/restart_sweep.jsonl.
mkdir -p gpurun_out
for R in 1024 2048 4096 8192 16384 32768 65536; do
  python bench.py --restarts $R --steps 3 --warmup 3 --no-e2e --no-tts --no-cpu-baseline > gpurun_out/rs_$R.log 2>&1
  tail -1 gpurun_out/rs_$R.log >> gpurun_out/restart_sweep.jsonl
done
