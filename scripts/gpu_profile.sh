#!/bin/bash
# One GPU session: launch list + full ncu capture of the top kernel (K1) on the bench workload.
# usage (under gpurun): bash scripts/gpu_profile.sh <tag> [bench args...]
tag=$1; shift
mkdir -p gpurun_out
ncu --metrics gpu__time_duration.sum --clock-control none -c 400 --csv --log-file gpurun_out/launches_${tag}.csv \
    python bench.py --steps 2 --warmup 1 --no-e2e --no-tts --no-cpu-baseline "$@" > gpurun_out/ncu_launch_${tag}.log 2>&1
ncu --set full --clock-control none --import-source on -k regex:'^fsmt_k1_(jit|c0)$' -s 2 -c 1 -o gpurun_out/k1_${tag} \
    python bench.py --steps 1 --warmup 1 --no-e2e --no-tts --no-cpu-baseline "$@" > gpurun_out/ncu_full_${tag}.log 2>&1
ls -la gpurun_out/
