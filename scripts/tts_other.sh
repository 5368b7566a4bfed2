#!/bin/bash
# Time-to-SAT recipes on cfg2 (random hybrid) and cfg3 (scheduling): one JSON line per recipe in
# gpurun_out/tts_other.jsonl (4 seeds each, 20 s limit per solve).
mkdir -p gpurun_out
out=gpurun_out/tts_other.jsonl
: > $out
run() {
  timeout 400 python scripts/time_to_sat.py --seeds 0 1 2 3 --time-limit 20 "$@" > /tmp/t.jsonl 2>&1
  echo "{\"args\": \"$*\", \"seeds\": [$(grep '"seed"' /tmp/t.jsonl | paste -sd, -)], \"result\": $(tail -1 /tmp/t.jsonl)}" >> $out
}
run --config cfg2 --restarts 1024
run --config cfg2 --restarts 1024 --rounding 1 --n-roundings 8
run --config cfg2 --restarts 1024 --eta 0.1 --schedule geo1-100-hold10
run --config cfg3 --restarts 1024
run --config cfg3 --restarts 1024 --proj-iters 10
run --config cfg3 --restarts 256 --proj-iters 10 --schedule geo1-300-hold30
