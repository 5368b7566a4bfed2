#!/bin/bash
# Time-to-SAT on the paper's random hybrid family (rand<n>): one JSON line per (n, recipe)
# in gpurun_out/tts_random_family.jsonl (4 seeds, 20 s per solve).
mkdir -p gpurun_out
out=gpurun_out/tts_random_family.jsonl
[ -n "$APPEND" ] || : > $out
run() {
  timeout 400 python scripts/time_to_sat.py --seeds 0 1 2 3 --time-limit 20 "$@" > /tmp/t.jsonl 2>&1
  echo "{\"args\": \"$*\", \"seeds\": [$(grep '"seed"' /tmp/t.jsonl | paste -sd, -)], \"result\": $(tail -1 /tmp/t.jsonl)}" >> $out
}
for n in ${NS:-100 300 500 700 1000}; do
  run --config rand$n --restarts 1024
done
