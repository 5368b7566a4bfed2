#!/bin/bash
# Time-to-SAT exploration on the paper's routed placement instance (place9856, 9,856 vars / 415,424
# constraints): R33 projection of the routing adjacency atoms, restart counts, steps, eta.
mkdir -p gpurun_out
out=gpurun_out/tts_routed_sweep.jsonl
: > $out
for args in "--restarts 256 --proj-iters 10" "--restarts 1024 --proj-iters 10" "--restarts 256 --proj-iters 20 --steps 4 --eta 0.2" \
            "--restarts 256 --proj-iters 10 --schedule geo1-300-hold30" "--restarts 256 --proj-iters 10 --rounding 1" \
            "--restarts 256 --proj-iters 10 --erwa 0" "--restarts 256 --proj-iters 10 --eta 0.8"; do
  timeout 300 python scripts/time_to_sat.py --config place9856 --seeds 0 1 --time-limit 120 $args > /tmp/t.jsonl 2>&1
  echo "{\"args\": \"$args\", \"result\": $(tail -1 /tmp/t.jsonl)}" >> $out
  grep seed /tmp/t.jsonl | cut -c1-200
done
