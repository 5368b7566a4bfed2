#!/bin/bash
# A/B of the K5 (exact check) emission knobs on the bench workload: stage-end ms, K1 ms, bench value.
#   bash scripts/k5_ab.sh "" "FSMT_JIT_K5PF=0" ...
for v in "$@"; do
  env $v python bench.py --steps 5 --warmup 3 --no-e2e --no-cpu-baseline --no-tts 2>/dev/null | python -c "
import json,sys; d=json.loads(sys.stdin.read()); print('$v', d['kernel_ms']['k45_stage_end']['total_ms']/d['kernel_ms']['k45_stage_end']['groups'], d['roofline']['k1_ms_per_launch'], d['value']/1e9)"
done
