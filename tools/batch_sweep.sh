#!/bin/bash
# probes/s of BASELINE configs[0] and [2] vs rhs per solve call (batched
# groups of 4) and concurrent solve streams
for cfg in "4 8" "4 4" "8 4" "16 1" "16 2" "32 1" "8 2" "16 4"; do
  set -- $cfg
  MGT_SOLVE_BATCH=$1 MGT_SOLVE_STREAMS=$2 python bench.py --skip-eigen --skip-cpu --steps 3 --warmup 3 2>/dev/null | python -c "
import sys, json
d = json.loads(sys.stdin.readline())
print('batch', $1, 'streams', $2, 'config1', round(d['probes_per_sec']['value']), 'config3', round(d['deflated_probes_per_sec']['value']))"
done
