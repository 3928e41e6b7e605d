#!/bin/bash
# probes/s of BASELINE configs[0] and [2] vs the number of concurrent solve streams
for n in 1 2 3 4 6 8 12; do
  MGT_SOLVE_STREAMS=$n python bench.py --skip-eigen --skip-cpu --steps 3 --warmup 3 2>/dev/null | python -c "
import sys, json
d = json.loads(sys.stdin.readline())
print('streams', $n, 'config1', round(d['probes_per_sec']['value']), 'config3', round(d['deflated_probes_per_sec']['value']))"
done
