#!/bin/bash
# even-odd solver iteration time vs the L2 slab budget of the schedule
for mb in 4 8 16 32 64; do
  echo "slab_mb=$mb"
  MGT_SLAB_MB=$mb python tools/solver_bench.py --dims 16x16x16x16,32x32x32x32 --groups 4 --nprobe 8 2>&1 | python -c "
import sys, json
for l in sys.stdin:
    d = json.loads(l); print('  ', d['dims'], round(d['us_per_iter_per_rhs'], 1), 'us/iter/rhs', round(d['probes_per_s'], 1), 'probes/s')"
done
