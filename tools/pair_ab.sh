#!/bin/bash
# A/B of the two-sites-per-thread fp32 stencils (eo_pair.cuh) against the
# one-site kernels: MGT_F32_STENCIL_PAIRS=0/1 on the same box, twice.
DIMS=${1:-8x8x8x8,16x16x16x16,24x24x24x24,32x32x32x32,32x32x32x64}
for rep in 1 2; do
  for v in 0 1; do
    MGT_F32_STENCIL_PAIRS=$v python tools/solver_bench.py --dims $DIMS --groups 16 --nprobe 32 --mixed 1 | python -c "
import sys,json
for l in sys.stdin:
  d=json.loads(l); print('[pairs=$v] solver', d['dims'], round(d['probes_per_s'],1), 'probes/s', round(d['us_per_iter_per_rhs'],2), 'us/iter/rhs', 'iters', round(d['mean_iters'],2), 'relres', '%.2e' % d['max_relres'])"
  done
done
