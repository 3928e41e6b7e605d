#!/bin/bash
# A/B of compile-time variants: each argument is an MGT_NVCC_EXTRA string
# ("" = default).  Per variant: rebuild, then the headline dslash sweep and
# the mixed / fp64 even-odd solver bench, twice.
for v in "$@"; do
  rm -rf build
  MGT_NVCC_EXTRA="$v" python -c "from paper_1909_12234_b200 import _build; _build.build()" > /dev/null 2>&1 || { echo "build '$v' failed"; continue; }
  for rep in 1 2; do
    python tools/sweep.py --dims 32x32x32x32,48x48x48x96 --prec 64,32 --recon 12 --nrhs 1 | python -c "
import sys,json
for l in sys.stdin:
  d=json.loads(l); print('[$v] dslash', d['dims'], d['prec'], round(d['ms'],4), 'ms', round(d['GBps']), 'GB/s')"
    python tools/solver_bench.py --dims 16x16x16x16,32x32x32x32 --groups 16 --nprobe 32 --mixed 1,0 | python -c "
import sys,json
for l in sys.stdin:
  d=json.loads(l); print('[$v] solver', d['dims'], 'mixed' if d['mixed'] else 'fp64', round(d['probes_per_s'],1), 'probes/s', round(d['us_per_iter_per_rhs'],2), 'us/iter/rhs')"
  done
done
