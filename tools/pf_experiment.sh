#!/bin/bash
for pf in 0 1 2; do
  echo "prefetch=$pf"
  MGT_PREFETCH=$pf python tools/sweep.py --dims 16x16x16x16,32x32x32x32,48x48x48x96 --prec 64 --recon 12 --nrhs 1,4 2>&1 | python -c "
import sys,json
for l in sys.stdin:
  d=json.loads(l); print('  ', d['dims'], d['n_rhs'], round(d['ms'],4), 'ms', round(d['GBps']), 'GB/s')"
  MGT_PREFETCH=$pf python tools/solver_bench.py --groups 4 2>&1 | tail -2
done
