#!/bin/bash
# L2 slab budget (MGT_SLAB_MB) sweep of the plain fp64/fp32 apply, single rhs
for mb in ${MBS:-16 24 32 40 48 64 32}; do
  MGT_SLAB_MB=$mb python tools/sweep.py --dims ${DIMS:-32x32x32x32,48x48x48x96} --prec ${PREC:-64} --recon 12 --nrhs 1 --steps 30 | python -c "
import sys,json
for l in sys.stdin:
  d=json.loads(l); print('slab_mb=$mb', d['dims'], 'fp%d'%d['prec'], round(d['ms'],4), 'ms', round(d['GBps']), 'GB/s')"
done
