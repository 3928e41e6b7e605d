#!/bin/bash
# single-rhs dslash vs the L2 slab budget (MGT_SLAB_MB) at 48^3x96 / 32^4
for mb in 24 32 48 64 96 128 256; do
  MGT_SLAB_MB=$mb python tools/sweep.py --dims 32x32x32x32,48x48x48x96 --prec 64,32 --recon 12 --nrhs 1 2>&1 | python -c "
import sys,json
for l in sys.stdin:
  try: d=json.loads(l)
  except Exception: print(l.strip()); continue
  print('slab_mb=$mb', d['dims'], d['prec'], round(d['ms'],4), 'ms', round(d['GBps']), 'GB/s')"
done
