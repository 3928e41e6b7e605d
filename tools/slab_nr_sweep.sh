#!/bin/bash
for mb in 2 4 8 16 32; do
  echo "slab_mb=$mb"
  MGT_SLAB_MB=$mb python tools/sweep.py --dims 32x32x32x32,48x48x48x96 --prec 64 --recon 12 --nrhs 1,2,4 2>&1 | python -c "
import sys,json
for l in sys.stdin:
  try: d=json.loads(l)
  except Exception: print(l.strip()); continue
  print('  ', d['dims'], d['n_rhs'], round(d['ms'],4), 'ms', round(d['GBps']), 'GB/s')"
done
