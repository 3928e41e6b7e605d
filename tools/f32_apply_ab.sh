#!/bin/bash
# fp32 dslash: resident blocks per SM of wilson_apply_kernel<float> (A/B)
for v in 4 3 5 6; do
  rm -rf build
  MGT_NVCC_EXTRA="-DMGT_F32_APPLY_MINB=$v" python -c "from paper_1909_12234_b200 import _build; _build.build()" > /dev/null 2>&1 || { echo "build $v failed"; continue; }
  for rep in 1 2; do
    python tools/sweep.py --dims 24x24x24x24,32x32x32x32,48x48x48x96 --prec 32 --recon 12 --nrhs 1 | python -c "
import sys,json
for l in sys.stdin:
  d=json.loads(l); print('minb=$v', d['dims'], round(d['ms'],4), 'ms', round(d['GBps']), 'GB/s')"
  done
done
