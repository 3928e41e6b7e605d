#!/bin/bash
# A/B of a compile-time dslash variant: default build vs MGT_NVCC_EXTRA="$1"
# (the box rebuilds the library with nvcc), dslash sweep on each.
set -e
run() {
  python tools/sweep.py --dims 32x32x32x32,48x48x48x96 --prec 64,32 --recon 12 --nrhs 1 | python -c "
import sys,json
for l in sys.stdin:
  d=json.loads(l); print('$1', d['dims'], d['prec'], round(d['ms'],4), round(d['GBps']))"
}
run A
run A
rm -rf build
MGT_NVCC_EXTRA="$1" python -c "from paper_1909_12234_b200 import _build; _build.build()" > /dev/null 2>&1
run B
run B
