#!/bin/bash
# A/B of a compile-time variant: default build vs MGT_NVCC_EXTRA="$1" (the box
# rebuilds the library with nvcc): dslash sweep + even-odd solver bench on
# each, operator/solver GPU tests on the variant.
set -e
run() {
  python tools/sweep.py --dims 32x32x32x32,48x48x48x96 --prec 64,32 --recon 12 --nrhs 1 | python -c "
import sys,json
for l in sys.stdin:
  d=json.loads(l); print('$1', d['dims'], d['prec'], round(d['ms'],4), round(d['GBps']))"
  python tools/solver_bench.py --dims 16x16x16x16,32x32x32x32 --groups 4 --nprobe 8 | python -c "
import sys,json
for l in sys.stdin:
  d=json.loads(l); print('$1 solver', d['dims'], round(d['us_per_iter_per_rhs'],1), 'us/iter/rhs')"
}
run A
run A
rm -rf build
MGT_NVCC_EXTRA="$1" python -c "from paper_1909_12234_b200 import _build; _build.build()" > /dev/null 2>&1
run B
run B
python -m pytest tests/test_operator_gpu.py tests/test_solver_gpu.py tests/test_slab_gpu.py -q -x 2>&1 | tail -2
