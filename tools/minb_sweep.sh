#!/bin/bash
# Blocks-per-SM bound of the fp32 even-odd solver kernels: rebuild with
# -DMGT_F32_MINB=$v for each value and time the mixed solver.
for v in "$@"; do
  rm -rf build
  MGT_NVCC_EXTRA="-DMGT_F32_MINB=$v" python -c "from paper_1909_12234_b200 import _build; _build.build()" > /dev/null 2>&1 || { echo "build $v failed"; continue; }
  for rep in 1 2; do
    python tools/solver_bench.py --dims 16x16x16x16,32x32x32x32 --groups 16 --nprobe 32 --mixed 1 | python -c "
import sys,json
for l in sys.stdin:
  d=json.loads(l); print('minb=$v', d['dims'], round(d['probes_per_s'],1), 'probes/s', round(d['us_per_iter_per_rhs'],2), 'us/iter/rhs', d['mean_iters'])"
  done
done
