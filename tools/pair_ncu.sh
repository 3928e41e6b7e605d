#!/bin/bash
# ncu --set full of the fp32 stencil kernels (one-site vs pair variants) inside
# a 4-rhs mixed solve; only the raw-page CSV travels back.
D=${1:-32x32x32x32}
for v in 0 1; do
  MGT_F32_STENCIL_PAIRS=$v ncu --set full --clock-control none -k regex:"bi_k1_eo|bi_eo_first" -s 12 -c 2 \
    -o /tmp/pairs${v} -f python tools/solver_bench.py --dims $D --groups 4 --nprobe 4 --mixed 1 > gpurun_out/pairs${v}_ncu.log 2>&1
  ncu -i /tmp/pairs${v}.ncu-rep --page raw --csv > gpurun_out/pairs${v}_raw.csv
  ncu -i /tmp/pairs${v}.ncu-rep --page details > gpurun_out/pairs${v}_details.txt
done
