#!/bin/bash
# One GPU call: plain bench, launch list of the same probes command, and full
# ncu captures of the even-odd solver kernel and the headline dslash.
# Outputs under gpurun_out/ with prefix $1 (e.g. r01c).
P=${1:-prof}
O=gpurun_out
python bench.py --steps 20 --warmup 3 > $O/${P}_bench.json 2> $O/${P}_bench.err || exit 1
CMD="python bench.py --skip-eigen --skip-cpu --steps 3 --warmup 3"
MGT_SOLVE_STREAMS=1 $CMD > $O/${P}_plain_s1.log 2>&1 || exit 2
MGT_SOLVE_STREAMS=1 ncu --metrics gpu__time_duration.sum --clock-control none --csv \
   --log-file $O/${P}_launches.csv $CMD > $O/${P}_ncu_launch.log 2>&1
python tools/solver_bench.py --dims 32x32x32x32 --groups 4 --nprobe 8 > $O/${P}_solver_plain.log 2>&1 || exit 3
ncu --set full --clock-control none --import-source on -k regex:bi_k1_eo -s 20 -c 1 \
   -o $O/${P}_k1eo python tools/solver_bench.py --dims 32x32x32x32 --groups 4 --nprobe 8 > $O/${P}_ncu_k1eo.log 2>&1
ncu --set full --clock-control none --import-source on -k regex:bi_eo_first -s 20 -c 1 \
   -o $O/${P}_first python tools/solver_bench.py --dims 32x32x32x32 --groups 4 --nprobe 8 > $O/${P}_ncu_first.log 2>&1
ncu --set full --clock-control none --import-source on -k regex:wilson_apply_kernel -s 3 -c 1 \
   -o $O/${P}_dslash python bench.py --steps 5 --warmup 3 --skip-cpu --skip-probes > $O/${P}_ncu_dslash.log 2>&1
echo done
