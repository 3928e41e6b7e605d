#!/bin/bash
# One GPU call: plain bench, launch list of the same probes command, and full
# ncu captures of the even-odd solver kernels (fp32 inner of the mixed solve,
# fp64) and the headline dslash.  Outputs under gpurun_out/ with prefix $1.
P=${1:-prof}
O=gpurun_out
python bench.py --steps 20 --warmup 3 > $O/${P}_bench.json 2> $O/${P}_bench.err || exit 1
python tools/kernel_rooflines.py > $O/${P}_kernel_rooflines.jsonl 2> $O/${P}_kernel_rooflines.err
CMD="python bench.py --skip-eigen --skip-cpu --skip-config5 --skip-sustained --steps 3 --warmup 3"
MGT_SOLVE_STREAMS=1 $CMD > $O/${P}_plain_s1.log 2>&1 || exit 2
MGT_SOLVE_STREAMS=1 ncu --metrics gpu__time_duration.sum --clock-control none --csv \
   --log-file $O/${P}_launches.csv $CMD > $O/${P}_ncu_launch.log 2>&1
SB="python tools/solver_bench.py --dims 32x32x32x32 --groups 4 --nprobe 8 --mixed 1"
$SB > $O/${P}_solver_plain.log 2>&1 || exit 3
ncu --set full --clock-control none --import-source on -k regex:bi_k1_eo -s 20 -c 1 \
   -o $O/${P}_k1eo_f32 $SB > $O/${P}_ncu_k1eo_f32.log 2>&1
ncu --set full --clock-control none --import-source on -k regex:bi_k4v -s 20 -c 1 \
   -o $O/${P}_k4_f32 $SB > $O/${P}_ncu_k4_f32.log 2>&1
ncu --set full --clock-control none --import-source on -k regex:bi_k1_eo -s 20 -c 1 \
   -o $O/${P}_k1eo_f64 python tools/solver_bench.py --dims 32x32x32x32 --groups 4 --nprobe 8 --mixed 0 \
   > $O/${P}_ncu_k1eo_f64.log 2>&1
ncu --set full --clock-control none --import-source on -k regex:wilson_apply_kernel -s 3 -c 1 \
   -o $O/${P}_dslash python bench.py --steps 5 --warmup 3 --skip-cpu --skip-probes --skip-sustained > $O/${P}_ncu_dslash.log 2>&1

# keep the call's output under gpurun's 64 MiB merge limit: text summaries
# of every capture, the dslash report itself, the launch list gzipped
for f in $O/${P}_*.ncu-rep; do
  python tools/ncu_summary.py $f > ${f%.ncu-rep}_ncu.txt 2>&1
  ncu -i $f --page details > ${f%.ncu-rep}_details.txt 2>&1
done
python tools/launch_summary.py $O/${P}_launches.csv > $O/${P}_launch_summary.txt 2>&1
gzip -f $O/${P}_launches.csv
mkdir -p /tmp/ncu_keep && for f in $O/${P}_*.ncu-rep; do case $f in *dslash*) ;; *) mv $f /tmp/ncu_keep/ ;; esac; done
du -sh $O
