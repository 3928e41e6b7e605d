#!/bin/bash
# ncu --set full captures of the auxiliary hot-path kernels (one launch each,
# after warm-up): P / P^H (16^4, nv 24), the projection kernels (V^H X s=1,
# s=16 tile, X - VH), the coarse apply at the config-5 size (8 rhs, fp32 C)
# and the PCG64 noise kernel.  Summaries under gpurun_out/$1_*_ncu.txt.
P=${1:-aux}
O=gpurun_out
NCU="ncu --set full --clock-control none --import-source on -c 1"
$NCU -k regex:restrict_mrhs_kernel -s 4 -o $O/${P}_restrict python tools/kernel_rooflines.py > $O/${P}_ncu_restrict.log 2>&1 || true
$NCU -k regex:prolong_kernel -s 4 -o $O/${P}_prolong python tools/kernel_rooflines.py > $O/${P}_ncu_prolong.log 2>&1 || true
$NCU -k regex:vhx_small_kernel -s 4 -o $O/${P}_vhx_s1 python tools/proj_probe.py > $O/${P}_ncu_vhx1.log 2>&1 || true
$NCU -k regex:vhx_tile_kernel -s 4 -o $O/${P}_vhx_tile16 python tools/proj_probe.py > $O/${P}_ncu_vhx16.log 2>&1 || true
$NCU -k regex:proj_sub_kernel -s 4 -o $O/${P}_proj_sub python tools/proj_probe.py > $O/${P}_ncu_psub.log 2>&1 || true
$NCU -k regex:coarse_apply_dir_kernel -s 40 -o $O/${P}_coarse8 python tools/coarse_apply_probe.py > $O/${P}_ncu_coarse.log 2>&1 || true
$NCU -k regex:noise_kernel -s 2 -o $O/${P}_noise python tools/kernel_rooflines.py > $O/${P}_ncu_noise.log 2>&1 || true
for f in $O/${P}_*.ncu-rep; do
  python tools/ncu_summary.py $f > ${f%.ncu-rep}_ncu.txt 2>&1
  rm -f $f
done
ls $O | grep ${P}_
