#!/bin/bash
# ncu --set full of the pipelined DMMA projection kernels (V^H X and X - V H,
# k = 64, 16^4) at s = 8 and s = 16; text summaries under gpurun_out/$1_*.
P=${1:-projpipe}
O=gpurun_out
NCU="ncu --set full --clock-control none -c 1"
for S in 8 16; do
  S=$S $NCU -k regex:vhx_bulk_kernel -o /tmp/${P}_vhx_s$S -f python tools/vhx_once.py > $O/${P}_vhx_s$S.log 2>&1
  S=$S $NCU -k regex:proj_sub_pipe_kernel -o /tmp/${P}_sub_s$S -f python tools/vhx_once.py > $O/${P}_sub_s$S.log 2>&1
  for kname in vhx sub; do
    python tools/ncu_summary.py /tmp/${P}_${kname}_s$S.ncu-rep > $O/${P}_${kname}_s${S}_ncu.txt 2>&1
  done
done
ls $O | grep $P
