#!/bin/bash
# dslash tuning grid (run under gpurun): variant x slab budget x recon
for v in 0 1; do for mb in 4 8 16 24 48; do
  MGT_DSLASH_VARIANT=$v MGT_SLAB_MB=$mb python tools/sweep.py --dims 32x32x32x32,48x48x48x96 --prec 64 --recon 12,18 --steps 20 2>&1 | sed "s/^/v=$v mb=$mb /" | cut -c1-200
done; done
