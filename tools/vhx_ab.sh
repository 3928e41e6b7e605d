#!/bin/bash
# A/B of the V^H X few-column kernel: A = in-tree build (unrolled e-loop),
# B = -DMGT_VHX_NO_UNROLL (one element per lane per trip).  Deflation GPU
# tests on A first.
set -e
python -m pytest tests/test_deflation_gpu.py -q -x 2>&1 | tail -2
python tools/proj_probe.py | grep '"vhx"' | sed 's/^/A /'
python tools/proj_probe.py | grep '"vhx"' | sed 's/^/A /'
rm -rf build
MGT_NVCC_EXTRA="-DMGT_VHX_NO_UNROLL" python -c "from paper_1909_12234_b200 import _build; _build.build()" > /dev/null 2>&1
python tools/proj_probe.py | grep '"vhx"' | sed 's/^/B /'
python tools/proj_probe.py | grep '"vhx"' | sed 's/^/B /'
