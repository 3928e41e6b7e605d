#!/bin/bash
# A/B of the V^H X few-column kernel: A = in-tree build (one-wave grid),
# B = -DMGT_VHX_OLD_GRID (6 blocks per SM + 1).  Deflation GPU
# tests on A first.
set -e
python -m pytest tests/test_deflation_gpu.py -q -x 2>&1 | tail -2
python tools/proj_probe.py | grep -E '"(vhx|sub_vh)"' | sed 's/^/A /'
python tools/proj_probe.py | grep -E '"(vhx|sub_vh)"' | sed 's/^/A /'
rm -rf build
MGT_NVCC_EXTRA="-DMGT_VHX_OLD_GRID" python -c "from paper_1909_12234_b200 import _build; _build.build()" > /dev/null 2>&1
python tools/proj_probe.py | grep -E '"(vhx|sub_vh)"' | sed 's/^/B /'
python tools/proj_probe.py | grep -E '"(vhx|sub_vh)"' | sed 's/^/B /'
