#!/usr/bin/env python
"""cProfile (cumulative) of the BASELINE configs[4] coarse Davidson alone:
where the non-solve time of Algorithm 2's setup goes."""
import cProfile
import os
import pstats
import sys
import time

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import torch  # noqa: E402

import paper_1909_12234_b200 as M  # noqa: E402
from paper_1909_12234_b200 import multigrid as MG  # noqa: E402
from paper_1909_12234_b200 import trace as TR  # noqa: E402

geo = M.LatticeGeometry((32, 32, 32, 64), "antiperiodic")
op = M.build_wilson(M.generate_gauge(geo, "su3", eps=0.3, seed=0), 0.05)
nvs = MG.generate_null_vectors(op, 24, tol=1e-12, max_iter=8, seed=7)
pro = MG.build_prolongator(nvs, MG.BlockingScheme((4, 4, 4, 4)), layout_op=op)
del nvs
coarse = MG.build_coarse_operator(op, pro)
torch.cuda.synchronize()
pr = cProfile.Profile()
t0 = time.perf_counter()
pr.enable()
trip, cres = TR.coarse_deflation_triplets(coarse, 64, tol=1e-3, inner_tol=1e-3, block=8)
torch.cuda.synchronize()
pr.disable()
print(f"coarse Davidson {time.perf_counter() - t0:.2f} s ({cres.inversions} inversions)")
pstats.Stats(pr).sort_stats("cumulative").print_stats(45)
