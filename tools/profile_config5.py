#!/usr/bin/env python
"""cProfile of the BASELINE configs[4] setup (null vectors, P, C, coarse
Davidson) -- host-side time split."""
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
torch.cuda.synchronize()
pr = cProfile.Profile()
pr.enable()
t0 = time.perf_counter()
nvs = MG.generate_null_vectors(op, 24, tol=1e-12, max_iter=8, seed=7)
torch.cuda.synchronize()
t1 = time.perf_counter()
pro = MG.build_prolongator(nvs, MG.BlockingScheme((4, 4, 4, 4)), layout_op=op)
coarse = MG.build_coarse_operator(op, pro)
torch.cuda.synchronize()
t2 = time.perf_counter()
trip, cres = TR.coarse_deflation_triplets(coarse, 64, tol=1e-3, inner_tol=1e-3, block=8)
torch.cuda.synchronize()
t3 = time.perf_counter()
pr.disable()
print(f"null vectors {t1 - t0:.2f} s, P + C {t2 - t1:.2f} s, coarse Davidson {t3 - t2:.2f} s "
      f"({cres.inversions} inversions)")
pstats.Stats(pr).sort_stats("tottime").print_stats(18)
geo_p = M.build_probe_set(geo, 12, 64, hp_count=1, dilution=False, kind="rademacher", seed=300)
inv = M.TruncatedInverse(op, M.SolveConfig(tol=1e-8))
pr2 = cProfile.Profile()
torch.cuda.synchronize()
t4 = time.perf_counter()
pr2.enable()
est = TR.deflate_oblique_coarse(op, inv, pro, trip, 64, geo_p, coarse_op=coarse)
torch.cuda.synchronize()
pr2.disable()
t5 = time.perf_counter()
print(f"estimator, 64 probes: {t5 - t4:.2f} s, mean iterations {inv.total_iterations / max(1, inv.n_solves):.1f}")
pstats.Stats(pr2).sort_stats("tottime").print_stats(15)
