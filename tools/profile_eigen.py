#!/usr/bin/env python
"""cProfile of the GPU Davidson (host-side time split)."""
import cProfile
import os
import pstats
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import paper_1909_12234_b200 as M  # noqa: E402
from paper_1909_12234_b200 import eigen as E  # noqa: E402

k = int(sys.argv[1]) if len(sys.argv) > 1 else 16
geo = M.LatticeGeometry((16, 16, 16, 16), "antiperiodic")
op = M.build_wilson(M.generate_gauge(geo, "su3", eps=0.2, seed=0), 0.1)
conf = E.EigenConfig(k=k, tol=1e-3, inner=M.SolveConfig(tol=1e-3))
E.inexact_eigensolve(op, op.gamma5_diag, E.EigenConfig(k=2, tol=1e-3, inner=M.SolveConfig(tol=1e-3)),
                     E.shift_inverter_factory(op, conf.inner))
pr = cProfile.Profile()
pr.enable()
res = E.inexact_eigensolve(op, op.gamma5_diag, conf, E.shift_inverter_factory(op, conf.inner))
pr.disable()
print("inversions", res.inversions)
pstats.Stats(pr).sort_stats("cumulative").print_stats(25)
