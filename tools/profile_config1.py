#!/usr/bin/env python
"""Host-side time split of BASELINE configs[0] (8^4 Hutchinson, 32 probes)."""
import cProfile
import os
import pstats
import sys
import time

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import torch  # noqa: E402

import paper_1909_12234_b200 as M  # noqa: E402

geo = M.LatticeGeometry((8, 8, 8, 8), "antiperiodic")
op = M.build_wilson(M.generate_gauge(geo, "su3", eps=0.2, seed=0), 0.1)
inv = M.TruncatedInverse(op, M.SolveConfig(tol=1e-8))
probes = M.build_probe_set(geo, 12, 32, hp_count=1, dilution=False, kind="rademacher", seed=0)
for _ in range(3):
    M.hutchinson(inv, probes)
torch.cuda.synchronize()
t0 = time.perf_counter()
for _ in range(20):
    M.hutchinson(inv, probes)
torch.cuda.synchronize()
print(f"hutchinson: {(time.perf_counter() - t0) / 20 * 1e3:.3f} ms per 32 probes")
z = probes.noise_native(0, 32)
solver = M.krylov._solver_for(op)
torch.cuda.synchronize()
t0 = time.perf_counter()
for _ in range(20):
    solver.solve_native(z, 1e-8, 2000, want_dot=True, mixed=True)
torch.cuda.synchronize()
print(f"solve_native alone: {(time.perf_counter() - t0) / 20 * 1e3:.3f} ms per 32 rhs")
pr = cProfile.Profile()
pr.enable()
for _ in range(20):
    M.hutchinson(inv, probes)
pr.disable()
pstats.Stats(pr).sort_stats("tottime").print_stats(15)
