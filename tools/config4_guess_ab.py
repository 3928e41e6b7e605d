#!/usr/bin/env python
"""BASELINE configs[3] estimator: deflated start (guess=True, per-rhs
tolerances) vs zero start with the projection correction (guess=False);
probes/s, mean iterations, estimate."""
import os, sys, time
ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import torch
import paper_1909_12234_b200 as M
from paper_1909_12234_b200 import eigen as E, trace as TR
geo = M.LatticeGeometry((16, 16, 16, 16), "antiperiodic")
op = M.build_wilson(M.generate_gauge(geo, "su3", eps=0.2, seed=0), 0.1)
conf = E.EigenConfig(k=64, tol=1e-3, inner=M.SolveConfig(tol=1e-3), block=8)
res = E.inexact_eigensolve(op, op.gamma5_diag, conf, E.shift_inverter_factory(op, conf.inner))
probes = M.build_probe_set(geo, 12, 128, hp_count=1, dilution=False, kind="rademacher", seed=200)
for guess in (True, False, True, False):
    inv = M.TruncatedInverse(op, M.SolveConfig(tol=1e-8))
    for rep in range(2):
        inv.n_solves = inv.total_iterations = 0
        torch.cuda.synchronize(); t0 = time.perf_counter()
        est = TR.deflate_orthogonal(inv, res.vectors, probes, guess=guess)
        torch.cuda.synchronize(); el = time.perf_counter() - t0
    print(f"guess={guess}: {128 / el:.1f} probes/s, {el * 1e3:.1f} ms, mean iterations "
          f"{inv.total_iterations / max(1, inv.n_solves):.2f}, estimate {est.mean.real:.6f}", flush=True)
