import time, sys, os
sys.path.insert(0, os.getcwd())
import torch, numpy as np
import paper_1909_12234_b200 as M
from paper_1909_12234_b200 import eigen as E, trace as TR
geo = M.LatticeGeometry((16,16,16,16), "antiperiodic")
op = M.build_wilson(M.generate_gauge(geo, "su3", eps=0.2, seed=0), 0.1)
for k, tol in [(16, 1e-3), (64, 1e-3)]:
    conf = E.EigenConfig(k=k, tol=tol, inner=M.SolveConfig(tol=1e-3))
    torch.cuda.synchronize(); t0 = time.perf_counter()
    res = E.inexact_eigensolve(op, op.gamma5_diag, conf, E.shift_inverter_factory(op, conf.inner))
    torch.cuda.synchronize(); el = time.perf_counter() - t0
    print(k, tol, "eig seconds", round(el,2), "inversions", res.inversions, "converged", int(res.converged.sum()), "lam", res.lambdas[:4], "res", res.residuals[:4], flush=True)
inv = M.TruncatedInverse(op, M.SolveConfig(tol=1e-8))
probes = M.build_probe_set(geo, 12, 128, dilution=False, kind="rademacher", seed=200)
for rep in range(2):
    torch.cuda.synchronize(); t0 = time.perf_counter()
    est = TR.deflate_orthogonal(inv, res.vectors, probes)
    torch.cuda.synchronize(); el = time.perf_counter() - t0
print("deflated probes/s", 128/el, "t0", est.t0, "mean", est.mean, "var", est.variance)
est0 = M.hutchinson(inv, probes)
print("undeflated var", est0.variance, "mean", est0.mean)
