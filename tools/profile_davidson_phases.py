#!/usr/bin/env python
"""Phase split of the block Davidson (config 4): every building block wrapped
in a device-synchronised timer (the syncs perturb the total a little; the
unperturbed total is printed first)."""
import collections
import os
import sys
import time

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import torch  # noqa: E402

import paper_1909_12234_b200 as M  # noqa: E402
from paper_1909_12234_b200 import eigen as E  # noqa: E402

block = int(os.environ.get("MGT_EIG_BLOCK", "8"))
k = int(os.environ.get("MGT_EIG_K", "64"))
geo = M.LatticeGeometry((16, 16, 16, 16), "antiperiodic")
op = M.build_wilson(M.generate_gauge(geo, "su3", eps=0.2, seed=0), 0.1)
conf = E.EigenConfig(k=k, tol=1e-3, inner=M.SolveConfig(tol=1e-3), block=block)


def run():
    torch.cuda.synchronize()
    t0 = time.perf_counter()
    res = E.inexact_eigensolve(op, op.gamma5_diag, conf, E.shift_inverter_factory(op, conf.inner))
    torch.cuda.synchronize()
    return res, time.perf_counter() - t0


run()
for _ in range(2):
    res, t = run()
    print(f"unperturbed: {t:.3f} s, inversions {res.inversions}, converged {int(res.converged.sum())}")

acc = collections.defaultdict(lambda: [0, 0.0])


def wrap(mod, name, label=None):
    f = getattr(mod, name)

    def g(*a, **kw):
        torch.cuda.synchronize()
        t0 = time.perf_counter()
        out = f(*a, **kw)
        torch.cuda.synchronize()
        e = acc[label or name]
        e[0] += 1
        e[1] += time.perf_counter() - t0
        return out

    setattr(mod, name, g)


for n in ["vhx", "cgs2", "_rot", "_extract", "_norms", "_orth_block"]:
    wrap(E, n)
from paper_1909_12234_b200 import krylov as K  # noqa: E402
wrap(K.TruncatedInverse, "solve_native", "solve_native")
wrap(E._FineOps, "random", "random")
wrap(E._FineOps, "g5", "g5")
res, t = run()
print(f"instrumented: {t:.3f} s")
for n, (c, s) in sorted(acc.items(), key=lambda kv: -kv[1][1]):
    print(f"  {n:14s} {c:6d} calls {s:8.3f} s  ({1e3 * s / c:7.3f} ms each)")
print("  (_orth_block includes its cgs2 / vhx / _rot / _norms calls)")
