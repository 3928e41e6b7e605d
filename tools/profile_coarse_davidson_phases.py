#!/usr/bin/env python
"""Phase split of the BASELINE configs[4] coarse block Davidson (device-
synchronised timers around every building block; unperturbed total first)."""
import collections
import os
import sys
import time

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import torch  # noqa: E402

import paper_1909_12234_b200 as M  # noqa: E402
from paper_1909_12234_b200 import eigen as E  # noqa: E402
from paper_1909_12234_b200 import multigrid as MG  # noqa: E402
from paper_1909_12234_b200 import trace as TR  # noqa: E402

dims = tuple(int(v) for v in os.environ.get("MGT_DIMS", "32x32x32x64").split("x"))
geo = M.LatticeGeometry(dims, "antiperiodic")
op = M.build_wilson(M.generate_gauge(geo, "su3", eps=0.3, seed=0), 0.05)
nvs = MG.generate_null_vectors(op, 24, tol=1e-12, max_iter=8, seed=7)
pro = MG.build_prolongator(nvs, MG.BlockingScheme((4, 4, 4, 4)), layout_op=op)
del nvs
coarse = MG.build_coarse_operator(op, pro)


def run():
    torch.cuda.synchronize()
    t0 = time.perf_counter()
    trip, cres = TR.coarse_deflation_triplets(coarse, 64, tol=1e-3, inner_tol=1e-3, block=8)
    torch.cuda.synchronize()
    return cres, time.perf_counter() - t0


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
wrap(E.CoarseTruncatedInverse, "solve_native")
wrap(E._CoarseOps, "random")
wrap(E._CoarseOps, "g5")
wrap(E._CoarseOps, "apply_h")
res, t = run()
print(f"instrumented: {t:.3f} s")
for n, (c, s) in sorted(acc.items(), key=lambda kv: -kv[1][1]):
    print(f"  {n:14s} {c:6d} calls {s:8.3f} s  ({1e3 * s / c:7.3f} ms each)")
print("  (_orth_block includes its cgs2 / vhx / _rot / _norms calls)")
