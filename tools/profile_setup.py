#!/usr/bin/env python
"""Setup time split of BASELINE configs[2] (null vectors, P, C, dense C^-1)
(coarse Schur C^-1 factors) and configs[3] (inexact Davidson), plus a cProfile of the eigensolve."""
import cProfile
import os
import pstats
import sys
import time

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import torch  # noqa: E402

import paper_1909_12234_b200 as M  # noqa: E402
from paper_1909_12234_b200 import eigen as E  # noqa: E402
from paper_1909_12234_b200 import multigrid as MG  # noqa: E402

block = int(os.environ.get("MGT_EIG_BLOCK", "1"))
geo = M.LatticeGeometry((16, 16, 16, 16), "antiperiodic")
op = M.build_wilson(M.generate_gauge(geo, "su3", eps=0.2, seed=0), 0.1)


def tick():
    torch.cuda.synchronize()
    return time.perf_counter()


for rep in range(int(os.environ.get("MGT_SETUP_REPS", "3"))):
    t0 = tick()
    nvs = MG.generate_null_vectors(op, 24, tol=1e-12, max_iter=8, seed=7)
    t1 = tick()
    pro = MG.build_prolongator(nvs, MG.BlockingScheme((4, 4, 4, 4)), layout_op=op)
    t2 = tick()
    coarse = MG.build_coarse_operator(op, pro)
    t3 = tick()
    coarse.exact_inverse()
    t4 = tick()
    print(f"[config3 rep {rep}] null vectors {t1 - t0:.3f} s, P {t2 - t1:.3f} s, C {t3 - t2:.3f} s, "
          f"exact C^-1 factors {t4 - t3:.3f} s, total {t4 - t0:.3f} s", flush=True)

kw = {"block": block} if block > 1 else {}
conf = E.EigenConfig(k=64, tol=1e-3, inner=M.SolveConfig(tol=1e-3), **kw)
E.inexact_eigensolve(op, op.gamma5_diag, E.EigenConfig(k=2, tol=1e-3, inner=M.SolveConfig(tol=1e-3)),
                     E.shift_inverter_factory(op, conf.inner))
pr = cProfile.Profile()
t0 = tick()
pr.enable()
res = E.inexact_eigensolve(op, op.gamma5_diag, conf, E.shift_inverter_factory(op, conf.inner))
pr.disable()
t1 = tick()
print(f"[config4 block {block}] eigensolve {t1 - t0:.3f} s, inversions {res.inversions}, "
      f"converged {int(res.converged.sum())}, max residual {res.residuals.max():.2e}", flush=True)
pstats.Stats(pr).sort_stats("cumulative").print_stats(40)
