#!/usr/bin/env python
"""Null-vector generation split at 32^3 x 64 (config 5): host normal stream
(NormalStream.take of 2N values) vs H2D + GCR(8) relaxation on the GPU, per
vector, synchronised timers."""
import os, sys, time
ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import numpy as np, torch
import paper_1909_12234_b200 as M
from paper_1909_12234_b200 import multigrid as MG
from paper_1909_12234_b200.rng import NormalStream
from paper_1909_12234_b200._device import device
dims = tuple(int(v) for v in (sys.argv[1] if len(sys.argv) > 1 else "32x32x32x64").split("x"))
geo = M.LatticeGeometry(dims, "antiperiodic")
op = M.build_wilson(M.generate_gauge(geo, "su3", eps=0.3, seed=0), 0.05)
N = op.dim
for rep in range(2):
    normals = NormalStream(np.random.default_rng(7))
    re_h = torch.empty(N, dtype=torch.float64).pin_memory()
    im_h = torch.empty(N, dtype=torch.float64).pin_memory()
    t_take = t_gpu = 0.0
    torch.cuda.synchronize()
    T0 = time.perf_counter()
    for i in range(8):
        t0 = time.perf_counter()
        normals.take(N, out=re_h.numpy())
        normals.take(N, out=im_h.numpy())
        t1 = time.perf_counter()
        y0 = op.to_native(torch.complex(re_h.to(device(), non_blocking=True), im_h.to(device(), non_blocking=True)))
        b = -op.apply_native(y0)
        d, its, conv, why, _ = MG.gcr_relax(op, b, 1e-12, 8, 8)
        y = y0 + d
        yn = torch.linalg.vector_norm(y).item()
        torch.cuda.synchronize()
        t2 = time.perf_counter()
        t_take += t1 - t0
        t_gpu += t2 - t1
    print(f"rep {rep}: 8 vectors {time.perf_counter() - T0:.3f} s: take {t_take:.3f} s, H2D+relax {t_gpu:.3f} s",
          flush=True)
t0 = time.perf_counter()
nv = MG.generate_null_vectors(op, 24, tol=1e-12, max_iter=8, seed=7)
torch.cuda.synchronize()
print(f"generate_null_vectors(24): {time.perf_counter() - t0:.3f} s")
