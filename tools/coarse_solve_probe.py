#!/usr/bin/env python
"""Coarse inner solves of config 5 (32^3x64, 4^4 aggregates, nv 24): time and
iterations of 8-rhs BiCGStab at tol 1e-3 on C (full) vs its even-odd Schur
complement, and one C apply vs one S apply."""
import os, sys, time
ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import numpy as np, torch
import paper_1909_12234_b200 as M
from paper_1909_12234_b200 import multigrid as MG, _lib
from paper_1909_12234_b200._device import ptr, stream_ptr
dims = tuple(int(v) for v in (sys.argv[1] if len(sys.argv) > 1 else "32x32x32x64").split("x"))
geo = M.LatticeGeometry(dims, "antiperiodic")
op = M.build_wilson(M.generate_gauge(geo, "su3", eps=0.3, seed=0), 0.05)
nvs = MG.generate_null_vectors(op, 24, tol=1e-12, max_iter=8, seed=7)
pro = MG.build_prolongator(nvs, MG.BlockingScheme((4, 4, 4, 4)), layout_op=op)
del nvs
C = MG.build_coarse_operator(op, pro)
g = torch.Generator(device="cuda").manual_seed(1)
b = torch.randn((8, pro.n_blocks, pro.nc), dtype=torch.complex128, device="cuda", generator=g)
def ev(fn, reps=5):
    fn(); torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(True), torch.cuda.Event(True)
    e0.record()
    for _ in range(reps): fn()
    e1.record(); torch.cuda.synchronize()
    return e0.elapsed_time(e1) / reps
for low in (True, False):
    print(f"C apply 8 rhs (low={low}): {ev(lambda: C.apply_native(b, low=low)):.3f} ms")
F = C.schur_factors(0.0)
F.D32, F.E32 = F.D.to(torch.complex64), F.E.to(torch.complex64)
d, bk = pro._dims()
xe = b[:, F.ie].contiguous(); ye = torch.empty_like(xe); to = torch.empty_like(xe)
for low in (True, False):
    Dm, Em = (F.D32, F.E32) if low else (F.D, F.E)
    print(f"S apply 8 rhs (low={low}): "
          f"{ev(lambda: _lib.lib().mgt_coarse_schur_apply(d, bk, pro.nv, ptr(Dm), ptr(Em), int(low), ptr(xe), ptr(ye), ptr(to), 8, stream_ptr())):.3f} ms")
for tau in (0.0, 0.2):
    for tol in (1e-3, 1e-8):
        for eo in (False, True):
            MG.coarse_bicgstab(C, b, tol, 2000, tau, even_odd=eo)
            torch.cuda.synchronize(); t0 = time.perf_counter()
            x, reps = MG.coarse_bicgstab(C, b, tol, 2000, tau, even_odd=eo)
            torch.cuda.synchronize(); el = time.perf_counter() - t0
            print(f"tau={tau} tol={tol:g} even_odd={eo}: {el*1e3:8.1f} ms, iterations {[r[0] for r in reps]}, "
                  f"max relres {max(r[1] for r in reps):.2e}", flush=True)
