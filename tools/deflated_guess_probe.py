#!/usr/bin/env python
"""Iterations per probe solve from a zero start vs from the deflated initial
guess x0 = Y (U^H z) (config 4, Y = A^-1 U) or x0 = P C^-1 P^H z (config 3):
the solve of A e = z - A x0 to the same absolute residual tol ||z||."""
import os
import sys
import time

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import numpy as np  # noqa: E402
import torch  # noqa: E402

import paper_1909_12234_b200 as M  # noqa: E402
from paper_1909_12234_b200 import eigen as E  # noqa: E402
from paper_1909_12234_b200 import krylov as K  # noqa: E402
from paper_1909_12234_b200 import multigrid as MG  # noqa: E402
from paper_1909_12234_b200.linalg import vhx  # noqa: E402

tol = 1e-8
geo = M.LatticeGeometry((16, 16, 16, 16), "antiperiodic")
op = M.build_wilson(M.generate_gauge(geo, "su3", eps=0.2, seed=0), 0.1)
z = M.build_probe_set(geo, 12, 16, dilution=False, kind="rademacher", seed=200).noise_native(0, 16)
sol = K.BiCGStab(op, max_rhs=16)


def solve(b, t):
    torch.cuda.synchronize()
    t0 = time.perf_counter()
    x, reps, _ = sol.solve_native(b, t, 4000, mixed=True)
    torch.cuda.synchronize()
    return x, np.mean([r.iterations for r in reps]), time.perf_counter() - t0


def nrm(x):
    return torch.linalg.vector_norm(x.reshape(x.shape[0], -1), dim=1)


x, it0, el0 = solve(z, tol)
x, it0, el0 = solve(z, tol)
print(f"zero start: {it0:.2f} iterations, {el0 * 1e3:.1f} ms for 16 rhs", flush=True)

# config 4: 64 eigenvectors of A g5
conf = E.EigenConfig(k=64, tol=1e-3, inner=M.SolveConfig(tol=1e-3), block=8)
res = E.inexact_eigensolve(op, op.gamma5_diag, conf, E.shift_inverter_factory(op, conf.inner))
U = res.vectors
Y, _, _ = sol.solve_native(U, tol, 4000, mixed=True)
for name, x0 in [("config4 x0 = Y U^H z", torch.einsum("kn,kcv->ncv", vhx(U, z), Y))]:
    r0 = z - op.apply_native(x0)
    ratio = (nrm(z) / nrm(r0)).min().item()
    e, it1, el1 = solve(r0.contiguous(), min(0.99, tol * ratio))
    e, it1, el1 = solve(r0.contiguous(), min(0.99, tol * ratio))
    print(f"{name}: |r0|/|z| = {1 / ratio:.4f}, {it1:.2f} iterations, {el1 * 1e3:.1f} ms", flush=True)

# config 3: P from 24 null vectors, x0 = P C^-1 P^H z
nvs = MG.generate_null_vectors(op, 24, tol=1e-12, max_iter=8, seed=7)
pro = MG.build_prolongator(nvs, MG.BlockingScheme((4, 4, 4, 4)), layout_op=op)
coarse = MG.build_coarse_operator(op, pro)
Dinv = coarse.dense_inverse_native()
zc = pro.restrict_native(z)
shp = zc.shape
xc = (zc.reshape(16, -1) @ Dinv.transpose(0, 1)).reshape(shp)
x0 = pro.prolong_native(xc.contiguous())
r0 = z - op.apply_native(x0)
ratio = (nrm(z) / nrm(r0)).min().item()
e, it2, el2 = solve(r0.contiguous(), min(0.99, tol * ratio))
e, it2, el2 = solve(r0.contiguous(), min(0.99, tol * ratio))
print(f"config3 x0 = P C^-1 P^H z: |r0|/|z| = {1 / ratio:.4f}, {it2:.2f} iterations, {el2 * 1e3:.1f} ms", flush=True)
