"""GPU BiCGStab (TruncatedInverse plugin) against the oracle's exact solves."""

import numpy as np
import pytest
import scipy.sparse.linalg as spla

from oracle import pcg64 as P
from oracle import wilson4d as W

pytestmark = pytest.mark.gpu


def _setup(dims, eps=0.2, mass=0.1, seed=0):
    import paper_1909_12234_b200 as M
    geo = M.LatticeGeometry(dims, "antiperiodic")
    gauge = M.generate_gauge(geo, "su3", eps=eps, seed=seed)
    op = M.build_wilson(gauge, mass)
    A = W.build_wilson4d_csr(gauge.links.cpu().numpy(), dims, mass)
    return M, geo, op, A


def test_bicgstab_explicit_residual_and_exact_solution(cuda):
    M, geo, op, A = _setup((4, 4, 4, 8))
    rng = np.random.default_rng(0)
    b = rng.normal(size=op.dim) + 1j * rng.normal(size=op.dim)
    x, rep = M.bicgstab_solve(op, b, M.SolveConfig(tol=1e-10))
    assert rep.converged and rep.final_relres <= 1e-10
    r = b - A @ x
    assert np.linalg.norm(r) <= 1.01e-10 * np.linalg.norm(b)
    xe = spla.spsolve(A.tocsc(), b)
    assert np.linalg.norm(x - xe) / np.linalg.norm(xe) < 1e-8
    assert rep.matvecs >= 2 * rep.iterations


def test_zero_rhs_and_max_iter(cuda):
    M, geo, op, A = _setup((4, 4, 4, 4))
    x, rep = M.bicgstab_solve(op, np.zeros(op.dim, dtype=complex), M.SolveConfig())
    assert rep.converged and rep.iterations == 0 and not np.any(x)
    b = np.ones(op.dim, dtype=complex)
    x, rep = M.bicgstab_solve(op, b, M.SolveConfig(tol=1e-14, max_iter=3))
    assert not rep.converged and rep.reason == "max_iter" and rep.iterations == 3


def test_truncated_inverse_counters_and_batch(cuda):
    M, geo, op, A = _setup((4, 4, 4, 8), eps=0.3)
    inv = M.TruncatedInverse(op, M.SolveConfig(tol=1e-9))
    N = op.dim
    z = [P.rademacher_numpy(N, 100 + j) for j in range(5)]
    ys = [inv(v) for v in z]
    assert inv.n_solves == 5 and inv.n_failed == 0
    import torch
    zn = op.to_native(torch.as_tensor(np.stack(z)).cuda())
    xb, reps, q = inv.solve_native(zn, want_dot=True)
    xr = op.from_native(xb).cpu().numpy()
    for j in range(5):
        assert np.linalg.norm(xr[j] - ys[j]) / np.linalg.norm(ys[j]) < 1e-8
        assert abs(q[j] - np.vdot(z[j], xr[j])) < 1e-12 * abs(q[j])
    assert inv.n_solves == 10


def test_hutchinson_matches_exact_quadratic_forms(cuda):
    dims = (4, 4, 4, 8)
    M, geo, op, A = _setup(dims)
    s = 6
    probes = M.build_probe_set(geo, 12, s, hp_count=1, dilution=False, kind="rademacher", seed=17)
    inv = M.TruncatedInverse(op, M.SolveConfig(tol=1e-10))
    est = M.hutchinson(inv, probes)
    lu = spla.splu(A.tocsc())
    exact = np.array([np.vdot(z, lu.solve(z)) for z in
                      (P.rademacher_numpy(op.dim, 17 + j) for j in range(s))])
    assert np.max(np.abs(est.samples - exact) / np.abs(exact)) < 1e-9
    assert est.s == s and est.inversions == s
    assert abs(est.mean - exact.mean()) / abs(exact.mean()) < 1e-9
