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


@pytest.mark.parametrize("flags,tau", [(0, 0.0), (1, 0.0), (2, 0.0), (4, 0.4), (3, -0.3), (0, 0.7)])
def test_schur_complement_identity(cuda, flags, tau):
    """S x_e = M_ee x_e - M_eo M_oo^-1 M_oe x_e, every block taken from the
    full operator (A applied to parity-masked fields); split/merge exact."""
    import torch
    M, geo, op, A = _setup((4, 6, 4, 8), eps=0.4)
    g = torch.Generator(device="cuda").manual_seed(3)
    n, Vh = 2, geo.site_count // 2
    xe = torch.randn((n, 12, Vh), dtype=torch.complex128, device="cuda", generator=g)
    eo = torch.randn_like(xe)
    z = torch.zeros_like(xe)
    full = op.eo_merge(xe, eo)
    e2, o2 = op.eo_split(full)
    assert torch.equal(e2, xe) and torch.equal(o2, eo)
    y1e, y1o = op.eo_split(op.apply_native(op.eo_merge(xe, z), flags=flags, tau=tau))
    _, doo = op.eo_split(op.apply_native(op.eo_merge(z, eo), flags=flags, tau=tau))
    moo = doo / eo                       # M_oo is site-diagonal
    y2e, _ = op.eo_split(op.apply_native(op.eo_merge(z, y1o / moo), flags=flags, tau=tau))
    ref = y1e - y2e
    S = op.schur_apply(xe, flags=flags, tau=tau)
    rel = (torch.linalg.vector_norm(S - ref) / torch.linalg.vector_norm(ref)).item()
    assert rel < 1e-13


def test_even_odd_solve_matches_full_solve(cuda):
    """Same stopping test (full residual), half the iterations, same answer."""
    import torch
    M, geo, op, A = _setup((8, 8, 8, 8))
    N = op.dim
    z = np.stack([P.rademacher_numpy(N, 300 + j) for j in range(4)])
    zn = op.to_native(torch.as_tensor(z).cuda())
    sol = M.krylov.BiCGStab(op)
    xe, re, qe = sol.solve_native(zn, 1e-10, 2000, want_dot=True, even_odd=True)
    xf, rf, qf = sol.solve_native(zn, 1e-10, 2000, want_dot=True, even_odd=False)
    X = op.from_native(xe).cpu().numpy()
    for j in range(4):
        assert re[j].converged and rf[j].converged
        assert re[j].iterations < 0.7 * rf[j].iterations
        r = z[j] - A @ X[j]
        assert np.linalg.norm(r) <= 1.01e-10 * np.linalg.norm(z[j])
        assert abs(re[j].final_relres - np.linalg.norm(r) / np.linalg.norm(z[j])) < 1e-11
        assert abs(qe[j] - np.vdot(z[j], X[j])) < 1e-12 * abs(qe[j])
        assert abs(qe[j] - qf[j]) < 1e-8 * abs(qf[j])
    xx = (torch.linalg.vector_norm(xe - xf) / torch.linalg.vector_norm(xf)).item()
    assert xx < 1e-8


@pytest.mark.parametrize("flags,tau", [(0, 0.5), (3, -0.2), (4, 0.0)])
def test_even_odd_solve_operator_variants(cuda, flags, tau):
    import torch
    from paper_1909_12234_b200.lattice import FormOperator
    M, geo, op, A = _setup((4, 4, 4, 8), eps=0.3)
    form = FormOperator(op, flags, tau, "t")
    rng = np.random.default_rng(5)
    b = rng.normal(size=op.dim) + 1j * rng.normal(size=op.dim)
    x, rep = M.bicgstab_solve(form, b, M.SolveConfig(tol=1e-10))
    assert rep.converged
    r = b - form.apply(x)
    assert np.linalg.norm(r) <= 1.01e-10 * np.linalg.norm(b)


def test_odd_extent_solves_full_system(cuda):
    M, geo, op, A = _setup((4, 4, 4, 5))
    rng = np.random.default_rng(6)
    b = rng.normal(size=op.dim) + 1j * rng.normal(size=op.dim)
    x, rep = M.bicgstab_solve(op, b, M.SolveConfig(tol=1e-10))
    assert rep.converged
    assert np.linalg.norm(b - A @ x) <= 1.01e-10 * np.linalg.norm(b)
    import torch
    with pytest.raises(ValueError):
        op.eo_split(torch.zeros((1, 12, geo.site_count), dtype=torch.complex128, device="cuda"))


@pytest.mark.parametrize("tol", [1e-3, 1e-8, 1e-11])
def test_mixed_precision_solve_contract(cuda, tol):
    """fp32 inner cycles + fp64 defect correction: the same explicit-residual
    contract ||b - A x|| <= tol ||b|| (checked here against the oracle CSR),
    the same solution and quadratic forms as the fp64 solve within tol."""
    import torch
    M, geo, op, A = _setup((8, 8, 8, 8))
    N = op.dim
    z = np.stack([P.rademacher_numpy(N, 500 + j) for j in range(6)])
    zn = op.to_native(torch.as_tensor(z).cuda())
    sol = M.krylov.BiCGStab(op, max_rhs=8)
    xm, rm, qm = sol.solve_native(zn, tol, 4000, want_dot=True, mixed=True)
    xd, rd, qd = sol.solve_native(zn, tol, 4000, want_dot=True)
    X = op.from_native(xm).cpu().numpy()
    for j in range(6):
        assert rm[j].converged and rm[j].final_relres <= tol
        r = z[j] - A @ X[j]
        assert np.linalg.norm(r) <= 1.01 * tol * np.linalg.norm(z[j])
        assert abs(rm[j].final_relres - np.linalg.norm(r) / np.linalg.norm(z[j])) < 1e-3 * tol + 1e-13
        assert abs(qm[j] - np.vdot(z[j], X[j])) < 1e-12 * abs(qm[j])
        assert abs(qm[j] - qd[j]) < 10 * tol * abs(qd[j])
        assert rm[j].iterations <= 3 * rd[j].iterations + 16


@pytest.mark.parametrize("flags,tau", [(0, 0.5), (3, -0.2), (4, 0.0), (1, 0.3)])
def test_mixed_precision_operator_variants(cuda, flags, tau):
    from paper_1909_12234_b200.lattice import FormOperator
    M, geo, op, A = _setup((4, 4, 4, 8), eps=0.3)
    form = FormOperator(op, flags, tau, "t")
    rng = np.random.default_rng(7)
    b = rng.normal(size=op.dim) + 1j * rng.normal(size=op.dim)
    x, rep = M.bicgstab_solve(form, b, M.SolveConfig(tol=1e-10, mixed=True))
    assert rep.converged
    assert np.linalg.norm(b - form.apply(x)) <= 1.01e-10 * np.linalg.norm(b)


def test_mixed_precision_edge_cases(cuda):
    """zero rhs (done at once), max_iter exhausted (reported, not converged),
    odd extent (falls back to the fp64 full-system solve)."""
    M, geo, op, A = _setup((4, 4, 4, 4))
    cfg = M.SolveConfig(mixed=True)
    x, rep = M.bicgstab_solve(op, np.zeros(op.dim, dtype=complex), cfg)
    assert rep.converged and rep.iterations == 0 and not np.any(x)
    x, rep = M.bicgstab_solve(op, np.ones(op.dim, dtype=complex), M.SolveConfig(tol=1e-14, max_iter=3, mixed=True))
    assert not rep.converged and rep.iterations <= 3 + 8
    M2, geo2, op2, A2 = _setup((4, 4, 4, 5))
    b = np.random.default_rng(8).normal(size=op2.dim) + 0j
    x, rep = M2.bicgstab_solve(op2, b, M2.SolveConfig(tol=1e-10, mixed=True))
    assert rep.converged and np.linalg.norm(b - A2 @ x) <= 1.01e-10 * np.linalg.norm(b)


def test_mixed_hutchinson_within_tolerance(cuda):
    dims = (4, 4, 4, 8)
    M, geo, op, A = _setup(dims)
    s = 8
    probes = M.build_probe_set(geo, 12, s, hp_count=1, dilution=False, kind="rademacher", seed=23)
    est = M.hutchinson(M.TruncatedInverse(op, M.SolveConfig(tol=1e-10, mixed=True)), probes)
    lu = spla.splu(A.tocsc())
    exact = np.array([np.vdot(z, lu.solve(z)) for z in
                      (P.rademacher_numpy(op.dim, 23 + j) for j in range(s))])
    assert np.max(np.abs(est.samples - exact) / np.abs(exact)) < 1e-9


@pytest.mark.parametrize("restart", [8, 32])
def test_gmres_exact_solution_and_contract(cuda, restart):
    """Restarted GMRES(m) (C ABI mgt_gmres_solve): explicit residual within
    tol, x vs the oracle's sparse LU, counters (one matvec per Arnoldi step
    plus one explicit residual per cycle)."""
    M, geo, op, A = _setup((4, 4, 4, 8))
    rng = np.random.default_rng(11)
    b = rng.normal(size=op.dim) + 1j * rng.normal(size=op.dim)
    cfg = M.SolveConfig(tol=1e-10, kind="gmres", restart=restart)
    x, rep = M.bicgstab_solve(op, b, cfg)
    assert rep.converged and rep.final_relres <= 1e-10
    assert np.linalg.norm(b - A @ x) <= 1.01e-10 * np.linalg.norm(b)
    xe = spla.spsolve(A.tocsc(), b)
    assert np.linalg.norm(x - xe) / np.linalg.norm(xe) < 1e-8
    cycles = -(-rep.iterations // restart)
    assert rep.matvecs == rep.iterations + cycles


@pytest.mark.parametrize("flags,tau", [(0, 0.5), (3, -0.2), (4, 0.0)])
def test_gmres_operator_variants(cuda, flags, tau):
    from paper_1909_12234_b200.lattice import FormOperator
    M, geo, op, A = _setup((4, 4, 4, 8), eps=0.3)
    form = FormOperator(op, flags, tau, "t")
    rng = np.random.default_rng(12)
    b = rng.normal(size=op.dim) + 1j * rng.normal(size=op.dim)
    x, rep = M.bicgstab_solve(form, b, M.SolveConfig(tol=1e-10, kind="gmres", restart=16))
    assert rep.converged
    assert np.linalg.norm(b - form.apply(x)) <= 1.01e-10 * np.linalg.norm(b)


def test_gmres_and_gcr_edge_cases_and_estimator(cuda):
    """zero rhs, max_iter, the GCR kind, and Hutchinson through
    TruncatedInverse(kind='gmres') vs the exact quadratic forms."""
    import torch
    M, geo, op, A = _setup((4, 4, 4, 4))
    x, rep = M.bicgstab_solve(op, np.zeros(op.dim, dtype=complex), M.SolveConfig(kind="gmres"))
    assert rep.converged and rep.iterations == 0 and not np.any(x)
    b = np.ones(op.dim, dtype=complex)
    x, rep = M.bicgstab_solve(op, b, M.SolveConfig(tol=1e-14, max_iter=5, kind="gmres", restart=4))
    assert not rep.converged and rep.reason == "max_iter" and rep.iterations == 5
    x, rep = M.bicgstab_solve(op, b, M.SolveConfig(tol=1e-10, kind="gcr", restart=16))
    assert rep.converged and np.linalg.norm(b - A @ x) <= 1.01e-10 * np.linalg.norm(b)
    with pytest.raises(ValueError):
        M.SolveConfig(kind="cg")
    inv = M.TruncatedInverse(op, M.SolveConfig(tol=1e-10, kind="gmres", restart=16))
    probes = M.build_probe_set(geo, 12, 3, hp_count=1, dilution=False, kind="rademacher", seed=5)
    est = M.hutchinson(inv, probes)
    lu = spla.splu(A.tocsc())
    for j, s in enumerate(est.samples):
        z = P.rademacher_numpy(op.dim, 5 + j)
        q = np.vdot(z, lu.solve(z.astype(complex)))
        assert abs(s - q) <= 1e-8 * abs(q)
    assert inv.n_solves == 3 and inv.n_failed == 0
    zn = op.to_native(torch.as_tensor(np.stack([P.rademacher_numpy(op.dim, 5)])).cuda())
    xb, reps, dq = inv.solve_native(zn, want_dot=True)
    assert reps[0].converged and abs(dq[0] - est.samples[0]) <= 1e-9 * abs(est.samples[0])


def test_device_controlled_iteration_loop(cuda, monkeypatch):
    """MGT_SOLVE_WHILE=1: a cycle of the mixed solve is one CUDA graph launch
    whose WHILE conditional node repeats the iteration kernels on the device
    until no rhs is running (no host round trip between iteration chunks).
    Same kernels in the same order as the chunked replay: bitwise the same
    solutions, quadratic forms, iteration counts and reports."""
    import torch
    import paper_1909_12234_b200 as M
    from paper_1909_12234_b200 import krylov as K
    dims = (8, 8, 8, 8)
    geo = M.LatticeGeometry(dims, "antiperiodic")
    op = M.build_wilson(M.generate_gauge(geo, "su3", eps=0.2, seed=0), 0.1)
    probes = M.build_probe_set(geo, 12, 9, dilution=False, kind="rademacher", seed=3)
    z = probes.noise_native(0, 9)
    solver = K.BiCGStab(op, max_rhs=12)
    monkeypatch.delenv("MGT_SOLVE_WHILE", raising=False)
    x0, r0, q0 = solver.solve_native(z, 1e-8, 4000, want_dot=True, mixed=True)
    monkeypatch.setenv("MGT_SOLVE_WHILE", "1")
    x1, r1, q1 = solver.solve_native(z, 1e-8, 4000, want_dot=True, mixed=True)
    x2, r2, q2 = solver.solve_native(z, 1e-3, 4000, want_dot=True, mixed=True)
    monkeypatch.delenv("MGT_SOLVE_WHILE", raising=False)
    assert torch.equal(x0, x1) and torch.equal(torch.as_tensor(q0), torch.as_tensor(q1))
    assert [r.iterations for r in r0] == [r.iterations for r in r1]
    assert all(r.converged and r.final_relres <= 1e-8 for r in r1)
    assert all(r.converged and r.final_relres <= 1e-3 for r in r2)
    # max_iter is honoured on the device (the loop ends when every rhs stopped)
    monkeypatch.setenv("MGT_SOLVE_WHILE", "1")
    x3, r3, _ = solver.solve_native(z[:2], 1e-12, 3, want_dot=True, mixed=True)
    assert all((not r.converged) and r.iterations <= 4 for r in r3)
