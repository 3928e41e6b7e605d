"""Coarse even-odd form at the production block size (2 nv = 48, as BASELINE
configs[2]/[4]): the Schur apply S = C_ee - C_eo C_oo^-1 C_oe through the
half-stencil kernels (mgt_coarse_half_apply / mgt_coarse_schur_apply, fp64
and fp32 blocks, 1..9 rhs per call) against the dense complement built in
numpy from the same random 9-block operator; and the Schur BiCGStab's
solution against a dense solve."""

import numpy as np
import pytest

pytestmark = pytest.mark.gpu

CD = (2, 2, 4, 2)
NV = 24


def _coarse_nbr(b, d):
    C0, C1, C2, C3 = CD
    c2 = b % C2
    r = b // C2
    c1 = r % C1
    r //= C1
    c0, c3 = r % C0, r // C0
    if d == 0:
        return b
    mu, s = (d - 1) >> 1, (-1 if (d - 1) & 1 else 1)
    c = [c0, c1, c2, c3]
    c[mu] = (c[mu] + s) % CD[mu]
    return ((c[3] * C0 + c[0]) * C1 + c[1]) * C2 + c[2]


@pytest.fixture(scope="module")
def coarse_case():
    import torch
    rng = np.random.default_rng(11)
    nb, nc = int(np.prod(CD)), 2 * NV
    C = (rng.normal(size=(nb, 9, nc, nc)) + 1j * rng.normal(size=(nb, 9, nc, nc))) * 0.05
    C[:, 0] += 4.0 * np.eye(nc)
    dense = np.zeros((nb * nc, nb * nc), complex)
    for b in range(nb):
        for d in range(9):
            n = _coarse_nbr(b, d)
            dense[b * nc:(b + 1) * nc, n * nc:(n + 1) * nc] += C[b, d].T  # storage is column-major
    return torch.as_tensor(C.reshape(-1)).cuda(), dense, nb, nc


@pytest.mark.parametrize("tau", [0.0, 0.25])
def test_schur_apply_matches_dense(cuda, coarse_case, tau):
    import torch
    from paper_1909_12234_b200 import _lib, multigrid as MG
    from paper_1909_12234_b200._device import ptr, stream_ptr
    Cd, dense, nb, nc = coarse_case
    F = MG.coarse_schur_blocks(Cd, CD, NV, tau)
    g5 = np.tile(np.r_[np.ones(NV), -np.ones(NV)], nb)
    Dt = dense + np.diag(1j * tau * g5)
    ie, io = F.ie.cpu().numpy(), F.io.cpu().numpy()
    iE = (ie[:, None] * nc + np.arange(nc)).ravel()
    iO = (io[:, None] * nc + np.arange(nc)).ravel()
    S = Dt[np.ix_(iE, iE)] - Dt[np.ix_(iE, iO)] @ np.linalg.solve(Dt[np.ix_(iO, iO)], Dt[np.ix_(iO, iE)])
    d, bk = _lib.dims_arg(CD), _lib.dims_arg((1, 1, 1, 1))
    rng = np.random.default_rng(3)
    for n in (1, 2, 3, 4, 8, 9):
        xh = rng.normal(size=(n, nb // 2, nc)) + 1j * rng.normal(size=(n, nb // 2, nc))
        x = torch.as_tensor(xh).cuda()
        ref = np.einsum("ij,nj->ni", S, xh.reshape(n, -1))
        for fp32, tol in ((0, 1e-12), (1, 2e-6)):
            D, E = (F.D, F.E) if not fp32 else (F.D.to(torch.complex64), F.E.to(torch.complex64))
            y, t = torch.empty_like(x), torch.empty_like(x)
            _lib.check(_lib.lib().mgt_coarse_schur_apply(d, bk, NV, ptr(D), ptr(E), fp32, ptr(x), ptr(y), ptr(t), n,
                                                         stream_ptr()))
            err = np.abs(y.cpu().numpy().reshape(n, -1) - ref).max() / np.abs(ref).max()
            assert err < tol, (n, fp32, err)


def test_schur_bicgstab_solution(cuda, coarse_case):
    """The even-odd coarse BiCGStab (multigrid._schur_bicgstab through a
    CoarseOperator-shaped stand-in) solves the full system to tol."""
    import types

    import torch
    from paper_1909_12234_b200 import multigrid as MG
    Cd, dense, nb, nc = coarse_case

    class _Pr:
        nv = NV
        n_blocks = nb
        geometry = types.SimpleNamespace(dims=CD)
        blocking = types.SimpleNamespace(block_dims=(1, 1, 1, 1))

        def _dims(self):
            from paper_1909_12234_b200 import _lib
            return _lib.dims_arg(CD), _lib.dims_arg((1, 1, 1, 1))

    coarse = types.SimpleNamespace(prolongator=_Pr(), C=Cd)
    rng = np.random.default_rng(5)
    bh = rng.normal(size=(5, nb, nc)) + 1j * rng.normal(size=(5, nb, nc))
    bh[2] = 0.0
    b = torch.as_tensor(bh).cuda()
    for tau, tol in ((0.0, 1e-10), (0.3, 1e-4)):
        F = MG.coarse_schur_blocks(Cd, CD, NV, tau)
        x, reps = MG._schur_bicgstab(coarse, F, b, tol, 400)
        g5 = np.tile(np.r_[np.ones(NV), -np.ones(NV)], nb)
        Dt = dense + np.diag(1j * tau * g5)
        xr = x.cpu().numpy().reshape(5, -1)
        for i in range(5):
            its, rel, conv, mv = reps[i]
            assert conv
            if i == 2:
                assert its == 0 and not np.any(xr[i])
                continue
            true_rel = np.linalg.norm(bh[i].ravel() - Dt @ xr[i]) / np.linalg.norm(bh[i])
            assert true_rel <= tol * 1.0001, (tau, i, true_rel)
