"""CPU tests: pin the oracle restatements against the reference's golden
fixtures (tests/golden/, made by make_golden.py from the real reference) and,
in the build container, against the importable reference itself."""

import os

import numpy as np
import pytest

from oracle import krylov as K
from oracle import multigrid as MG
from oracle import pcg64 as P
from oracle import trace as T
from oracle import wilson4d as W

GOLD = os.path.join(os.path.dirname(__file__), "golden", "golden_4x4x4x4.npz")


@pytest.fixture(scope="module")
def gold():
    return dict(np.load(GOLD, allow_pickle=False))


@pytest.fixture(scope="module")
def small_op(gold):
    dims = tuple(int(d) for d in gold["dims"])
    A = W.build_wilson4d_csr(gold["links"], dims, float(gold["mass"]))
    return dims, A


# ---- operator restatement -------------------------------------------------

def test_gamma_algebra():
    for a in range(4):
        for b in range(4):
            ac = W.GAMMAS[a] @ W.GAMMAS[b] + W.GAMMAS[b] @ W.GAMMAS[a]
            assert np.allclose(ac, 2 * np.eye(4) * (a == b), atol=0)
    assert np.array_equal(np.diag(W.GAMMA5).real, [1, 1, -1, -1])


def test_links_are_su3_and_match_golden(gold):
    dims = tuple(int(d) for d in gold["dims"])
    U = W.su3_links(dims, float(gold["eps"]), 0)
    assert np.abs(U - gold["links"]).max() == 0.0
    eye = np.einsum("...ij,...kj->...ik", U, U.conj())
    assert np.abs(eye - np.eye(3)).max() < 1e-14
    assert np.abs(np.linalg.det(U) - 1).max() < 1e-14


def test_operator_matches_golden(gold, small_op):
    dims, A = small_op
    assert np.abs(A @ gold["x"] - gold["Ax"]).max() == 0.0
    assert np.abs(A.conj().T @ gold["x"] - gold["Adx"]).max() == 0.0
    assert A.nnz == 49 * A.shape[0]


def test_stencil_matches_csr(small_op, gold):
    dims, A = small_op
    y = W.apply_stencil(gold["links"], dims, float(gold["mass"]), gold["x"])
    assert np.linalg.norm(y - gold["Ax"]) / np.linalg.norm(gold["Ax"]) < 1e-14


def test_site_local_stencil_matches_csr(small_op, gold):
    dims, A = small_op
    sites = [0, 1, 5, 63, 100, 255]
    got = W.apply_at_sites(gold["links"], dims, float(gold["mass"]), gold["x"], sites)
    want = gold["Ax"].reshape(-1, 12)[sites]
    assert np.abs(got - want).max() < 1e-14 * np.abs(want).max()


def test_gamma5_hermiticity(small_op):
    dims, A = small_op
    g5 = W.gamma5_diag(A.shape[0] // 12)
    D = A.toarray()
    assert np.abs(g5[:, None] * D * g5[None, :] - D.conj().T).max() == 0.0


def test_plane_wave_kat():
    dims = (4, 4, 6, 8)
    A = W.build_wilson4d_csr(W.unit_links(dims), dims, 0.1)
    rng = np.random.default_rng(0)
    for k in [(1, 2, 3, 4), (0, 0, 0, 0), (3, 1, 5, 7)]:
        p, M = W.plane_wave_symbol(dims, 0.1, k)
        chi = rng.normal(size=(4, 3)) + 1j * rng.normal(size=(4, 3))
        v = W.plane_wave(dims, p, chi)
        e = W.plane_wave(dims, p, M @ chi)
        assert np.linalg.norm(A @ v - e) / np.linalg.norm(e) < 1e-14


@pytest.mark.reference
def test_free_field_spectrum_vs_reference(mgtrace_ref):
    geo = mgtrace_ref.lattice.LatticeGeometry((2, 2, 4, 4), "antiperiodic")
    A = W.build_wilson4d_csr(W.unit_links(geo.dims), geo.dims, 0.1)
    ev = np.sort_complex(np.round(np.linalg.eigvals(A.toarray()), 8))
    ff = np.sort_complex(np.round(np.repeat(mgtrace_ref.lattice.free_field_eigenvalues(geo, 0.1), 6), 8))
    assert np.abs(ev - ff).max() < 1e-7


@pytest.mark.reference
def test_reference_lattice_operator_wraps_oracle(mgtrace_ref, gold, small_op):
    dims, A = small_op
    L = mgtrace_ref.lattice
    geo = L.LatticeGeometry(dims, "antiperiodic")
    op = L.LatticeOperator(geo, 12, A, L.gamma5_pattern(geo.site_count, 12))
    assert np.array_equal(op.apply(gold["x"]), gold["Ax"])
    assert np.array_equal(op.apply_shifted(0.5, gold["x"]), gold["Ashift"])
    fwd, bwd, fph, bph = geo.neighbor_tables()
    f2, b2, fp2, bp2 = W.neighbor_tables(dims, True)
    assert np.array_equal(fwd, f2) and np.array_equal(bwd, b2)
    assert np.array_equal(fph, fp2) and np.array_equal(bph, bp2)


# ---- probes ---------------------------------------------------------------

def test_pcg64_restatement_vs_numpy_and_golden(gold):
    N = gold["probes"].shape[1]
    for j in range(gold["probes"].shape[0]):
        seed = int(gold["probe_seed0"]) + j
        v = P.rademacher(N, seed)
        assert np.array_equal(v.view(np.uint64), gold["probes"][j].view(np.uint64))
    for seed in (0, 3, 2**40 + 7):
        st, inc = P.seed_state(seed)
        bg = np.random.PCG64(seed)
        assert list(map(int, bg.random_raw(8))) == P.raw64(st, inc, 8)[0]
        bg2 = np.random.PCG64(seed)
        bg2.advance(1000003)
        assert P.jump(st, inc, 1000003) == int(bg2.state["state"]["state"])


@pytest.mark.reference
def test_make_noise_vs_reference(mgtrace_ref):
    for kind, fn in (("rademacher", P.rademacher), ("z4", P.z4)):
        for seed in (0, 17):
            ref = mgtrace_ref.probing.make_noise(1000, kind, seed).values
            got = fn(1000, seed)
            assert np.array_equal(ref.view(np.uint64), got.view(np.uint64))


# ---- Krylov / estimators --------------------------------------------------

def test_gcr_restatement_matches_golden(gold, small_op):
    dims, A = small_op
    x, rep = K.gcr(lambda v: A @ v, gold["probes"][0], 1e-10, 2000, 32)
    assert np.array_equal(x, gold["gcr_x"])
    assert rep.iterations == int(gold["gcr_iters"]) and rep.matvecs == int(gold["gcr_matvecs"])


def test_hutchinson_restatement_matches_golden(gold, small_op):
    dims, A = small_op
    inv = K.TruncatedInverse(lambda v: A @ v, 1e-8)
    est = T.hutchinson(inv, [[z] for z in gold["probes"]])
    assert np.array_equal(est["samples"], gold["hutch_samples"])
    assert est["mean"] == complex(gold["hutch_mean"])
    assert est["variance"] == float(gold["hutch_variance"])
    assert est["jackknife_err"] == float(gold["hutch_jk"])
    assert inv.total_iterations == int(gold["hutch_iters"])


@pytest.mark.reference
def test_jackknife_vs_reference(mgtrace_ref):
    s = np.random.default_rng(3).normal(size=17) + 1j
    assert T.jackknife(s) == mgtrace_ref.trace.jackknife(s)


# ---- multigrid --------------------------------------------------------------

def test_null_vectors_restatement_matches_golden(gold, small_op):
    dims, A = small_op
    Y = MG.null_vectors(lambda v: A @ v, A.shape[0], int(gold["null_nv"]), tol=1e-12, max_iter=8,
                        seed=int(gold["null_seed"]))
    assert np.array_equal(Y, gold["null_vectors"])


def test_prolongator_and_coarse_restatement_match_golden(gold, small_op):
    dims, A = small_op
    g5 = W.gamma5_diag(A.shape[0] // 12)
    Pm, g5c, counts, dropped = MG.prolongator(gold["null_vectors"], dims, tuple(gold["block"]), g5)
    import scipy.sparse as sp
    Pg = sp.coo_matrix((gold["P_val"], (gold["P_row"], gold["P_col"])), shape=tuple(gold["P_shape"])).tocsr()
    assert dropped == 0 and np.array_equal(g5c, gold["coarse_gamma5"])
    assert abs(Pm - Pg).max() < 1e-15
    C = MG.coarse_operator(A, Pm, g5c).toarray()
    assert np.abs(C - gold["C_dense"]).max() < 1e-13 * np.abs(C).max()


def test_full_coarse_deflation_restatement_matches_golden(gold, small_op):
    dims, A = small_op
    import scipy.sparse as sp
    Pg = sp.coo_matrix((gold["P_val"], (gold["P_row"], gold["P_col"])), shape=tuple(gold["P_shape"])).tocsr()
    inv = K.TruncatedInverse(lambda v: A @ v, 1e-8)
    N = A.shape[0]
    probes = [[P.rademacher(N, int(gold["obl_seed0"]) + j)] for j in range(3)]
    est = T.deflate_full_coarse(inv, Pg, gold["C_dense"], probes)
    assert abs(est["t0"] - complex(gold["obl_t0"])) < 1e-10 * abs(complex(gold["obl_t0"]))
    # the reference uses Y = A^-1_xi (A P) in place of P: differences O(xi)
    assert np.max(np.abs(est["samples"] - gold["obl_samples"]) / np.abs(gold["obl_samples"])) < 1e-6


def test_orthogonal_deflation_restatement_matches_golden(gold, small_op):
    dims, A = small_op
    inv = K.TruncatedInverse(lambda v: A @ v, 1e-8)
    N = A.shape[0]
    probes = [[P.rademacher(N, int(gold["orth_seed0"]) + j)] for j in range(3)]
    est = T.deflate_orthogonal(inv, gold["eig_vectors"], probes)
    assert est["t0"] == complex(gold["orth_t0"])
    assert np.array_equal(est["samples"], gold["orth_samples"])


def test_reference_eigenvalues_are_accurate(gold):
    # the reference Davidson's Rayleigh-Ritz values vs the dense oracle
    assert np.max(np.abs(gold["eig_lambdas"] - gold["eig_exact"]) / np.abs(gold["eig_exact"])) < 1e-6
