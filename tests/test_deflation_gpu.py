"""GPU projection kernels, Algorithm-1 (orthogonal) deflation and the
inexact Davidson eigensolver against numpy and the reference's golden
fixtures.  Tolerances: projections 1e-12 relative (fp64); eigenvalues
within the eigen tolerance of the dense oracle; trace within xi + 1e-10."""

import os

import numpy as np
import pytest
import torch

from oracle import wilson4d as W

pytestmark = pytest.mark.gpu
GOLD = os.path.join(os.path.dirname(__file__), "golden", "golden_4x4x4x4.npz")


@pytest.fixture(scope="module")
def gold():
    return dict(np.load(GOLD))


@pytest.fixture(scope="module")
def setup(gold):
    import paper_1909_12234_b200 as M
    dims = tuple(int(d) for d in gold["dims"])
    geo = M.LatticeGeometry(dims, "antiperiodic")
    op = M.build_wilson(M.gauge_from_array(geo, gold["links"]), float(gold["mass"]))
    return M, geo, op


@pytest.mark.parametrize("k,s,n", [(64, 1, 49152), (64, 4, 49152), (64, 128, 20000), (5, 3, 1001), (70, 9, 777),
                                   (208, 8, 49152), (70, 6, 777), (8, 136, 49152), (3, 20, 1001), (1, 9, 513),
                                   (64, 16, 49152), (144, 16, 7777), (40, 32, 3001), (64, 33, 2049),
                                   # even lengths, 4 < s <= 16, k > 8: the FP64 tensor-core (DMMA) kernel,
                                   # ragged vector / column / length tails
                                   (70, 9, 778), (20, 5, 1002), (144, 16, 7778), (65, 12, 4098), (9, 8, 6),
                                   (129, 7, 49154),
                                   # whole 32-element tiles: the bulk-copy (cp.async.bulk + mbarrier) pipeline,
                                   # fewer tiles than CTAs, ragged vector blocks
                                   (129, 7, 49248), (70, 9, 800), (9, 8, 32), (200, 16, 64), (65, 5, 12288),
                                   # at least two 256-element tiles per SM: the pipelined X - V H kernel
                                   (70, 9, 76800), (144, 16, 75776), (203, 8, 78848), (12, 5, 76032)])
def test_projection_kernels_vs_numpy(cuda, k, s, n):
    from paper_1909_12234_b200 import linalg as LA
    rng = np.random.default_rng(k + s)
    V = rng.normal(size=(k, n)) + 1j * rng.normal(size=(k, n))
    X = rng.normal(size=(s, n)) + 1j * rng.normal(size=(s, n))
    Vd, Xd = torch.as_tensor(V, device=cuda), torch.as_tensor(X, device=cuda)
    H = LA.vhx(Vd, Xd).cpu().numpy()
    Hr = V.conj() @ X.T
    assert np.linalg.norm(H - Hr) / np.linalg.norm(Hr) < 1e-13
    # the C-ABI projection kernels themselves at every shape (vhx hands
    # k > 8, s >= 32 to cuBLAS by default); deterministic
    Hk = LA.vhx(Vd, Xd, gemm=False)
    assert np.linalg.norm(Hk.cpu().numpy() - Hr) / np.linalg.norm(Hr) < 1e-13
    assert torch.equal(Hk, LA.vhx(Vd, Xd, gemm=False))
    LA.sub_vh(Vd, torch.as_tensor(Hr, device=cuda), Xd)
    Xr = X - (V.T @ Hr).T
    assert np.linalg.norm(Xd.cpu().numpy() - Xr) / np.linalg.norm(Xr) < 1e-13
    # determinism
    assert torch.equal(LA.vhx(Vd, Xd), LA.vhx(Vd, Xd))


def test_orthogonal_deflation_matches_reference(gold, setup):
    M, geo, op = setup
    from paper_1909_12234_b200 import trace as TR
    inv = M.TruncatedInverse(op, M.SolveConfig(tol=1e-8))
    probes = M.build_probe_set(geo, 12, 3, hp_count=1, dilution=False, kind="rademacher",
                               seed=int(gold["orth_seed0"]))
    est = TR.deflate_orthogonal(inv, gold["eig_vectors"], probes)
    t0 = complex(gold["orth_t0"])
    assert abs(est.t0 - t0) < 1e-8 * abs(t0) + 1e-10
    rel = np.abs(est.samples - gold["orth_samples"]) / np.abs(gold["orth_samples"])
    assert rel.max() < 1e-8 + 1e-10
    with pytest.raises(TR.DeflationContractError):
        TR.deflate_orthogonal(inv, 2.0 * gold["eig_vectors"], probes)


def test_orthogonal_deflation_guess_matches_zero_start(gold, setup):
    """The deflated start x0 = Y U^H z computes the same slot values
    z^H (x - Y U^H z) within the solver tolerance; residuals are reported
    relative to the probe and meet tol."""
    M, geo, op = setup
    from paper_1909_12234_b200 import trace as TR
    probes = M.build_probe_set(geo, 12, 6, hp_count=1, dilution=False, kind="rademacher", seed=77)
    tol = 1e-9
    inv_g = M.TruncatedInverse(op, M.SolveConfig(tol=tol))
    inv_z = M.TruncatedInverse(op, M.SolveConfig(tol=tol))
    eg = TR.deflate_orthogonal(inv_g, gold["eig_vectors"], probes, guess=True)
    ez = TR.deflate_orthogonal(inv_z, gold["eig_vectors"], probes, guess=False)
    assert eg.t0 == ez.t0
    assert np.max(np.abs(eg.samples - ez.samples) / np.abs(ez.samples)) < 10 * tol
    assert inv_g.n_solves == inv_z.n_solves
    assert inv_g.n_failed == 0 and inv_g.last_report.final_relres <= tol


def test_davidson_eigenpairs_match_reference(gold, setup):
    M, geo, op = setup
    from paper_1909_12234_b200 import eigen as E
    conf = E.EigenConfig(k=6, tol=1e-4, inner=M.SolveConfig(tol=1e-10))
    res = E.inexact_eigensolve(op, op.gamma5_diag, conf, E.shift_inverter_factory(op, conf.inner))
    assert res.converged.all()
    exact = gold["eig_exact"]
    assert np.max(np.abs(res.lambdas - exact) / np.abs(exact)) < 1e-6
    assert np.max(np.abs(res.lambdas - gold["eig_lambdas"]) / np.abs(exact)) < 1e-6
    # orthonormal eigenvectors of A gamma5
    from paper_1909_12234_b200 import linalg as LA
    G = LA.vhx(res.vectors, res.vectors).cpu().numpy()
    assert np.abs(G - np.eye(6)).max() < 1e-10
    trip = E.to_singular_triplets(res)
    assert np.all(np.diff(trip.sigmas) >= 0)


@pytest.mark.parametrize("block", [2, 4])
def test_block_davidson_eigenpairs(gold, setup, block):
    """Block Davidson (BASELINE configs[3] block size): the same eigenpairs as
    the dense oracle / the reference's block-1 run within the eigen tolerance."""
    M, geo, op = setup
    from paper_1909_12234_b200 import eigen as E
    from paper_1909_12234_b200 import linalg as LA
    conf = E.EigenConfig(k=6, tol=1e-4, inner=M.SolveConfig(tol=1e-10), block=block)
    res = E.inexact_eigensolve(op, op.gamma5_diag, conf, E.shift_inverter_factory(op, conf.inner))
    assert res.converged.all()
    exact = gold["eig_exact"]
    assert np.max(np.abs(res.lambdas - exact) / np.abs(exact)) < 1e-6
    G = LA.vhx(res.vectors, res.vectors).cpu().numpy()
    assert np.abs(G - np.eye(6)).max() < 1e-10
    assert res.residuals.max() < 1e-3
    # the batched applications are counted per vector
    assert res.inversions >= 6


def test_block_davidson_config_errors():
    from paper_1909_12234_b200 import eigen as E
    with pytest.raises(ValueError):
        E.EigenConfig(k=4, block=0)
    with pytest.raises(ValueError):
        E.EigenConfig(k=4, max_basis=8, block=5)


GOLD_SWEEP = os.path.join(os.path.dirname(__file__), "golden", "golden_sweep.npz")


def test_orthogonal_rank_sweep_matches_reference(cuda, gold, setup):
    """experiments.py:205-243 (the reference's golden run, tol 1e-10 solves):
    per-rank mean, t0, variance and inversion counts; rank r of the sweep
    equals deflate_orthogonal with the first r vectors on the same probes."""
    M, geo, op = setup
    from paper_1909_12234_b200 import trace as TR
    g = np.load(GOLD_SWEEP)
    U = gold["eig_vectors"]
    Un = op.to_native(torch.as_tensor(np.ascontiguousarray(U.T)).cuda())
    inv = M.TruncatedInverse(op, M.SolveConfig(tol=1e-10))
    lefts, _, _ = inv.solve_native(Un)
    ps = M.build_probe_set(geo, 12, int(g["sweep_s"]), hp_count=1, dilution=False, kind="rademacher",
                           seed=int(g["sweep_seed"]))
    grid = [int(r) for r in g["sweep_grid"]]
    res = TR.orthogonal_rank_sweep(M.TruncatedInverse(op, M.SolveConfig(tol=1e-10)), Un, lefts, ps, grid)
    for i, r in enumerate(grid):
        assert abs(res[r].mean - g["sweep_mean"][i]) < 1e-8 * abs(g["sweep_mean"][i])
        assert abs(res[r].t0 - g["sweep_t0"][i]) < 1e-8 * max(abs(g["sweep_t0"][i]), 1.0)
        assert abs(res[r].variance - g["sweep_var"][i]) < 1e-6 * g["sweep_var"][i]
        assert res[r].inversions == int(g["sweep_inv"][i])
    r = 3
    est = TR.deflate_orthogonal(M.TruncatedInverse(op, M.SolveConfig(tol=1e-10)), Un[:r], ps)
    assert abs(est.mean - res[r].mean) < 1e-9 * abs(est.mean)


def test_subspace_angles_match_reference(cuda, gold, setup):
    M, geo, op = setup
    from paper_1909_12234_b200 import multigrid as MG
    g = np.load(GOLD_SWEEP)
    nvs = MG.null_vectors_from_array(op, gold["null_vectors"])
    pro = MG.build_prolongator(nvs, MG.BlockingScheme(tuple(gold["block"])), layout_op=op)
    ang = MG.subspace_angles(pro, g["angles_vectors"])
    assert np.abs(ang - g["angles"]).max() < 1e-7
