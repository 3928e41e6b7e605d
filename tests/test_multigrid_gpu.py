"""GPU multigrid setup and Algorithm-2 deflation against the reference's
golden fixtures (tests/golden/golden_4x4x4x4.npz) and the oracle
restatements (oracle/multigrid.py).  Tolerance (BASELINE north star):
P / P^H to 1e-12 relative; trace estimate within xi + 1e-10."""

import os

import numpy as np
import pytest
import scipy.sparse as sp
import torch

from oracle import multigrid as OMG
from oracle import pcg64 as P
from oracle import wilson4d as W

pytestmark = pytest.mark.gpu
GOLD = os.path.join(os.path.dirname(__file__), "golden", "golden_4x4x4x4.npz")


@pytest.fixture(scope="module")
def gold():
    return dict(np.load(GOLD))


@pytest.fixture(scope="module")
def setup(gold):
    import paper_1909_12234_b200 as M
    from paper_1909_12234_b200 import multigrid as MG
    dims = tuple(int(d) for d in gold["dims"])
    geo = M.LatticeGeometry(dims, "antiperiodic")
    gauge = M.gauge_from_array(geo, gold["links"])
    op = M.build_wilson(gauge, float(gold["mass"]))
    A = W.build_wilson4d_csr(gold["links"], dims, float(gold["mass"]))
    Pg = sp.coo_matrix((gold["P_val"], (gold["P_row"], gold["P_col"])), shape=tuple(gold["P_shape"])).tocsr()
    return M, MG, geo, op, A, Pg


def test_golden_operator(gold, setup):
    M, MG, geo, op, A, Pg = setup
    assert np.linalg.norm(op.apply(gold["x"]) - gold["Ax"]) / np.linalg.norm(gold["Ax"]) < 1e-13


def test_null_vectors_match_reference(gold, setup):
    M, MG, geo, op, A, Pg = setup
    nv = MG.generate_null_vectors(op, int(gold["null_nv"]), tol=1e-12, max_iter=8, seed=int(gold["null_seed"]))
    Y = nv.ref_vectors(op)
    G = gold["null_vectors"]
    assert np.max(np.linalg.norm(Y - G, axis=1) / np.linalg.norm(G, axis=1)) < 1e-12


def test_prolongator_matches_reference(gold, setup):
    M, MG, geo, op, A, Pg = setup
    nvs = MG.null_vectors_from_array(op, gold["null_vectors"])
    pro = MG.build_prolongator(nvs, MG.BlockingScheme(tuple(gold["block"])), layout_op=op)
    assert pro.uniform and pro.dropped == 0
    assert np.array_equal(pro.coarse_gamma5, gold["coarse_gamma5"])
    D = pro.dense()
    assert np.abs(D - Pg.toarray()).max() < 1e-12
    # P and P^H applications against the reference CSR on the same P
    rng = np.random.default_rng(1)
    x = rng.normal(size=op.dim) + 1j * rng.normal(size=op.dim)
    xc = rng.normal(size=pro.coarse_dim) + 1j * rng.normal(size=pro.coarse_dim)
    r_ref = Pg.conj().T @ x
    p_ref = Pg @ xc
    assert np.linalg.norm(pro.restrict(x) - r_ref) / np.linalg.norm(r_ref) < 1e-12
    assert np.linalg.norm(pro.prolong(xc) - p_ref) / np.linalg.norm(p_ref) < 1e-12
    # V^H V = I
    assert np.abs(D.conj().T @ D - np.eye(pro.coarse_dim)).max() < 1e-13


def test_coarse_operator_matches_reference(gold, setup):
    M, MG, geo, op, A, Pg = setup
    nvs = MG.null_vectors_from_array(op, gold["null_vectors"])
    pro = MG.build_prolongator(nvs, MG.BlockingScheme(tuple(gold["block"])), layout_op=op)
    C = MG.build_coarse_operator(op, pro)
    Cd = C.dense()
    G = gold["C_dense"]
    assert np.abs(Cd - G).max() < 1e-12 * np.abs(G).max()
    xc = np.random.default_rng(2).normal(size=C.dim) + 0.5j
    assert np.linalg.norm(C.apply(xc) - G @ xc) / np.linalg.norm(G @ xc) < 1e-12


def test_coarse_apply_multi_rhs_bitwise(gold, setup):
    """8 + 4 + 2 + 1 rhs per launch (C read once per launch): every rhs
    bitwise equal to its single-rhs apply, fp64 and fp32 C."""
    M, MG, geo, op, A, Pg = setup
    nvs = MG.null_vectors_from_array(op, gold["null_vectors"])
    pro = MG.build_prolongator(nvs, MG.BlockingScheme(tuple(gold["block"])), layout_op=op)
    C = MG.build_coarse_operator(op, pro)
    g = torch.Generator(device="cuda").manual_seed(5)
    X = torch.randn((15, pro.n_blocks, pro.nc), dtype=torch.complex128, device="cuda", generator=g)
    for low in (False, True):
        Y = C.apply_native(X, low=low)
        for r in range(15):
            assert torch.equal(Y[r], C.apply_native(X[r:r + 1].contiguous(), low=low)[0])


def test_full_coarse_deflation_matches_reference(gold, setup):
    M, MG, geo, op, A, Pg = setup
    from paper_1909_12234_b200 import trace as TR
    nvs = MG.null_vectors_from_array(op, gold["null_vectors"])
    pro = MG.build_prolongator(nvs, MG.BlockingScheme(tuple(gold["block"])), layout_op=op)
    inv = M.TruncatedInverse(op, M.SolveConfig(tol=1e-8))
    probes = M.build_probe_set(geo, 12, 3, hp_count=1, dilution=False, kind="rademacher",
                               seed=int(gold["obl_seed0"]))
    est = TR.deflate_oblique_coarse(op, inv, pro, TR.IdentityTriplets(pro.coarse_dim), pro.coarse_dim, probes)
    t0 = complex(gold["obl_t0"])
    assert abs(est.t0 - t0) < 1e-10 * abs(t0)
    # reference: GCR(32) + Y = A^-1_xi(A P); ours: BiCGStab + Y = P; both O(xi)
    rel = np.abs(est.samples - gold["obl_samples"]) / np.abs(gold["obl_samples"])
    assert rel.max() < 1e-6
    assert abs(est.mean - complex(gold["obl_mean"])) / abs(complex(gold["obl_mean"])) < 1e-8 + 1e-10


def test_coarse_bicgstab_solves(gold, setup):
    M, MG, geo, op, A, Pg = setup
    nvs = MG.null_vectors_from_array(op, gold["null_vectors"])
    pro = MG.build_prolongator(nvs, MG.BlockingScheme(tuple(gold["block"])), layout_op=op)
    C = MG.build_coarse_operator(op, pro)
    G = gold["C_dense"]
    g5c = gold["coarse_gamma5"]
    rng = np.random.default_rng(4)
    bh = rng.normal(size=(3, C.dim)) + 1j * rng.normal(size=(3, C.dim))
    b = pro.coarse_from_ref(torch.as_tensor(bh, device="cuda").reshape(3, pro.n_blocks, pro.nc))
    assert C.schur_factors() is not None  # even coarse extents: the Schur path is the default
    for tau, eo in ((0.0, True), (0.3, True), (0.0, False), (0.3, False)):
        x, reps = MG.coarse_bicgstab(C, b, 1e-11, 500, tau, even_odd=eo)
        assert all(r[2] for r in reps)
        xr = pro.coarse_to_ref(x).reshape(3, -1).cpu().numpy()
        for i in range(3):
            exact = np.linalg.solve(G + 1j * tau * np.diag(g5c), bh[i])
            assert np.linalg.norm(xr[i] - exact) / np.linalg.norm(exact) < 1e-9


def test_coarse_bicgstab_loose_fp32_path_and_edge_cases(gold, setup):
    """tol >= 1e-5 iterates with the fp32 copy of C (fp32 stencil
    arithmetic, fused device-side iteration); the contract stays the
    reference's explicit fp64 residual.  9 rhs (one 8-rhs launch + 1), one of
    them zero; a rhs at max_iter=1 reports not converged."""
    M, MG, geo, op, A, Pg = setup
    nvs = MG.null_vectors_from_array(op, gold["null_vectors"])
    pro = MG.build_prolongator(nvs, MG.BlockingScheme(tuple(gold["block"])), layout_op=op)
    C = MG.build_coarse_operator(op, pro)
    G = gold["C_dense"]
    g5c = gold["coarse_gamma5"]
    rng = np.random.default_rng(9)
    bh = rng.normal(size=(9, C.dim)) + 1j * rng.normal(size=(9, C.dim))
    bh[4] = 0.0
    b = pro.coarse_from_ref(torch.as_tensor(bh, device="cuda").reshape(9, pro.n_blocks, pro.nc))
    for tol, tau, eo in ((1e-3, 0.0, True), (1e-5, 0.2, True), (1e-3, 0.0, False), (1e-5, 0.2, False)):
        x, reps = MG.coarse_bicgstab(C, b, tol, 500, tau, even_odd=eo)
        xr = pro.coarse_to_ref(x).reshape(9, -1).cpu().numpy()
        Gt = G + 1j * tau * np.diag(g5c)
        for i in range(9):
            its, rel, conv, mv = reps[i]
            assert conv
            if i == 4:
                assert its == 0 and np.all(xr[i] == 0)
                continue
            true_rel = np.linalg.norm(bh[i] - Gt @ xr[i]) / np.linalg.norm(bh[i])
            assert true_rel <= tol and abs(true_rel - rel) <= 1e-3 * tol
    for eo in (True, False):
        _, reps = MG.coarse_bicgstab(C, b[:2], 1e-12, 1, 0.0, even_odd=eo)
        assert all(not r[2] and r[0] == 1 for r in reps)


def test_coarse_davidson_and_rank_r_oblique_deflation(gold, setup):
    M, MG, geo, op, A, Pg = setup
    from paper_1909_12234_b200 import trace as TR
    nvs = MG.null_vectors_from_array(op, gold["null_vectors"])
    pro = MG.build_prolongator(nvs, MG.BlockingScheme(tuple(gold["block"])), layout_op=op)
    C = MG.build_coarse_operator(op, pro)
    trip, res = TR.coarse_deflation_triplets(C, 8, tol=1e-6, inner_tol=1e-12)
    assert res.converged.all()
    exact = gold["ceig_exact"]
    assert np.max(np.abs(res.lambdas - exact) / np.abs(exact)) < 1e-9
    assert np.max(np.abs(res.lambdas - gold["ceig_lambdas"]) / np.abs(exact)) < 1e-9
    inv = M.TruncatedInverse(op, M.SolveConfig(tol=1e-8))
    probes = M.build_probe_set(geo, 12, 3, hp_count=1, dilution=False, kind="rademacher",
                               seed=int(gold["oblr_seed0"]))
    rank = int(gold["oblr_rank"])
    # with the reference's own coarse triplets: same t0, samples within xi
    class RefTrip:
        left = gold["ctrip_left"]
        count = gold["ctrip_left"].shape[1]
    est = TR.deflate_oblique_coarse(op, inv, pro, RefTrip, rank, probes)
    t0 = complex(gold["oblr_t0"])
    assert abs(est.t0 - t0) < 1e-10 * abs(t0)
    assert np.max(np.abs(est.samples - gold["oblr_samples"]) / np.abs(gold["oblr_samples"])) < 1e-7
    # with the GPU triplets: the same deflation subspace up to the eigen tolerance
    est2 = TR.deflate_oblique_coarse(op, inv, pro, trip, rank, probes)
    assert abs(est2.t0 - t0) < 1e-6 * abs(t0)
    assert np.max(np.abs(est2.samples - gold["oblr_samples"]) / np.abs(gold["oblr_samples"])) < 1e-6


@pytest.mark.parametrize("block", [2, 4])
def test_coarse_block_davidson(gold, setup, block):
    """Block Davidson on the coarse operator (batched coarse BiCGStab inner
    solves): the reference's coarse eigenvalues within the eigen tolerance."""
    M, MG, geo, op, A, Pg = setup
    from paper_1909_12234_b200 import trace as TR
    nvs = MG.null_vectors_from_array(op, gold["null_vectors"])
    pro = MG.build_prolongator(nvs, MG.BlockingScheme(tuple(gold["block"])), layout_op=op)
    C = MG.build_coarse_operator(op, pro)
    trip, res = TR.coarse_deflation_triplets(C, 8, tol=1e-6, inner_tol=1e-12, block=block)
    assert res.converged.all()
    exact = gold["ceig_exact"]
    assert np.max(np.abs(res.lambdas - exact) / np.abs(exact)) < 1e-9
    assert np.all(np.diff(trip.sigmas) >= 0)


def test_posterior_rank_sweep_matches_reference(gold, setup):
    M, MG, geo, op, A, Pg = setup
    from paper_1909_12234_b200 import trace as TR
    nvs = MG.null_vectors_from_array(op, gold["null_vectors"])
    pro = MG.build_prolongator(nvs, MG.BlockingScheme(tuple(gold["block"])), layout_op=op)

    class RefTrip:
        left = gold["ctrip_left"]
        count = gold["ctrip_left"].shape[1]
    inv = M.TruncatedInverse(op, M.SolveConfig(tol=1e-8))
    probes = M.build_probe_set(geo, 12, 3, hp_count=1, dilution=False, kind="rademacher",
                               seed=int(gold["oblr_seed0"]))
    post = TR.posterior_rank_sweep(op, inv, pro, RefTrip, probes, list(gold["post_grid"]))
    est = np.array([post.estimates[int(r)] for r in gold["post_grid"]])
    assert np.max(np.abs(est - gold["post_estimates"]) / np.abs(gold["post_estimates"])) < 1e-8
    var = np.array([post.variances[int(r)] for r in gold["post_grid"]])
    assert np.max(np.abs(var - gold["post_variances"]) / np.abs(gold["post_variances"])) < 1e-5
    assert post.storage_entries() == int(gold["post_storage"])
    # per-rank estimates equal a from-scratch deflate_oblique_coarse at that rank
    inv2 = M.TruncatedInverse(op, M.SolveConfig(tol=1e-8))
    e4 = TR.deflate_oblique_coarse(op, inv2, pro, RefTrip, 4, probes)
    assert abs(e4.mean - post.estimates[4]) < 1e-12 * abs(e4.mean)


@pytest.mark.parametrize("coarsest", ["lu", "bicgstab"])
def test_two_grid_inverter_matches_reference(gold, setup, coarsest):
    M, MG, geo, op, A, Pg = setup
    from paper_1909_12234_b200 import mgsolve
    nvs = MG.null_vectors_from_array(op, gold["null_vectors"])
    pro = MG.build_prolongator(nvs, MG.BlockingScheme(tuple(gold["block"])), layout_op=op)
    hier = mgsolve.Hierarchy([op, MG.build_coarse_operator(op, pro)], [pro])
    mg = mgsolve.MultigridSolver(hier, smoother_iters=4, coarse_tol=1e-1, coarsest=coarsest)
    x, rep = mg.solve(gold["probes"][0], 1e-10, max_cycles=100)
    assert rep.converged and rep.final_relres <= 1e-10
    xe = gold["mg_x"]
    assert np.linalg.norm(x - xe) / np.linalg.norm(xe) < 1e-8
    if coarsest == "lu":  # same cycle structure as the reference (exact coarse solve)
        assert abs(rep.iterations - int(gold["mg_cycles"])) <= 1
    # as a TruncatedInverse plugin (experiments.py:50-62)
    inv = M.TruncatedInverse(op, M.SolveConfig(tol=1e-10, max_iter=100), solver=mg.solver_plugin())
    y = inv(gold["probes"][1])
    r = gold["probes"][1] - A @ y
    assert np.linalg.norm(r) <= 1.01e-10 * np.linalg.norm(gold["probes"][1]) and inv.n_solves == 1


def test_config3_shape_against_oracle(cuda):
    """8^4, 4^4 aggregates, nv = 24 (the config-3 blocking at reduced volume):
    GPU null vectors + P + C against the oracle restatement."""
    import paper_1909_12234_b200 as M
    from paper_1909_12234_b200 import multigrid as MG
    dims = (8, 8, 8, 8)
    geo = M.LatticeGeometry(dims, "antiperiodic")
    gauge = M.generate_gauge(geo, "su3", eps=0.2, seed=0)
    op = M.build_wilson(gauge, 0.1)
    links = gauge.links.cpu().numpy()
    A = W.build_wilson4d_csr(links, dims, 0.1)
    nvs = MG.generate_null_vectors(op, 24, tol=1e-12, max_iter=8, seed=9)
    Yo = OMG.null_vectors(lambda v: A @ v, A.shape[0], 24, tol=1e-12, max_iter=8, seed=9)
    Yg = nvs.ref_vectors(op)
    assert np.max(np.linalg.norm(Yg - Yo, axis=1)) < 1e-11
    pro = MG.build_prolongator(nvs, MG.BlockingScheme((4, 4, 4, 4)), layout_op=op)
    Po, g5c, counts, dropped = OMG.prolongator(Yo, dims, (4, 4, 4, 4), W.gamma5_diag(geo.site_count))
    rng = np.random.default_rng(3)
    x = rng.normal(size=op.dim) + 1j * rng.normal(size=op.dim)
    assert np.linalg.norm(pro.restrict(x) - Po.conj().T @ x) / np.linalg.norm(Po.conj().T @ x) < 1e-11
    C = MG.build_coarse_operator(op, pro)
    Co = OMG.coarse_operator(A, Po, g5c).toarray()
    assert np.abs(C.dense() - Co).max() < 1e-11 * np.abs(Co).max()


GOLD_IO = os.path.join(os.path.dirname(__file__), "golden", "golden_io.npz")


def test_hierarchy_load_dump_reference_format(gold, setup, tmp_path):
    """load_hierarchy reads the REFERENCE's dump of the golden hierarchy
    (multigrid.py:409-435): P exactly, C recomputed on the GPU; dumping the
    loaded hierarchy reproduces the reference's files byte for byte."""
    M, MG, geo, op, A, Pg = setup
    g = np.load(GOLD_IO)
    src = tmp_path / "ref"
    src.mkdir()
    (src / "hierarchy_manifest.csv").write_bytes(g["hier_manifest"].tobytes())
    (src / "level0_columns.csv").write_bytes(g["hier_columns"].tobytes())
    hier = M.load_hierarchy(op, str(src))
    P = hier.prolongators[0]
    assert np.array_equal(P.dense(), Pg.toarray())
    C = hier.operators[1].dense()
    assert np.abs(C - gold["C_dense"]).max() <= 1e-12 * np.abs(gold["C_dense"]).max()
    out = tmp_path / "ours"
    M.dump_hierarchy(hier, str(out))
    assert (out / "hierarchy_manifest.csv").read_bytes() == g["hier_manifest"].tobytes()
    assert (out / "level0_columns.csv").read_bytes() == g["hier_columns"].tobytes()


def test_hierarchy_dump_of_gpu_prolongator(gold, setup, tmp_path):
    """A GPU-built P dumps with the reference's (col, site, spin) sequence
    and values within the P tolerance; the dump loads back exactly."""
    import csv
    M, MG, geo, op, A, Pg = setup
    nvs = MG.null_vectors_from_array(op, gold["null_vectors"])
    pro = MG.build_prolongator(nvs, MG.BlockingScheme(tuple(gold["block"])), layout_op=op)
    hier = M.Hierarchy([op, MG.build_coarse_operator(op, pro)], [pro])
    M.dump_hierarchy(hier, str(tmp_path))
    with open(tmp_path / "level0_columns.csv", newline="") as f:
        ours = list(csv.reader(f))
    ref = list(csv.reader(np.load(GOLD_IO)["hier_columns"].tobytes().decode().splitlines()))
    assert ours[0] == ref[0] and len(ours) == len(ref)
    assert [r[:3] for r in ours] == [r[:3] for r in ref]
    a = np.array([[float(r[3]), float(r[4])] for r in ours[1:]])
    b = np.array([[float(r[3]), float(r[4])] for r in ref[1:]])
    assert np.abs(a - b).max() < 1e-12
    back = M.load_hierarchy(op, str(tmp_path))
    assert np.array_equal(back.prolongators[0].dense(), pro.dense())


def test_tsm_correction(gold, setup):
    """trace.py:388-407: exactly 0 for equal tolerances (deterministic
    solver); otherwise the mean of z^H (A^-1_hi z - A^-1_lo z), small
    against the trace and equal to an independent evaluation."""
    M, MG, geo, op, A, Pg = setup
    assert M.tsm_correction(op, 1e-6, 1e-6, 5, seed=3) == 0.0
    with pytest.raises(ValueError):
        M.tsm_correction(op, 1e-8, 1e-6, 2, seed=3)
    c = M.tsm_correction(op, 1e-3, 1e-10, 6, seed=3, kind="rademacher")
    ps = M.build_probe_set(geo, 12, 6, hp_count=1, dilution=False, kind="rademacher", seed=3)
    acc = []
    for j0, j1 in ((0, 4), (4, 6)):
        z = ps.noise_native(j0, j1)
        _, _, qh = M.TruncatedInverse(op, M.SolveConfig(tol=1e-10)).solve_native(z, want_dot=True)
        _, _, ql = M.TruncatedInverse(op, M.SolveConfig(tol=1e-3)).solve_native(z, want_dot=True)
        acc.extend(qh - ql)
    assert c == np.mean(np.array(acc))
    z0 = P.rademacher_numpy(op.dim, 3)
    xe = np.vdot(z0, np.linalg.solve(A.toarray(), z0))
    assert 0 < abs(c) < 1e-2 * abs(xe)


def test_coarse_schur_inverse_matches_dense(gold, setup):
    """Coarse even-odd Schur factors (config 3's exact tr(C^-1) and C^-1 h):
    t0 and C^-1 h equal the dense inverse's to 1e-12, and the golden
    reference C's dense inverse (numpy) to 1e-11."""
    M, MG, geo, op, A, Pg = setup
    nvs = MG.null_vectors_from_array(op, gold["null_vectors"])
    pro = MG.build_prolongator(nvs, MG.BlockingScheme(tuple(gold["block"])), layout_op=op)
    C = MG.build_coarse_operator(op, pro)
    sch = MG.CoarseSchurInverse(C)
    Dinv = C.dense_inverse_native()
    t0d = complex(torch.diagonal(Dinv).sum().item())
    assert abs(sch.t0 - t0d) <= 1e-12 * abs(t0d)
    t0g = np.trace(np.linalg.inv(gold["C_dense"]))
    assert abs(sch.t0 - t0g) <= 1e-11 * abs(t0g)
    g = torch.Generator(device="cuda").manual_seed(8)
    H = torch.randn((5, pro.coarse_dim), dtype=torch.complex128, device="cuda", generator=g)
    Y = sch.apply_rows(H)
    Yd = H @ Dinv.transpose(0, 1)
    assert ((Y - Yd).abs().max() / Yd.abs().max()).item() < 1e-12
    assert isinstance(C.exact_inverse(), MG.CoarseSchurInverse)
