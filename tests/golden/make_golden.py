#!/usr/bin/env python
"""Generate the golden fixtures of tests/golden/ by running the REFERENCE
package (`/root/reference/pkg/src/mgtrace`, importable only in the build
container) on the 4D SU(3) Wilson operator of oracle/wilson4d.py wrapped in
the reference's own `LatticeOperator` (lattice.py:194-256).

Everything downstream of the operator is the reference's code: probes
(probing.py:94-165), GCR / TruncatedInverse (krylov.py:52-229), null
vectors, prolongator and Galerkin coarse operator (multigrid.py:74-259),
Hutchinson and full-V oblique deflation (trace.py:122-274).

    python tests/golden/make_golden.py      # writes tests/golden/*.npz
"""

import os
import sys

import numpy as np

HERE = os.path.dirname(os.path.abspath(__file__))
ROOT = os.path.dirname(os.path.dirname(HERE))
sys.path.insert(0, ROOT)
sys.path.insert(0, "/root/reference/pkg/src")

from mgtrace import krylov, lattice, multigrid, probing, trace  # noqa: E402

from oracle import wilson4d as W  # noqa: E402


def reference_operator(dims, eps, mass, seed):
    geo = lattice.LatticeGeometry(tuple(dims), "antiperiodic")
    links = W.su3_links(dims, eps, seed)
    A = W.build_wilson4d_csr(links, dims, mass)
    op = lattice.LatticeOperator(geo, 12, A, lattice.gamma5_pattern(geo.site_count, 12))
    return geo, links, op


def main():
    dims, eps, mass = (4, 4, 4, 4), 0.2, 0.1
    geo, links, op = reference_operator(dims, eps, mass, 0)
    N = op.dim
    rng = np.random.default_rng(2024)
    x = (rng.normal(size=N) + 1j * rng.normal(size=N)) / np.sqrt(2)
    out = {"dims": np.array(dims), "eps": eps, "mass": mass, "links": links, "x": x,
           "Ax": op.apply(x), "Adx": op.apply_dagger(x), "Ashift": op.apply_shifted(0.5, x)}

    # probes (bitwise) and Hutchinson with the reference GCR(32), tol 1e-8
    s, seed0 = 6, 11
    ps = probing.build_probe_set(geo, 12, s, hp_count=1, dilution=False, kind="rademacher", seed=seed0)
    out["probes"] = np.stack([g.slots[0] for g in ps.groups])
    out["probe_seed0"] = seed0
    inv = krylov.TruncatedInverse(op, krylov.SolveConfig(tol=1e-8))
    est = trace.hutchinson(inv, ps)
    out["hutch_samples"] = est.samples
    out["hutch_mean"] = est.mean
    out["hutch_variance"] = est.variance
    out["hutch_jk"] = est.jackknife_err
    out["hutch_iters"] = inv.total_iterations
    # one explicit GCR solve
    xs, rep = krylov.gcr_solve(op, out["probes"][0], krylov.SolveConfig(tol=1e-10))
    out["gcr_x"] = xs
    out["gcr_iters"] = rep.iterations
    out["gcr_matvecs"] = rep.matvecs

    # multigrid: 6 null vectors relaxed by GCR(8), 2^4 aggregates
    nv, block, nseed = 6, (2, 2, 2, 2), 5
    nulls = multigrid.generate_null_vectors(op, nv, tol=1e-12, max_iter=8, seed=nseed)
    out["null_vectors"] = nulls.vectors
    out["null_seed"] = nseed
    out["null_nv"] = nv
    out["block"] = np.array(block)
    P = multigrid.build_prolongator(nulls, multigrid.BlockingScheme(block))
    Pc = P.matrix.tocoo()
    out["P_row"], out["P_col"], out["P_val"] = Pc.row, Pc.col, Pc.data
    out["P_shape"] = np.array(P.matrix.shape)
    out["coarse_gamma5"] = P.coarse_gamma5
    C = multigrid.build_coarse_operator(op, P)
    out["C_dense"] = C.matrix.toarray()
    # full-V oblique deflation = deflate_oblique_coarse with identity triplets
    Nc = P.coarse_dim

    class Identity:
        count = Nc
        left = np.eye(Nc, dtype=np.complex128)

    inv2 = krylov.TruncatedInverse(op, krylov.SolveConfig(tol=1e-8))
    ps2 = probing.build_probe_set(geo, 12, 3, hp_count=1, dilution=False, kind="rademacher", seed=40)
    est2 = trace.deflate_oblique_coarse(op, inv2, P, Identity(), Nc, ps2)
    out["obl_t0"] = est2.t0
    out["obl_samples"] = est2.samples
    out["obl_mean"] = est2.mean
    out["obl_seed0"] = 40
    # Algorithm 1: inexact Davidson eigenpairs of A gamma5, then orthogonal
    # deflation with the reference's own U
    from mgtrace import eigen
    econf = eigen.EigenConfig(k=6, tol=1e-4, inner=krylov.SolveConfig(tol=1e-10))
    fac = eigen.shift_inverter_factory(op, econf.inner)
    res = eigen.inexact_eigensolve(op, op.gamma5_diag, econf, fac)
    out["eig_lambdas"] = res.lambdas
    out["eig_residuals"] = res.residuals
    out["eig_converged"] = res.converged
    out["eig_vectors"] = res.vectors
    out["eig_exact"] = eigen.dense_triplets(op).lambdas[:6]
    inv3 = krylov.TruncatedInverse(op, krylov.SolveConfig(tol=1e-8))
    ps3 = probing.build_probe_set(geo, 12, 3, hp_count=1, dilution=False, kind="rademacher", seed=70)
    est3 = trace.deflate_orthogonal(inv3, res.vectors, ps3)
    out["orth_t0"] = est3.t0
    out["orth_samples"] = est3.samples
    out["orth_seed0"] = 70
    # hierarchical probing + dilution slots (probing.py:146-165), 2 groups each
    out["hp_seed"] = 21
    for hp, dil, kind in [(1, True, "z4"), (16, False, "rademacher"), (16, True, "z4"), (256, False, "z4")]:
        ps_hp = probing.build_probe_set(geo, 12, 2, hp_count=hp, dilution=dil, kind=kind, seed=21)
        out[f"hp_{hp}_{int(dil)}_{kind}"] = np.stack([g.slots for g in ps_hp.groups])

    ps_hp = probing.build_probe_set(geo, 12, 2, hp_count=16, dilution=False, kind="z4", seed=21)
    inv_hp = krylov.TruncatedInverse(op, krylov.SolveConfig(tol=1e-8))
    est_hp = trace.hutchinson(inv_hp, ps_hp)
    out["hp16_samples"] = est_hp.samples
    out["hp16_mean"] = est_hp.mean

    # Algorithm 2 at rank r: coarse Davidson triplets (experiments.py:65-74),
    # then the rank-r oblique deflation
    cconf = eigen.EigenConfig(k=8, tol=1e-6, inner=krylov.SolveConfig(tol=1e-12))
    cfac = eigen.shift_inverter_factory(C, cconf.inner)
    cres = eigen.inexact_eigensolve(C, C.gamma5_diag, cconf, cfac)
    ctrip = eigen.to_singular_triplets(cres, C.gamma5_diag)
    out["ceig_lambdas"] = cres.lambdas
    out["ceig_exact"] = eigen.dense_triplets(C).lambdas[:8]
    out["ctrip_left"] = ctrip.left
    inv4 = krylov.TruncatedInverse(op, krylov.SolveConfig(tol=1e-8))
    ps4 = probing.build_probe_set(geo, 12, 3, hp_count=1, dilution=False, kind="rademacher", seed=90)
    est4 = trace.deflate_oblique_coarse(op, inv4, P, ctrip, 6, ps4)
    out["oblr_rank"] = 6
    out["oblr_t0"] = est4.t0
    out["oblr_samples"] = est4.samples
    out["oblr_seed0"] = 90
    inv5 = krylov.TruncatedInverse(op, krylov.SolveConfig(tol=1e-8))
    post = trace.posterior_rank_sweep(op, inv5, P, ctrip, ps4, [0, 2, 4, 6])
    out["post_grid"] = np.array([0, 2, 4, 6])
    out["post_estimates"] = np.array([post.estimates[r] for r in (0, 2, 4, 6)])
    out["post_variances"] = np.array([post.variances[r] for r in (0, 2, 4, 6)])
    out["post_storage"] = post.storage_entries()
    # two-grid MG inverter (multigrid.py:262-381) with the golden hierarchy
    hier = multigrid.Hierarchy([op, C], [P])
    mg = multigrid.MultigridSolver(hier, smoother_iters=4, coarse_tol=1e-1)
    xmg, repmg = mg.solve(out["probes"][0], 1e-10, max_cycles=100)
    out["mg_x"] = xmg
    out["mg_cycles"] = repmg.iterations
    out["mg_matvecs"] = repmg.matvecs
    np.savez_compressed(os.path.join(HERE, "golden_4x4x4x4.npz"), **out)
    print("wrote golden_4x4x4x4.npz", {k: np.shape(v) for k, v in out.items()})


if __name__ == "__main__":
    main()
