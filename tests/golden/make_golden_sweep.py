#!/usr/bin/env python
"""Golden values of the reference's orthogonal-deflation rank sweep
(experiments.py:205-243) and principal-angle diagnostics
(multigrid.py:303-313) on the 4^4 golden problem (tests/golden/golden_4x4x4x4.npz),
computed by the REFERENCE.  Writes tests/golden/golden_sweep.npz.

    python tests/golden/make_golden_sweep.py
"""

import os
import sys

import numpy as np
import scipy.sparse as sp

HERE = os.path.dirname(os.path.abspath(__file__))
ROOT = os.path.dirname(os.path.dirname(HERE))
sys.path.insert(0, ROOT)
sys.path.insert(0, "/root/reference/pkg/src")

from mgtrace import experiments, krylov, lattice, multigrid, probing  # noqa: E402

from oracle import wilson4d as W  # noqa: E402


def main():
    g = np.load(os.path.join(HERE, "golden_4x4x4x4.npz"))
    dims = tuple(int(v) for v in g["dims"])
    geo = lattice.LatticeGeometry(dims, "antiperiodic")
    A = W.build_wilson4d_csr(g["links"], dims, float(g["mass"]))
    op = lattice.LatticeOperator(geo, 12, A, lattice.gamma5_pattern(geo.site_count, 12))
    U = g["eig_vectors"]
    inv = krylov.TruncatedInverse(op, krylov.SolveConfig(tol=1e-10))
    lefts = np.stack([inv(U[:, i]) for i in range(U.shape[1])], axis=1)
    ps = probing.build_probe_set(geo, 12, 8, hp_count=1, dilution=False, kind="rademacher", seed=120)
    inv2 = krylov.TruncatedInverse(op, krylov.SolveConfig(tol=1e-10))
    grid = [0, 1, 3, 6]
    res = experiments.orthogonal_rank_sweep(inv2, U, lefts, ps, grid)
    Pm = sp.coo_matrix((g["P_val"], (g["P_row"], g["P_col"])), shape=tuple(g["P_shape"])).tocsr()
    blocking = multigrid.BlockingScheme(tuple(int(v) for v in g["block"]))
    m = blocking.block_count(geo)
    P = multigrid.Prolongator(Pm, g["coarse_gamma5"], blocking, geo, 12, np.full((m, 2), int(g["null_nv"])), 0)
    vecs = np.concatenate([U.T, g["null_vectors"][:2] / np.linalg.norm(g["null_vectors"][:2], axis=1)[:, None]])
    out = {"sweep_grid": np.array(grid), "sweep_seed": 120, "sweep_s": 8,
           "sweep_mean": np.array([res[r].mean for r in grid]),
           "sweep_var": np.array([res[r].variance for r in grid]),
           "sweep_t0": np.array([res[r].t0 for r in grid]),
           "sweep_inv": np.array([res[r].inversions for r in grid]),
           "angles_vectors": vecs, "angles": multigrid.subspace_angles(P, vecs)}
    np.savez_compressed(os.path.join(HERE, "golden_sweep.npz"), **out)
    print({k: np.shape(v) for k, v in out.items()}, out["angles"])


if __name__ == "__main__":
    main()
