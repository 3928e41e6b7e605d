#!/usr/bin/env python
"""Golden fixtures for a 3-level hierarchy and its MG inverter, produced by
the REFERENCE (`build_hierarchy` with two blockings, multigrid.py:328-341;
`MultigridSolver` recursing through level 1, :344-381) on the 8^4 SU(3)
operator of oracle/wilson4d.py wrapped in the reference's LatticeOperator.
Writes tests/golden/golden_mg3_8x8x8x8.npz (the links are regenerated from
the oracle's seeded generator in the test).

    python tests/golden/make_golden_mg3.py
"""

import os
import sys

import numpy as np

HERE = os.path.dirname(os.path.abspath(__file__))
ROOT = os.path.dirname(os.path.dirname(HERE))
sys.path.insert(0, ROOT)
sys.path.insert(0, "/root/reference/pkg/src")

from mgtrace import lattice, multigrid, probing  # noqa: E402

from oracle import wilson4d as W  # noqa: E402


def main():
    dims, eps, mass, lseed = (8, 8, 8, 8), 0.2, 0.1, 1
    geo = lattice.LatticeGeometry(dims, "antiperiodic")
    links = W.su3_links(dims, eps, lseed)
    A = W.build_wilson4d_csr(links, dims, mass)
    op = lattice.LatticeOperator(geo, 12, A, lattice.gamma5_pattern(geo.site_count, 12))
    blockings, counts, seed = [(2, 2, 2, 2), (2, 2, 2, 2)], [6, 4], 17
    hier = multigrid.build_hierarchy(op, blockings, counts, null_tol=1e-12, null_max_iter=8, seed=seed)
    C1, C2 = hier.operators[1], hier.operators[2]
    P1 = hier.prolongators[1].matrix.tocoo()
    # level-1 null vectors exactly as build_hierarchy drew them
    nv1 = multigrid.generate_null_vectors(C1, counts[1], tol=1e-12, max_iter=8, seed=seed + 7)
    b = probing.make_noise(op.dim, "rademacher", seed=5).values
    out = {"dims": np.array(dims), "eps": eps, "mass": mass, "links_seed": lseed,
           "blockings": np.array(blockings), "counts": np.array(counts), "seed": seed,
           "nv1": nv1.vectors, "P1_row": P1.row, "P1_col": P1.col, "P1_val": P1.data,
           "P1_shape": np.array(P1.shape), "C2_dense": C2.matrix.toarray(), "b": b}
    for coarsest in ("lu", "gcr"):
        mg = multigrid.MultigridSolver(hier, smoother_iters=4, coarse_tol=1e-1, coarsest=coarsest)
        x, rep = mg.solve(b, 1e-10, max_cycles=100)
        out[f"x_{coarsest}"] = x
        out[f"cycles_{coarsest}"] = rep.iterations
        out[f"converged_{coarsest}"] = rep.converged
    np.savez_compressed(os.path.join(HERE, "golden_mg3_8x8x8x8.npz"), **out)
    print({k: np.shape(v) for k, v in out.items()}, out["cycles_lu"], out["cycles_gcr"])


if __name__ == "__main__":
    main()
