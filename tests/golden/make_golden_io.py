#!/usr/bin/env python
"""Golden files for the reference's file formats, written
by the REFERENCE's own functions (importable only in the build container):
hierarchy dump (multigrid.py:384-407) of the golden 4^4 prolongator, results
CSV / angles CSV (experiments.py:93-146) and MANIFEST (:149-161).  The file
texts are stored in tests/golden/golden_io.npz.

    python tests/golden/make_golden_io.py
"""

import os
import sys
import tempfile

import numpy as np
import scipy.sparse as sp

HERE = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, "/root/reference/pkg/src")

from mgtrace import experiments, lattice, multigrid  # noqa: E402


def main():
    g = np.load(os.path.join(HERE, "golden_4x4x4x4.npz"))
    dims = tuple(int(v) for v in g["dims"])
    geo = lattice.LatticeGeometry(dims, "antiperiodic")
    block = tuple(int(v) for v in g["block"])
    Pm = sp.coo_matrix((g["P_val"], (g["P_row"], g["P_col"])), shape=tuple(g["P_shape"])).tocsr()
    blocking = multigrid.BlockingScheme(block)
    m = blocking.block_count(geo)
    nv = int(g["null_nv"])
    P = multigrid.Prolongator(Pm, g["coarse_gamma5"], blocking, geo, 12, np.full((m, 2), nv), 0)
    out = {}
    with tempfile.TemporaryDirectory() as d:
        multigrid.dump_hierarchy(multigrid.Hierarchy([None, None], [P]), d)
        out["hier_manifest"] = np.frombuffer(open(os.path.join(d, "hierarchy_manifest.csv"), "rb").read(), np.uint8)
        out["hier_columns"] = np.frombuffer(open(os.path.join(d, "level0_columns.csv"), "rb").read(), np.uint8)
        rows = [{"rank": r, "hp_count": 1, "variance": float(v), "jackknife_err": float(v) / 3,
                 "t0_re": 1.0 / 3, "t0_im": -2.0 / 7, "estimate_re": float(e), "estimate_im": 1e-17 * r,
                 "inversions": 10 + r}
                for r, (e, v) in enumerate(zip(g["post_estimates"].real, g["post_variances"]))]
        experiments.write_results_csv(os.path.join(d, "results.csv"), rows)
        experiments.write_angles_csv(os.path.join(d, "angles.csv"), [0.0, 1e-3 / 3, 0.5, 1.0])
        experiments.write_manifest(d, ["results.csv", "angles.csv"], status="ok")
        for name in ("results.csv", "angles.csv", "MANIFEST.csv"):
            out[name.replace(".", "_")] = np.frombuffer(open(os.path.join(d, name), "rb").read(), np.uint8)
        out["results_rows_rank"] = np.array([r["rank"] for r in rows])
        out["results_rows_variance"] = np.array([r["variance"] for r in rows])
        out["results_rows_estimate_re"] = np.array([r["estimate_re"] for r in rows])
    np.savez_compressed(os.path.join(HERE, "golden_io.npz"), **out)
    print({k: v.shape for k, v in out.items()})


if __name__ == "__main__":
    main()
