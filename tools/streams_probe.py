#!/usr/bin/env python
"""Undeflated Hutchinson probes/s on a large lattice (default 32^3 x 64,
the BASELINE configs[4] volume, eps 0.3, m0 0.05) for combinations of
concurrent solve streams x rhs per solve call (MGT_SOLVE_STREAMS /
MGT_SOLVE_BATCH): does overlapping two solves' latency-bound stencils and
HBM-bound vector kernels pay at this size?"""
import argparse
import json
import os
import sys
import time

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)


def main():
    import torch
    import paper_1909_12234_b200 as M
    ap = argparse.ArgumentParser()
    ap.add_argument("--dims", default="32x32x32x64")
    ap.add_argument("--nprobe", type=int, default=32)
    ap.add_argument("--combos", default="1x4,2x4,3x4,1x8,2x8")
    args = ap.parse_args()
    dims = tuple(int(v) for v in args.dims.split("x"))
    geo = M.LatticeGeometry(dims, "antiperiodic")
    op = M.build_wilson(M.generate_gauge(geo, "su3", eps=0.3, seed=0), 0.05)
    probes = M.build_probe_set(geo, 12, args.nprobe, hp_count=1, dilution=False, kind="rademacher", seed=300)
    for combo in args.combos.split(","):
        ns, nb = combo.split("x")
        os.environ["MGT_SOLVE_STREAMS"] = ns
        os.environ["MGT_SOLVE_BATCH"] = nb
        inv = M.TruncatedInverse(op, M.SolveConfig(tol=1e-8))
        for rep in range(2):
            torch.cuda.synchronize()
            t0 = time.perf_counter()
            est = M.hutchinson(inv, probes)
            torch.cuda.synchronize()
            el = time.perf_counter() - t0
        print(json.dumps({"dims": args.dims, "streams": int(ns), "batch": int(nb), "probes_per_s": args.nprobe / el,
                          "mean_iterations": inv.total_iterations / max(1, inv.n_solves),
                          "estimate_re": float(est.mean.real)}), flush=True)


if __name__ == "__main__":
    main()
