#!/usr/bin/env python
"""Time the GPU BiCGStab on config-1/config-3 shaped problems with different
right-hand-side group sizes (CUDA events + wall clock)."""

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
    from paper_1909_12234_b200 import krylov as K
    ap = argparse.ArgumentParser()
    ap.add_argument("--dims", default="8x8x8x8,16x16x16x16")
    ap.add_argument("--groups", default="1,2,4")
    ap.add_argument("--nprobe", type=int, default=16)
    ap.add_argument("--recon", type=int, default=12)
    ap.add_argument("--tol", type=float, default=1e-8)
    ap.add_argument("--mixed", default="0", help="comma list of 0/1")
    args = ap.parse_args()
    for ds in args.dims.split(","):
        dims = tuple(int(v) for v in ds.split("x"))
        geo = M.LatticeGeometry(dims, "antiperiodic")
        op = M.build_wilson(M.generate_gauge(geo, "su3", eps=0.2, seed=0), 0.1, recon=args.recon)
        probes = M.build_probe_set(geo, 12, args.nprobe, dilution=False, kind="rademacher", seed=0)
        z = probes.noise_native(0, args.nprobe)
        solver = K.BiCGStab(op, max_rhs=max(4, max(int(v) for v in args.groups.split(","))))
        for g, mixed in [(int(v), int(m)) for v in args.groups.split(",") for m in args.mixed.split(",")]:
            for rep in range(2):
                torch.cuda.synchronize()
                t0 = time.perf_counter()
                its = []
                for j0 in range(0, args.nprobe, g):
                    x, reps, q = solver.solve_native(z[j0:j0 + g], args.tol, 4000, want_dot=True, mixed=bool(mixed))
                    its += [r.iterations for r in reps]
                torch.cuda.synchronize()
                el = time.perf_counter() - t0
            print(json.dumps({"dims": ds, "group": g, "mixed": mixed, "tol": args.tol,
                              "probes_per_s": args.nprobe / el, "max_relres": max(r.final_relres for r in reps),
                              "ms_per_probe": el / args.nprobe * 1e3, "mean_iters": sum(its) / len(its),
                              "us_per_iter_per_rhs": el / sum(its) * 1e6}), flush=True)


if __name__ == "__main__":
    main()
