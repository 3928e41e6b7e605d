#!/usr/bin/env python
"""BASELINE.json configs[1] sweep: Dslash / Dslash.gamma5 matvec GB/s on
16^4, 24^4, 32^4, 48^3x96 in complex128 and complex64, eps in {0.2, 0.5},
link storage 18 (full) or 12 (two rows + reconstruction), n_rhs 1 or 4.
Prints one JSON line per case (CUDA-event timing, inputs > L2 except 16^4)."""

import argparse
import json
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)


def main():
    import torch
    import paper_1909_12234_b200 as M
    ap = argparse.ArgumentParser()
    ap.add_argument("--dims", default="16x16x16x16,24x24x24x24,32x32x32x32,48x48x48x96")
    ap.add_argument("--prec", default="64,32")
    ap.add_argument("--recon", default="18,12")
    ap.add_argument("--eps", default="0.2")
    ap.add_argument("--nrhs", default="1")
    ap.add_argument("--flags", default="0")
    ap.add_argument("--steps", type=int, default=20)
    ap.add_argument("--layout", default="native", help="native or il (rhs-interleaved)")
    args = ap.parse_args()
    torch.cuda.set_device(0)
    for dims_s in args.dims.split(","):
        dims = tuple(int(v) for v in dims_s.split("x"))
        for eps in [float(e) for e in args.eps.split(",")]:
            geo = M.LatticeGeometry(dims, "antiperiodic")
            gauge = M.generate_gauge(geo, "su3", eps=eps, seed=0)
            for prec in [int(p) for p in args.prec.split(",")]:
                for recon in [int(r) for r in args.recon.split(",")]:
                    op = M.build_wilson(gauge, 0.1, prec=prec, recon=recon)
                    for nrhs in [int(n) for n in args.nrhs.split(",")]:
                        for flags in [int(f) for f in args.flags.split(",")]:
                            V = geo.site_count
                            il = args.layout == "il"
                            shape = (12, V, nrhs) if il else (nrhs, 12, V)
                            x = torch.randn(shape, dtype=op.dtype, device="cuda")
                            y = torch.empty_like(x)
                            fn = op.apply_interleaved if il else op.apply_native
                            for _ in range(3):
                                fn(x, out=y, flags=flags)
                            torch.cuda.synchronize()
                            e0, e1 = torch.cuda.Event(True), torch.cuda.Event(True)
                            e0.record()
                            for _ in range(args.steps):
                                fn(x, out=y, flags=flags)
                            e1.record()
                            torch.cuda.synchronize()
                            ms = e0.elapsed_time(e1) / args.steps
                            w = 8 if prec == 64 else 4
                            alg = V * (4 * 18 * w + nrhs * 48 * w)
                            print(json.dumps({"dims": dims_s, "eps": eps, "prec": prec, "recon": recon,
                                              "n_rhs": nrhs, "layout": args.layout, "flags": flags, "ms": ms,
                                              "GBps": alg / ms / 1e6,
                                              "Gsites_rhs_per_s": V * nrhs / ms / 1e6}), flush=True)
                            del x, y
                    del op
                    torch.cuda.empty_cache()
            del gauge
            torch.cuda.empty_cache()


if __name__ == "__main__":
    main()
