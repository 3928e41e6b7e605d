#!/usr/bin/env python
"""A/B of the cp.async-staged plain apply (MGT_DSLASH_VARIANT=2,
csrc/dslash_pipe.cuh) against the register-staged kernel (variant 0):
bitwise comparison on small / ragged lattices and every flag variant, then
CUDA-event timings on the BASELINE configs[1] lattices."""
import argparse
import json
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)


def make(M, gauge, prec, recon, variant):
    os.environ["MGT_DSLASH_VARIANT"] = str(variant)
    op = M.build_wilson(gauge, 0.1, prec=prec, recon=recon)
    os.environ["MGT_DSLASH_VARIANT"] = "0"
    return op


def main():
    import torch
    import paper_1909_12234_b200 as M
    ap = argparse.ArgumentParser()
    ap.add_argument("--dims", default="24x24x24x24,32x32x32x32,48x48x48x96")
    ap.add_argument("--prec", default="64,32")
    ap.add_argument("--steps", type=int, default=20)
    ap.add_argument("--variants", default="0,2")
    ap.add_argument("--skip-check", action="store_true")
    args = ap.parse_args()
    torch.cuda.set_device(0)
    tag = os.environ.get("MGT_LIB_PATH", "in-tree")
    if not args.skip_check:
        for dims, bc in (((4, 4, 4, 8), "antiperiodic"), ((4, 6, 2, 10), "periodic"), ((6, 10, 6, 6), "antiperiodic"),
                         ((8, 8, 8, 8), "antiperiodic")):
            geo = M.LatticeGeometry(dims, bc)
            gauge = M.generate_gauge(geo, "su3", eps=0.3, seed=1)
            for prec in (64, 32):
                for recon in (12, 18):
                    a, b = make(M, gauge, prec, recon, 0), make(M, gauge, prec, recon, 2)
                    x = torch.randn((3, 12, geo.site_count), dtype=a.dtype, device="cuda")
                    for flags, tau in ((0, 0.0), (1, 0.0), (2, 0.0), (4, 0.3), (3, -0.7)):
                        ya = a.apply_native(x, flags=flags, tau=tau)
                        yb = b.apply_native(x, flags=flags, tau=tau)
                        if not torch.equal(ya, yb):
                            d = (ya - yb).abs().max().item() / ya.abs().max().item()
                            print(f"[{tag}] MISMATCH dims={dims} prec={prec} recon={recon} flags={flags} rel={d:.3e}")
                            if d > (1e-13 if prec == 64 else 1e-5):
                                sys.exit(1)
        print(f"[{tag}] check ok", flush=True)
    for dims_s in args.dims.split(","):
        dims = tuple(int(v) for v in dims_s.split("x"))
        geo = M.LatticeGeometry(dims, "antiperiodic")
        gauge = M.generate_gauge(geo, "su3", eps=0.2, seed=0)
        V = geo.site_count
        for prec in [int(p) for p in args.prec.split(",")]:
            ops = {v: make(M, gauge, prec, 12, int(v)) for v in args.variants.split(",")}
            x = torch.randn((1, 12, V), dtype=ops[args.variants.split(",")[0]].dtype, device="cuda")
            y = torch.empty_like(x)
            for rep in range(2):
                for v, op in ops.items():
                    for _ in range(3):
                        op.apply_native(x, out=y)
                    torch.cuda.synchronize()
                    e0, e1 = torch.cuda.Event(True), torch.cuda.Event(True)
                    e0.record()
                    for _ in range(args.steps):
                        op.apply_native(x, out=y)
                    e1.record()
                    torch.cuda.synchronize()
                    ms = e0.elapsed_time(e1) / args.steps
                    w = 8 if prec == 64 else 4
                    print(json.dumps({"lib": tag, "dims": dims_s, "prec": prec, "variant": int(v), "rep": rep,
                                      "us": round(ms * 1e3, 1), "GBps": round(V * 120 * w / ms / 1e6)}), flush=True)
            del ops, x, y
            torch.cuda.empty_cache()
        del gauge
        torch.cuda.empty_cache()


if __name__ == "__main__":
    main()
