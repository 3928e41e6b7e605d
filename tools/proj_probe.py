#!/usr/bin/env python
"""V^H X and X - V H timings at 16^4 (len 786,432) for the Davidson / CGS2
shapes: k in {64, 144} vectors against s in {1, 2, 4, 8, 16} columns (CUDA
events, HBM-fraction of the 16 N (k + s) byte model)."""
import json
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)


def main():
    import torch
    from paper_1909_12234_b200 import linalg as LA
    from tools.kernel_rooflines import timeit
    peak = json.load(open(os.path.join(ROOT, "MEASURED_PEAKS.json")))["hbm_gbs"]
    n = 12 * 16 ** 4
    for k in (64, 144):
        V = torch.randn((k, n), dtype=torch.complex128, device="cuda")
        for s in ((1, 2, 4, 8, 16, 32, 128) if k == 64 else (1, 8, 16)):
            X = torch.randn((s, n), dtype=torch.complex128, device="cuda")
            t = timeit(lambda: LA.vhx(V, X), steps=20)
            b = 16 * n * (k + s)
            H = LA.vhx(V, X)
            ref = V.conj() @ X.T
            err = ((H - ref).abs().max() / ref.abs().max()).item()
            print(json.dumps({"op": "vhx", "k": k, "s": s, "us": t * 1e6, "GBps": b / t / 1e9,
                              "frac": b / t / 1e9 / peak, "rel_err": err}), flush=True)
            Vc = V.conj()
            t = timeit(lambda: Vc @ X.T, steps=20)
            print(json.dumps({"op": "cublas_zgemm", "k": k, "s": s, "us": t * 1e6, "GBps": b / t / 1e9,
                              "frac": b / t / 1e9 / peak}), flush=True)
            del Vc
            if s > 8:
                t = timeit(lambda: [LA.vhx(V, X[j:j + 8]) for j in range(0, s, 8)], steps=20)
                print(json.dumps({"op": "vhx_8col_chunks", "k": k, "s": s, "us": t * 1e6, "GBps": b / t / 1e9,
                                  "frac": b / t / 1e9 / peak}), flush=True)
            Hs = H.contiguous()
            X2 = X.clone()
            t = timeit(lambda: LA.sub_vh(V, Hs, X2), steps=20)
            b2 = 16 * n * (k + 2 * s)
            print(json.dumps({"op": "sub_vh", "k": k, "s": s, "us": t * 1e6, "GBps": b2 / t / 1e9,
                              "frac": b2 / t / 1e9 / peak}), flush=True)
            del X2
            del X
        del V
        torch.cuda.empty_cache()


if __name__ == "__main__":
    main()
