#!/usr/bin/env python
"""Coarse apply at the BASELINE configs[4] size (8192 aggregates, nc = 48):
time per call for 8 rhs (fp64 / fp32 C) -- random C of the right shape."""
import os
import sys
import time

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import torch  # noqa: E402

from paper_1909_12234_b200 import _lib  # noqa: E402
from paper_1909_12234_b200._device import ptr, stream_ptr  # noqa: E402

dims, block, nv = (32, 32, 32, 64), (4, 4, 4, 4), 24
nb, nc = 8 * 8 * 8 * 16, 48
C = torch.randn(nb * 9 * nc * nc, dtype=torch.complex128, device="cuda")
C32 = C.to(torch.complex64)
d = _lib.dims_arg(dims)
b = _lib.dims_arg(block)
for n in (1, 4, 8):
    x = torch.randn((n, nb, nc), dtype=torch.complex128, device="cuda")
    y = torch.empty_like(x)
    for name, fn in [("fp64", lambda: _lib.lib().mgt_coarse_apply(d, b, nv, ptr(C), ptr(x), ptr(y), n, stream_ptr())),
                     ("fp32", lambda: _lib.lib().mgt_coarse_apply_c32(d, b, nv, ptr(C32), ptr(x), ptr(y), n,
                                                                      stream_ptr()))]:
        for _ in range(3):
            fn()
        torch.cuda.synchronize()
        t0 = time.perf_counter()
        for _ in range(20):
            fn()
        torch.cuda.synchronize()
        el = (time.perf_counter() - t0) / 20
        cb = C.numel() * (16 if name == "fp64" else 8)
        print(f"n={n} {name}: {el * 1e6:8.1f} us  C stream {cb / el / 1e9:7.1f} GB/s", flush=True)
