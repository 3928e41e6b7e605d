"""Tall-skinny projections on device fields (C ABI `mgt_proj_vhx` /
`mgt_proj_sub`): the deflation projection X - V (V^H X) of trace.py:182-183,
:266-267 and the CGS2 of eigen.py:79-86.  Fields are complex128 CUDA tensors
whose leading dimension indexes vectors ((k, 12, V) native fields or (k, n))."""

import torch

from . import _lib
from ._device import ptr, stream_ptr


def _flat(t):
    t = t.contiguous()
    return t, t.reshape(t.shape[0], -1).shape[1]


# From this many columns (with more than 8 vectors) V^H X is a plain
# GEMM: cuBLAS ZGEMM on the FP64 tensor cores (DMMA: fp64 products, so the
# fp64 tolerance holds) beats the FP64-pipe tile kernel 1.6-2.8x
# (tools/proj_probe.py: k = 64, s = 32 / 128: 0.82 vs 1.35 ms, 1.74 vs
# 4.82 ms); below it the projection kernels win (s <= 16: they stream V at
# up to 70 % of HBM).
GEMM_MIN_COLS = 32


def vhx(V, X, gemm=None):
    """H = V^H X, shape (k, s).  gemm: None = by shape (cuBLAS for k > 8,
    s >= GEMM_MIN_COLS), False = always the projection kernels (C ABI)."""
    V, n = _flat(V)
    X, n2 = _flat(X)
    if n != n2:
        raise ValueError(f"dimension mismatch: {n} != {n2}")
    k, s = V.shape[0], X.shape[0]
    if gemm is None:
        gemm = k > 8 and s >= GEMM_MIN_COLS
    if gemm:
        return V.reshape(k, n).conj() @ X.reshape(s, n).transpose(0, 1)
    H = torch.empty((s, k), dtype=torch.complex128, device=V.device)  # column major k x s
    _lib.check(_lib.lib().mgt_proj_vhx(ptr(V), ptr(X), n, k, s, ptr(H), stream_ptr()), "proj_vhx")
    return H.transpose(0, 1)


def sub_vh(V, H, X):
    """In place X <- X - V H (X contiguous); H (k, s)."""
    V, n = _flat(V)
    k, s = H.shape
    Hc = H.transpose(0, 1).contiguous()  # column-major k x s
    if not X.is_contiguous():
        raise ValueError("X must be contiguous")
    _lib.check(_lib.lib().mgt_proj_sub(ptr(V), ptr(Hc), ptr(X), n, k, s, stream_ptr()), "proj_sub")
    return X


def project_out(V, X):
    """X <- X - V (V^H X) in place; returns V^H X."""
    H = vhx(V, X)
    sub_vh(V, H, X)
    return H


def cgs2(v, bases):
    """v orthogonalised against each basis in turn, twice (eigen.py:79-86)."""
    for _ in range(2):
        for B in bases:
            if B is None or B.shape[0] == 0:
                continue
            project_out(B, v)
    return v
