"""Device plumbing: torch owns device memory and streams; the native library
only sees raw pointers (C ABI)."""

import numpy as np
import torch


def require_cuda():
    if not torch.cuda.is_available():
        raise RuntimeError("mgtrace-b200 needs a CUDA device (sm_100a); there is no CPU fallback")


def device():
    require_cuda()
    return torch.device("cuda", torch.cuda.current_device())


def stream_ptr(stream=None):
    s = stream if stream is not None else torch.cuda.current_stream()
    return s.cuda_stream


def ptr(t):
    return t.data_ptr() if t is not None else None


def to_device_c128(x):
    """numpy / torch -> contiguous complex128 CUDA tensor (no copy if already)."""
    if isinstance(x, torch.Tensor):
        t = x
        if t.dtype != torch.complex128:
            t = t.to(torch.complex128)
        if t.device.type != "cuda":
            t = t.to(device(), non_blocking=True)
        return t.contiguous()
    arr = np.ascontiguousarray(np.asarray(x, dtype=np.complex128))
    return torch.from_numpy(arr).to(device(), non_blocking=False)


def complex_dtype(prec):
    return torch.complex128 if prec == 64 else torch.complex64
