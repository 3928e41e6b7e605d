"""ctypes access to the oracle's C restatements (TEST INFRASTRUCTURE ONLY).

`oracle/c/csr_matvec.c` restates scipy's csr_matvec (the arithmetic behind
the reference's `LatticeOperator.apply`, lattice.py:214-217) with POSIX
threads over rows; it is the CPU baseline's matvec.  Built by `make -C oracle`
(called from `__graft_entry__.build()`)."""

import ctypes as ct
import os
import subprocess

import numpy as np

HERE = os.path.dirname(os.path.abspath(__file__))
LIB = os.path.join(HERE, "build", "liboracle.so")
_lib = None


def build():
    subprocess.run(["make", "-s", "-C", HERE], check=True)
    return LIB


def lib():
    global _lib
    if _lib is None:
        if not os.path.exists(LIB):
            build()
        h = ct.CDLL(LIB)
        h.oracle_threads.restype = ct.c_int
        h.oracle_csr_matvec_c128.restype = None
        h.oracle_csr_matvec_c128.argtypes = [ct.c_int64] + [ct.c_void_p] * 5 + [ct.c_int]
        _lib = h
    return _lib


def csr_matvec_callable(A):
    """(matvec, cores, description) for a scipy CSR matrix."""
    try:
        h = lib()
    except Exception:
        return (lambda x: A @ x), 1, "scipy csr_matvec, 1 thread"
    indptr = np.ascontiguousarray(A.indptr, dtype=np.int64)
    indices = np.ascontiguousarray(A.indices, dtype=np.int64)
    data = np.ascontiguousarray(A.data, dtype=np.complex128)
    n = A.shape[0]
    cores = int(h.oracle_threads())

    def mv(x):
        x = np.ascontiguousarray(x, dtype=np.complex128)
        y = np.empty(n, dtype=np.complex128)
        h.oracle_csr_matvec_c128(n, indptr.ctypes.data, indices.ctypes.data, data.ctypes.data,
                                 x.ctypes.data, y.ctypes.data, cores)
        return y

    return mv, cores, f"C/pthreads csr_matvec restatement, {cores} threads"
