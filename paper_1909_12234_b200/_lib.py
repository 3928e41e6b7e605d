"""ctypes binding of the C ABI declared in `include/mgtrace_b200.h`.

The native library is REQUIRED: there is no CPU fallback.  Importing the
product on a machine where `libmgtrace_b200.so` is missing raises at the
first call that needs it (the build runs in `__graft_entry__.build()`).
"""

import ctypes as ct
import os
import threading

_PKG = os.path.dirname(os.path.abspath(__file__))
# MGT_LIB_PATH: load another build of the same library (A/B timing runs)
LIB_PATH = os.environ.get("MGT_LIB_PATH") or os.path.join(_PKG, "libmgtrace_b200.so")

MGT_OK = 0
MGT_ERR_INVALID = 1
MGT_ERR_CUDA = 2
MGT_ERR_SIZE = 3
MGT_ERR_BLOCKING = 4

G5_IN = 1
G5_OUT = 2
DAGGER = 4
HALO_PEER = 8
SOLVE_FULL = 16
SOLVE_MIXED = 32
IPC_HANDLE_BYTES = 64

_lock = threading.Lock()
_lib = None

c_int_p = ct.POINTER(ct.c_int)
c_i64_p = ct.POINTER(ct.c_int64)
c_dbl_p = ct.POINTER(ct.c_double)
c_u64_p = ct.POINTER(ct.c_uint64)
vp = ct.c_void_p

_SIGNATURES = {
    "mgt_last_error": (ct.c_char_p, []),
    "mgt_version": (ct.c_int, []),
    "mgt_launch_count": (ct.c_uint64, []),
    "mgt_spinor_from_ref": (ct.c_int, [c_int_p, ct.c_int, vp, vp, ct.c_int, vp]),
    "mgt_spinor_to_ref": (ct.c_int, [c_int_p, ct.c_int, vp, vp, ct.c_int, vp]),
    "mgt_su3_expm": (ct.c_int, [ct.c_double, vp, ct.c_int64, ct.c_int64, vp, vp]),
    "mgt_wilson_create": (ct.c_int, [ct.POINTER(vp), c_int_p, ct.c_int, ct.c_double, ct.c_int, ct.c_int, vp, vp]),
    "mgt_wilson_destroy": (ct.c_int, [vp]),
    "mgt_wilson_info": (ct.c_int, [vp, c_int_p, c_int_p, c_int_p, c_i64_p]),
    "mgt_wilson_apply": (ct.c_int, [vp, vp, vp, ct.c_int, ct.c_int, ct.c_double, vp]),
    "mgt_wilson_apply_il": (ct.c_int, [vp, vp, vp, ct.c_int, ct.c_int, ct.c_double, vp]),
    "mgt_rhs_interleave": (ct.c_int, [ct.c_int64, ct.c_int, ct.c_int, ct.c_int, vp, vp, vp]),
    "mgt_wilson_eo_split": (ct.c_int, [vp, vp, vp, vp, ct.c_int, vp]),
    "mgt_wilson_eo_merge": (ct.c_int, [vp, vp, vp, vp, ct.c_int, vp]),
    "mgt_wilson_schur_apply": (ct.c_int, [vp, vp, vp, ct.c_int, ct.c_int, ct.c_double, vp]),
    "mgt_comm_unique_id": (ct.c_int, [vp]),
    "mgt_comm_create": (ct.c_int, [ct.POINTER(ct.c_void_p), vp, ct.c_int, ct.c_int]),
    "mgt_comm_destroy": (ct.c_int, [vp]),
    "mgt_comm_allreduce": (ct.c_int, [vp, vp, ct.c_int64, vp]),
    "mgt_bicgstab_slab_workspace_bytes": (ct.c_size_t, [vp, ct.c_int]),
    "mgt_bicgstab_solve_slab": (ct.c_int, [vp, vp, vp, vp, ct.c_int, ct.c_int, ct.c_double, ct.c_double, ct.c_int,
                                           vp, c_i64_p, c_dbl_p, c_dbl_p, vp]),
    "mgt_ipc_alloc": (ct.c_int, [ct.c_size_t, ct.POINTER(ct.c_void_p), vp]),
    "mgt_ipc_free": (ct.c_int, [vp]),
    "mgt_ipc_open": (ct.c_int, [vp, ct.POINTER(ct.c_void_p)]),
    "mgt_ipc_close": (ct.c_int, [vp]),
    "mgt_wilson_apply_host": (ct.c_int, [vp, vp, vp, ct.c_int, ct.c_int, ct.c_double, ct.c_int, vp]),
    "mgt_wilson_create_slab": (ct.c_int, [ct.POINTER(vp), c_int_p, ct.c_int, ct.c_int, ct.c_int, ct.c_double,
                                          ct.c_int, ct.c_int, vp, vp]),
    "mgt_halo_pack": (ct.c_int, [vp, vp, vp, vp, ct.c_int, ct.c_int, ct.c_double, vp]),
    "mgt_wilson_apply_slab": (ct.c_int, [vp, vp, vp, vp, vp, ct.c_int, ct.c_int, ct.c_double, ct.c_int, vp]),
    "mgt_cdot": (ct.c_int, [vp, vp, ct.c_int64, ct.c_int, vp, vp]),
    "mgt_bicgstab_workspace_bytes": (ct.c_size_t, [vp, ct.c_int]),
    "mgt_bicgstab_solve": (ct.c_int, [vp, vp, vp, ct.c_int, ct.c_int, ct.c_double, ct.c_double, ct.c_int,
                                      vp, c_i64_p, c_dbl_p, c_dbl_p, vp]),
    "mgt_bicgstab_solve_ws": (ct.c_int, [vp, vp, vp, ct.c_int, ct.c_int, ct.c_double, ct.c_double, ct.c_int,
                                         vp, ct.c_size_t, c_i64_p, c_dbl_p, c_dbl_p, vp]),
    "mgt_bicgstab_solve_tols": (ct.c_int, [vp, vp, vp, ct.c_int, ct.c_int, ct.c_double, c_dbl_p, ct.c_int,
                                           vp, ct.c_size_t, c_i64_p, c_dbl_p, c_dbl_p, vp]),
    "mgt_gcr_workspace_bytes": (ct.c_size_t, [vp, ct.c_int]),
    "mgt_gcr_solve": (ct.c_int, [vp, vp, vp, ct.c_int, ct.c_int, ct.c_double, vp, c_i64_p, c_dbl_p, vp]),
    "mgt_wilson_apply_dot": (ct.c_int, [vp, vp, vp, vp, ct.c_int, ct.c_int, ct.c_double, vp, vp]),
    "mgt_gmres_workspace_bytes": (ct.c_size_t, [vp, ct.c_int]),
    "mgt_gmres_solve": (ct.c_int, [vp, vp, vp, ct.c_int, ct.c_int, ct.c_double, ct.c_int, ct.c_double, vp, c_i64_p,
                                   c_dbl_p, vp]),
    "mgt_noise": (ct.c_int, [c_int_p, ct.c_int, c_u64_p, ct.c_int, ct.c_int, vp, vp]),
    "mgt_noise_slab": (ct.c_int, [c_int_p, ct.c_int, ct.c_int, ct.c_int, c_u64_p, ct.c_int, vp, vp]),
    "mgt_prolong_build": (ct.c_int, [c_int_p, c_int_p, ct.c_int, vp, vp, c_int_p, vp]),
    "mgt_prolong": (ct.c_int, [c_int_p, c_int_p, ct.c_int, vp, vp, vp, ct.c_int, vp]),
    "mgt_restrict": (ct.c_int, [c_int_p, c_int_p, ct.c_int, vp, vp, vp, ct.c_int, ct.c_int, vp]),
    "mgt_coarse_perm": (ct.c_int, [c_int_p, c_int_p, ct.c_int, ct.c_int, vp, vp, ct.c_int, vp]),
    "mgt_coarse_build": (ct.c_int, [vp, c_int_p, ct.c_int, vp, vp, vp]),
    "mgt_coarse_apply": (ct.c_int, [c_int_p, c_int_p, ct.c_int, vp, vp, vp, ct.c_int, vp]),
    "mgt_coarse_apply_c32": (ct.c_int, [c_int_p, c_int_p, ct.c_int, vp, vp, vp, ct.c_int, vp]),
    "mgt_coarse_bicgstab_iter": (ct.c_int, [c_int_p, c_int_p, ct.c_int, vp, ct.c_int, ct.c_double, ct.c_int, vp, vp,
                                            vp, vp, vp, vp, vp, vp, vp]),
    "mgt_coarse_half_apply": (ct.c_int, [c_int_p, c_int_p, ct.c_int, vp, ct.c_int, ct.c_int, ct.c_int, ct.c_int,
                                         vp, vp, vp, ct.c_int, vp]),
    "mgt_coarse_schur_apply": (ct.c_int, [c_int_p, c_int_p, ct.c_int, vp, vp, ct.c_int, vp, vp, vp, ct.c_int, vp]),
    "mgt_coarse_schur_bicgstab": (ct.c_int, [c_int_p, c_int_p, ct.c_int, vp, vp, ct.c_int, ct.c_int, ct.c_int, vp, vp,
                                             vp, vp, vp, vp, vp, vp, vp, vp]),
    "mgt_proj_vhx": (ct.c_int, [vp, vp, ct.c_int64, ct.c_int, ct.c_int, vp, vp]),
    "mgt_proj_sub": (ct.c_int, [vp, vp, vp, ct.c_int64, ct.c_int, ct.c_int, vp]),
}


class NativeLibraryError(RuntimeError):
    pass


def lib():
    """The loaded native library (loaded once; raises if absent)."""
    global _lib
    if _lib is not None:
        return _lib
    with _lock:
        if _lib is None:
            if not os.path.exists(LIB_PATH):
                raise NativeLibraryError(
                    f"native library {LIB_PATH} is missing; run __graft_entry__.build() "
                    "(there is no CPU fallback)")
            h = ct.CDLL(LIB_PATH)
            for name, (res, args) in _SIGNATURES.items():
                fn = getattr(h, name, None)
                if fn is None:
                    continue
                fn.restype = res
                fn.argtypes = args
            _lib = h
    return _lib


def exported_symbols():
    return list(_SIGNATURES)


def check(code, what=""):
    """Map C-ABI status codes onto the reference's exception families."""
    if code == MGT_OK:
        return
    msg = lib().mgt_last_error().decode(errors="replace")
    if what:
        msg = f"{what}: {msg}"
    if code in (MGT_ERR_INVALID, MGT_ERR_SIZE):
        raise ValueError(msg)
    if code == MGT_ERR_BLOCKING:
        from .multigrid import BlockingError
        raise BlockingError(msg)
    raise RuntimeError(msg)


def dims_arg(dims):
    return (ct.c_int * 4)(*[int(d) for d in dims])


def launch_count():
    return int(lib().mgt_launch_count())
