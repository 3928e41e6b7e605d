"""Lattice geometry and the GPU Wilson-Dirac operator (host side).

Mirrors the reference's `mgtrace.lattice` interface
(`/root/reference/pkg/src/mgtrace/lattice.py`): `LatticeGeometry`
(`:44-103`), `build_lattice` (`:106-107`), `gamma5_pattern` (`:266-271`), the
`LatticeOperator` protocol (`:194-256`: `geometry`, `dof`, `dim`, `shape`,
`gamma5_diag`, `apply`, `apply_dagger`, `apply_gamma5`, `apply_shifted`,
`hermitian_form`, `a_gamma5`, `dense`) and `build_wilson` (`:274-318`) --
but for the 4D SU(3) Wilson-Dirac operator of BASELINE.json, applied by the
sm_100a stencil kernel behind the C ABI (`mgt_wilson_apply`).  There is no
sparse matrix: `.matrix` does not exist, and the reference functions that
reach into it are re-exported with GPU implementations instead
(SURVEY.md 8(b)).

Vectors at this interface use the reference layout (complex128, index
`site*12 + spin*3 + colour`, t fastest) and may be numpy arrays (host) or
CUDA tensors; the solver and estimators work on native-layout CUDA tensors
(shape (n, 12, V), t slowest) to avoid permutations in the hot loop.
"""

from dataclasses import dataclass

import numpy as np
import torch

from . import _lib
from ._device import complex_dtype, device, ptr, stream_ptr, to_device_c128

DOF = 12
DENSE_GUARD = 8192


class GeometryError(ValueError):
    pass


class SizeGuardError(ValueError):
    pass


@dataclass(frozen=True)
class LatticeGeometry:
    """Hypercubic lattice; `boundary='antiperiodic'` puts a -1 phase on the
    links wrapping in the LAST dimension (reference lattice.py:44-103)."""

    dims: tuple
    boundary: str = "periodic"

    def __post_init__(self):
        if len(self.dims) == 0:
            raise GeometryError("need at least one dimension")
        if any(int(L) < 2 for L in self.dims):
            raise GeometryError(f"extent < 2 in {tuple(self.dims)} is not a valid lattice")
        if self.boundary not in ("periodic", "antiperiodic"):
            raise GeometryError(f"unknown boundary {self.boundary!r}")
        object.__setattr__(self, "dims", tuple(int(L) for L in self.dims))

    @property
    def ndim(self):
        return len(self.dims)

    @property
    def site_count(self):
        return int(np.prod(self.dims))

    def site_index(self, coords):
        return int(np.ravel_multi_index(tuple(coords), self.dims))

    def site_coords(self, index):
        return tuple(int(c) for c in np.unravel_index(index, self.dims))

    def neighbor(self, index, mu, sign=+1):
        x = list(self.site_coords(index))
        x[mu] = (x[mu] + sign) % self.dims[mu]
        return self.site_index(x)


def build_lattice(dims, boundary="periodic"):
    return LatticeGeometry(tuple(dims), boundary)


def gamma5_pattern(site_count, dof=DOF):
    """+1 on the first dof/2 components of each site (DeGrand-Rossi gamma5 =
    diag(1,1,-1,-1) with comp = spin*3 + colour)."""
    if dof % 2:
        raise ValueError("gamma5 pattern needs an even number of components")
    return np.tile(np.concatenate([np.ones(dof // 2), -np.ones(dof // 2)]), site_count)


def _check4d(geometry):
    if geometry.ndim != 4:
        raise GeometryError("the B200 Wilson operator is 4D SU(3) (dims = (L0, L1, L2, T))")


class WilsonOperator:
    """GPU 4D SU(3) Wilson-Dirac operator A = (4+m0) I - 1/2 sum_mu [...]
    (reference protocol: lattice.py:194-263).  Immutable after construction;
    concurrent applies on different streams are safe."""

    def __init__(self, gauge, mass, prec=64, recon="auto"):
        geometry = gauge.geometry
        _check4d(geometry)
        if recon == "auto":
            # two-row storage + unitarity reconstruction is exact only for SU(3)
            recon = 12 if getattr(gauge, "kind", "") in ("su3", "unit") else 18
        self.geometry = geometry
        self.gauge = gauge
        self.mass = float(mass)
        self.dof = DOF
        self.prec = int(prec)
        self.recon = int(recon)
        self._gamma5 = None
        self._handle = _lib.ct.c_void_p()
        _lib.check(_lib.lib().mgt_wilson_create(
            _lib.ct.byref(self._handle), _lib.dims_arg(geometry.dims),
            1 if geometry.boundary == "antiperiodic" else 0, self.mass, self.prec, self.recon,
            ptr(gauge.links), stream_ptr()), "build_wilson")
        self._scratch = {}

    def __del__(self):
        h = getattr(self, "_handle", None)
        if h is not None and h.value:
            try:
                torch.cuda.synchronize()
                _lib.lib().mgt_wilson_destroy(h)
            except Exception:
                pass
            self._handle = None

    # -- protocol attributes ------------------------------------------------
    @property
    def handle(self):
        return self._handle

    @property
    def volume(self):
        return self.geometry.site_count

    @property
    def dim(self):
        return self.geometry.site_count * DOF

    @property
    def shape(self):
        return (self.dim, self.dim)

    @property
    def gamma5_diag(self):
        if self._gamma5 is None:
            self._gamma5 = gamma5_pattern(self.geometry.site_count)
        return self._gamma5

    @property
    def dtype(self):
        return complex_dtype(self.prec)

    # -- native-layout fields ---------------------------------------------
    def new_field(self, n=1, dtype=None):
        return torch.zeros((n, DOF, self.volume), dtype=dtype or self.dtype, device=device())

    def to_native(self, x_ref, out=None):
        """Reference layout (n, N) / (N,) complex128 CUDA tensor -> native (n, 12, V)."""
        x_ref = to_device_c128(x_ref)
        n = 1 if x_ref.dim() == 1 else x_ref.shape[0]
        if x_ref.numel() != n * self.dim:
            raise ValueError(f"dimension mismatch: {x_ref.numel() // n} != {self.dim}")
        out = self.new_field(n) if out is None else out
        _lib.check(_lib.lib().mgt_spinor_from_ref(_lib.dims_arg(self.geometry.dims), self.prec,
                                                   ptr(x_ref), ptr(out), n, stream_ptr()))
        return out

    def from_native(self, x_nat, out=None):
        n = x_nat.shape[0]
        out = torch.empty((n, self.dim), dtype=torch.complex128, device=x_nat.device) if out is None else out
        _lib.check(_lib.lib().mgt_spinor_to_ref(_lib.dims_arg(self.geometry.dims), self.prec,
                                                 ptr(x_nat), ptr(out), n, stream_ptr()))
        return out

    def apply_native(self, x, out=None, flags=0, tau=0.0):
        """out = variant(A) x on native fields (n, 12, V)."""
        if x.dim() != 3 or x.shape[1] != DOF or x.shape[2] != self.volume:
            raise ValueError(f"dimension mismatch: native field shape {tuple(x.shape)}")
        if x.dtype != self.dtype:
            raise ValueError(f"field dtype {x.dtype} != operator dtype {self.dtype}")
        x = x.contiguous()
        out = torch.empty_like(x) if out is None else out
        _lib.check(_lib.lib().mgt_wilson_apply(self._handle, ptr(x), ptr(out), x.shape[0], int(flags),
                                                float(tau), stream_ptr()), "apply")
        return out

    def apply_dot_native(self, x, u, out=None, flags=0, tau=0.0):
        """(out, d): out = variant(A) x and d[r] = vdot(u_r, out_r) from one
        fused pass (C ABI `mgt_wilson_apply_dot`, complex128 operators)."""
        if x.dim() != 3 or x.shape[1] != DOF or x.shape[2] != self.volume or u.shape != x.shape:
            raise ValueError(f"dimension mismatch: native field shapes {tuple(x.shape)}, {tuple(u.shape)}")
        if x.dtype != self.dtype or u.dtype != self.dtype:
            raise ValueError(f"field dtype {x.dtype} / {u.dtype} != operator dtype {self.dtype}")
        x, u = x.contiguous(), u.contiguous()
        out = torch.empty_like(x) if out is None else out
        d = torch.empty((x.shape[0], 2), dtype=torch.float64, device=x.device)
        _lib.check(_lib.lib().mgt_wilson_apply_dot(self._handle, ptr(x), ptr(out), ptr(u), x.shape[0], int(flags),
                                                    float(tau), ptr(d), stream_ptr()), "apply_dot")
        return out, torch.complex(d[:, 0], d[:, 1])

    def apply_interleaved(self, x, out=None, flags=0, tau=0.0):
        """out = variant(A) x on rhs-interleaved fields (12, V, n), n in
        {1, 2, 4, 8, 12}: the n rhs of a site share every link load (the
        multi-rhs form of a dilution / hierarchical-probing slot batch)."""
        if x.dim() != 3 or x.shape[0] != DOF or x.shape[1] != self.volume:
            raise ValueError(f"dimension mismatch: interleaved field shape {tuple(x.shape)}")
        if x.dtype != self.dtype:
            raise ValueError(f"field dtype {x.dtype} != operator dtype {self.dtype}")
        x = x.contiguous()
        out = torch.empty_like(x) if out is None else out
        _lib.check(_lib.lib().mgt_wilson_apply_il(self._handle, ptr(x), ptr(out), x.shape[2], int(flags),
                                                   float(tau), stream_ptr()), "apply_interleaved")
        return out

    def interleave(self, x, out=None):
        """native (n, 12, V) -> interleaved (12, V, n)."""
        n = x.shape[0]
        x = x.contiguous()
        out = torch.empty((DOF, self.volume, n), dtype=x.dtype, device=x.device) if out is None else out
        _lib.check(_lib.lib().mgt_rhs_interleave(self.volume, self.prec, n, 0, ptr(x), ptr(out), stream_ptr()),
                   "interleave")
        return out

    def deinterleave(self, x, out=None):
        """interleaved (12, V, n) -> native (n, 12, V)."""
        n = x.shape[2]
        x = x.contiguous()
        out = torch.empty((n, DOF, self.volume), dtype=x.dtype, device=x.device) if out is None else out
        _lib.check(_lib.lib().mgt_rhs_interleave(self.volume, self.prec, n, 1, ptr(x), ptr(out), stream_ptr()),
                   "deinterleave")
        return out

    # -- even-odd form (every extent even) ------------------------------
    def eo_split(self, x):
        """native (n, 12, V) -> (even, odd) parity fields (n, 12, V/2)."""
        x = x.contiguous()
        n = x.shape[0]
        e = torch.empty((n, DOF, self.volume // 2), dtype=x.dtype, device=x.device)
        o = torch.empty_like(e)
        _lib.check(_lib.lib().mgt_wilson_eo_split(self._handle, ptr(x), ptr(e), ptr(o), n, stream_ptr()), "eo split")
        return e, o

    def eo_merge(self, e, o):
        """(even, odd) parity fields -> native (n, 12, V)."""
        e, o = e.contiguous(), o.contiguous()
        n = e.shape[0]
        x = torch.empty((n, DOF, self.volume), dtype=e.dtype, device=e.device)
        _lib.check(_lib.lib().mgt_wilson_eo_merge(self._handle, ptr(e), ptr(o), ptr(x), n, stream_ptr()), "eo merge")
        return x

    def schur_apply(self, xe, flags=0, tau=0.0):
        """S x_e, the even-site Schur complement of the flags/tau variant."""
        xe = xe.contiguous()
        y = torch.empty_like(xe)
        _lib.check(_lib.lib().mgt_wilson_schur_apply(self._handle, ptr(xe), ptr(y), xe.shape[0], int(flags),
                                                     float(tau), stream_ptr()), "schur apply")
        return y

    # -- reference-layout API (lattice.py:214-247) ------------------------
    def apply_host(self, x, out=None, flags=0, tau=0.0, nchunks=64):
        """Host-memory reference-layout vector(s) (numpy or CPU tensor, (N,) or
        (n, N) rows) -> host result through the pipelined C-ABI path
        `mgt_wilson_apply_host` (PCIe copies overlapped with the layout
        permutation and the stencil).  Pinned CPU tensors overlap fully."""
        xt = x if isinstance(x, torch.Tensor) else torch.from_numpy(np.ascontiguousarray(x, dtype=np.complex128))
        if xt.dtype != torch.complex128:
            xt = xt.to(torch.complex128)
        xt = xt.contiguous()
        n = 1 if xt.dim() == 1 else xt.shape[0]
        if xt.numel() != n * self.dim:
            raise ValueError(f"dimension mismatch: {xt.shape[-1]} != {self.dim}")
        if out is None:
            out = torch.empty_like(xt, pin_memory=xt.is_pinned())
        _lib.check(_lib.lib().mgt_wilson_apply_host(self._handle, xt.data_ptr(), out.data_ptr(), n, int(flags),
                                                     float(tau), int(nchunks), stream_ptr()), "apply_host")
        return out if isinstance(x, torch.Tensor) else out.numpy()

    def _apply_ref(self, x, flags=0, tau=0.0):
        host = not isinstance(x, torch.Tensor)
        cpu_tensor = (not host) and x.device.type == "cpu"
        if (host or cpu_tensor) and np.ndim(x) == 1:
            return self.apply_host(x, flags=flags, tau=tau)
        xa = x
        if host:
            xa = np.asarray(x)
        if xa.shape[0] != self.dim:
            raise ValueError(f"dimension mismatch: {xa.shape[0]} != {self.dim}")
        two_d = xa.ndim == 2
        if two_d:
            xt = xa.T
        else:
            xt = xa[None, :] if host else xa.unsqueeze(0)
        xd = to_device_c128(np.ascontiguousarray(xt) if host else xt.contiguous())
        nat = self.to_native(xd)
        y = self.apply_native(nat, flags=flags, tau=tau)
        yr = self.from_native(y)
        if two_d:
            yr = yr.T
        else:
            yr = yr[0]
        if host:
            return yr.cpu().numpy()
        if cpu_tensor:
            out = torch.empty(yr.shape, dtype=yr.dtype, pin_memory=x.is_pinned())
            out.copy_(yr)
            return out
        return yr

    def apply(self, x):
        return self._apply_ref(x)

    def apply_dagger(self, x):
        return self._apply_ref(x, _lib.DAGGER)

    def apply_gamma5(self, x):
        g5 = self.gamma5_diag
        if isinstance(x, torch.Tensor):
            g = torch.as_tensor(g5, device=x.device, dtype=torch.float64)
            return g * x if x.dim() == 1 else g[:, None] * x
        x = np.asarray(x)
        return g5 * x if x.ndim == 1 else g5[:, None] * x

    def apply_shifted(self, tau, x):
        """(A + i tau gamma5) x; tau = 0 reduces to apply (lattice.py:229-233)."""
        return self._apply_ref(x, 0, float(tau))

    def hermitian_form(self):
        """gamma5 A (lattice.py:240-242) as an operator object."""
        return FormOperator(self, _lib.G5_OUT, 0.0, "gamma5 A")

    def a_gamma5(self):
        """A gamma5 (lattice.py:244-247) as an operator object."""
        return FormOperator(self, _lib.G5_IN, 0.0, "A gamma5")

    def shifted(self, tau):
        """A + i tau gamma5 as an operator object (eigen.py:140-151)."""
        return FormOperator(self, 0, float(tau), f"A + i{tau} gamma5")

    def dense(self):
        """Dense materialisation, guarded to N <= 8192 (lattice.py:249-256)."""
        if self.dim > DENSE_GUARD:
            raise SizeGuardError(f"refusing to densify N={self.dim} > {DENSE_GUARD}")
        eye = torch.eye(self.dim, dtype=torch.complex128, device=device())
        return self._apply_ref(eye).cpu().numpy()


class FormOperator:
    """A fixed flag/shift variant of a WilsonOperator with the protocol's
    apply/dim/geometry/gamma5_diag (what `krylov._as_matvec` accepts)."""

    def __init__(self, op, flags, tau, name):
        self.op = op
        self.flags = flags
        self.tau = tau
        self.name = name
        self.geometry = op.geometry
        self.dof = op.dof

    @property
    def dim(self):
        return self.op.dim

    @property
    def shape(self):
        return self.op.shape

    @property
    def gamma5_diag(self):
        return self.op.gamma5_diag

    def apply(self, x):
        return self.op._apply_ref(x, self.flags, self.tau)

    def apply_native(self, x, out=None):
        return self.op.apply_native(x, out=out, flags=self.flags, tau=self.tau)


def build_wilson(gauge, mass, prec=64, recon="auto"):
    """Assemble the GPU 4D Wilson operator (reference: lattice.py:274-318).
    recon 'auto': 12-real link storage for generated SU(3) fields, full 18
    reals for arbitrary user arrays."""
    return WilsonOperator(gauge, mass, prec=prec, recon=recon)
