"""GPU multigrid setup: null vectors, chirality-split prolongator P / P^H,
Galerkin coarse operator and its block-stencil matvec.

Mirrors `mgtrace.multigrid` (`/root/reference/pkg/src/mgtrace/multigrid.py`):
`BlockingError` (`:24`), `BlockingScheme` (`:28-57`), `NullVectors`
(`:60-71`), `generate_null_vectors` (`:74-113`), `Prolongator`
(`:116-160`), `build_prolongator` (`:163-225`), `CoarseOperator`
(`:228-243`), `build_coarse_operator` (`:246-259`).  P, P^H, the MGS
orthonormalisation and C = P^H A P are sm_100a kernels (`mgt_prolong_build`,
`mgt_prolong`, `mgt_restrict`, `mgt_coarse_build`, `mgt_coarse_apply`).

Null vectors follow the reference exactly: one `default_rng(seed)` stream,
`y0 = normal(N) + 1j normal(N)` per vector in reference layout, relaxed by
restarted GCR(max_iter, restart = max_iter) on A d = -A y0 from a zero start
(`gcr_relax`, GPU dslash; the GCR scalar recurrences follow krylov.py:52-118,
the short BLAS-1 on torch device tensors), y = y0 + d, normalised.
"""

import warnings
from dataclasses import dataclass

import numpy as np
import torch

from . import _lib
from ._device import device, ptr, stream_ptr
from .lattice import LatticeGeometry


class BlockingError(ValueError):
    pass


@dataclass(frozen=True)
class BlockingScheme:
    block_dims: tuple

    def __post_init__(self):
        object.__setattr__(self, "block_dims", tuple(int(b) for b in self.block_dims))
        if any(b < 1 for b in self.block_dims):
            raise BlockingError("block extents must be >= 1")

    def validate(self, geometry):
        if len(self.block_dims) != geometry.ndim:
            raise BlockingError("blocking dimensionality mismatch")
        for L, b in zip(geometry.dims, self.block_dims):
            if L % b:
                raise BlockingError(f"block extent {b} does not divide lattice extent {L}")

    def coarse_dims(self, geometry):
        return tuple(L // b for L, b in zip(geometry.dims, self.block_dims))

    def block_count(self, geometry):
        return int(np.prod(self.coarse_dims(geometry)))


# ---------------------------------------------------------------------------
# GCR relaxation on the GPU (krylov.py:52-118 semantics)


_GCR_WS = {}


def gcr_relax(op, b, tol, max_iter, restart):
    """Restarted GCR from x0 = 0 (C ABI `mgt_gcr_solve`, krylov.py:52-118
    semantics) on a native field (1, 12, V); returns
    (x, iterations, converged, reason, matvecs)."""
    import ctypes as ct
    key = (id(op), restart)
    ws = _GCR_WS.get(key)
    if ws is None or ws[0] is not op:
        nbytes = _lib.lib().mgt_gcr_workspace_bytes(op.handle, int(restart))
        ws = (op, torch.empty(int(nbytes), dtype=torch.uint8, device=device()))
        _GCR_WS[key] = ws
    x = torch.empty_like(b)
    rep = (ct.c_int64 * 4)()
    rel = (ct.c_double * 1)()
    _lib.check(_lib.lib().mgt_gcr_solve(op.handle, ptr(b.contiguous()), ptr(x), int(restart), int(max_iter),
                                         float(tol), ptr(ws[1]), rep, rel, stream_ptr()), "gcr")
    it, mv, conv, reason = (int(v) for v in rep)
    return x, it, bool(conv), ("" if conv else ("breakdown" if reason == 2 else "max_iter")), mv


@dataclass
class NullVectors:
    vectors: torch.Tensor  # (n, 12, V) native layout
    residual_ratios: np.ndarray
    seed: int
    geometry: LatticeGeometry
    dof: int
    gamma5_diag: np.ndarray
    degenerate: np.ndarray = None

    def ref_vectors(self, op):
        """(n, N) reference-layout numpy copy."""
        return op.from_native(self.vectors).cpu().numpy()


def generate_null_vectors(op, n, tol=1e-2, max_iter=200, seed=0):
    """Reference generate_null_vectors (multigrid.py:74-113) on the GPU."""
    if n < 1:
        raise ValueError("need n >= 1 null vectors")
    rng = np.random.default_rng(seed)
    N = op.dim
    # the start y0 = normal(N) + 1j normal(N) of the reference: the same
    # stream and values as rng.normal (loc 0, scale 1), replayed by parallel
    # host threads (rng.NormalStream, bitwise equal; the next vector's draws
    # are decoded while this one relaxes on the GPU) into pinned buffers and
    # combined on the device
    #
    # A producer thread decodes draw pair k + 1 (and k + 2) into spare pinned
    # buffers while vector k relaxes on the GPU: the host stream and the GPU
    # relaxation overlap (32^3 x 64: 57 + 45 ms per vector sequentially).
    import queue
    import threading

    from .rng import NormalStream
    normals = NormalStream(rng)
    free, full = queue.Queue(), queue.Queue()
    for _ in range(2):
        free.put((torch.empty(N, dtype=torch.float64).pin_memory(), torch.empty(N, dtype=torch.float64).pin_memory()))
    stop = threading.Event()

    def produce():
        try:
            while not stop.is_set():
                try:
                    bufs = free.get(timeout=0.05)
                except queue.Empty:
                    continue
                normals.take(N, out=bufs[0].numpy())
                normals.take(N, out=bufs[1].numpy())
                full.put(bufs)
        except BaseException as e:  # surfaced by the consumer
            full.put(e)

    producer = threading.Thread(target=produce, name="mgt-nullvec-draws", daemon=True)
    producer.start()

    def next_start():
        bufs = full.get()
        if isinstance(bufs, BaseException):
            raise bufs
        y0 = op.to_native(torch.complex(bufs[0].to(device(), non_blocking=True),
                                        bufs[1].to(device(), non_blocking=True)))
        ev = torch.cuda.Event()
        ev.record()
        ev.synchronize()  # the copies out of the pinned pair are done: hand it back
        free.put(bufs)
        return y0

    try:
        return _relax_null_vectors(op, n, tol, max_iter, seed, next_start)
    finally:
        stop.set()
        producer.join()


def _relax_null_vectors(op, n, tol, max_iter, seed, next_start):
    """The relaxation loop of generate_null_vectors (multigrid.py:83-113):
    next_start() yields the successive Gaussian starts y0."""
    vecs = op.new_field(n)
    ratios = np.empty(n)
    degenerate = np.zeros(n, dtype=bool)
    for i in range(n):
        for attempt in range(3):
            y0 = next_start()
            b = -op.apply_native(y0)
            d, its, conv, why, _ = gcr_relax(op, b, tol, max_iter, max_iter)
            y = y0 + d
            if conv or why != "breakdown":
                break
        else:
            raise RuntimeError(f"null-vector solve kept breaking down (vector {i})")
        yn = torch.linalg.vector_norm(y).item()
        y0n = torch.linalg.vector_norm(y0).item()
        if yn < 1e-8 * y0n:
            degenerate[i] = True
            d1, *_ = gcr_relax(op, b, tol, 1, 1)
            y = y0 + d1
            yn = torch.linalg.vector_norm(y).item()
            if yn < 1e-8 * y0n:
                y, yn = y0, y0n
        ratios[i] = torch.linalg.vector_norm(op.apply_native(y)).item() / max(
            torch.linalg.vector_norm(b).item(), 1e-300)
        vecs[i] = (y / yn)[0]
    return NullVectors(vecs, ratios, seed, op.geometry, op.dof, op.gamma5_diag, degenerate)


def null_vectors_from_array(op, vectors_ref, seed=0):
    """Wrap host reference-layout vectors (n, N) (e.g. the reference's own
    output) as NullVectors on the device."""
    v = torch.as_tensor(np.ascontiguousarray(vectors_ref, dtype=np.complex128)).to(device())
    return NullVectors(op.to_native(v), np.zeros(len(vectors_ref)), seed, op.geometry, op.dof,
                       op.gamma5_diag, np.zeros(len(vectors_ref), dtype=bool))


# ---------------------------------------------------------------------------


class Prolongator:
    """Block-orthonormal chirality-preserving basis V on the device
    (multigrid.py:116-160).  Coarse vectors use the reference order at the
    `restrict` / `prolong` interface and the native order (t slowest) in the
    `*_native` methods."""

    def __init__(self, P, geometry, blocking, nv, fine_dof, keep):
        self.P = P
        self.geometry = geometry
        self.blocking = blocking
        self.nv = nv
        self.fine_dof = fine_dof
        m = blocking.block_count(geometry)
        keep = keep.reshape(m, 2, nv)
        self.per_block_counts = keep.sum(axis=2)
        self.dropped = int(keep.size - keep.sum())
        self.coarse_gamma5 = np.tile(np.concatenate([np.ones(nv), -np.ones(nv)]), m)
        self.keep = np.asarray(keep).reshape(-1).astype(np.int32)

    @property
    def uniform(self):
        return bool(np.all(self.per_block_counts == self.per_block_counts[0, 0]))

    @property
    def n_blocks(self):
        return self.blocking.block_count(self.geometry)

    @property
    def nc(self):
        return 2 * self.nv

    @property
    def fine_dim(self):
        return self.geometry.site_count * self.fine_dof

    @property
    def coarse_dim(self):
        return self.n_blocks * self.nc

    @property
    def coarse_geometry(self):
        return LatticeGeometry(self.blocking.coarse_dims(self.geometry), self.geometry.boundary)

    def _dims(self):
        return _lib.dims_arg(self.geometry.dims), _lib.dims_arg(self.blocking.block_dims)

    def new_coarse(self, n=1):
        return torch.zeros((n, self.n_blocks, self.nc), dtype=torch.complex128, device=device())

    def coarse_to_ref(self, xc):
        out = torch.empty_like(xc)
        d, b = self._dims()
        _lib.check(_lib.lib().mgt_coarse_perm(d, b, self.nc, xc.shape[0], ptr(xc), ptr(out), 1, stream_ptr()))
        return out

    def coarse_from_ref(self, xc):
        out = torch.empty_like(xc)
        d, b = self._dims()
        _lib.check(_lib.lib().mgt_coarse_perm(d, b, self.nc, xc.shape[0], ptr(xc), ptr(out), 0, stream_ptr()))
        return out

    def restrict_native(self, x, gamma5_in=False, out=None):
        """P^H x (or P^H gamma5 x) for native fine fields (n, 12, V) ->
        native coarse (n, nb, 2nv)."""
        x = x.contiguous()
        out = self.new_coarse(x.shape[0]) if out is None else out
        d, b = self._dims()
        _lib.check(_lib.lib().mgt_restrict(d, b, self.nv, ptr(self.P), ptr(x), ptr(out), x.shape[0],
                                            1 if gamma5_in else 0, stream_ptr()), "restrict")
        return out

    def prolong_native(self, xc, out=None):
        xc = xc.contiguous()
        n = xc.shape[0]
        out = torch.empty((n, 12, self.geometry.site_count), dtype=torch.complex128,
                          device=device()) if out is None else out
        d, b = self._dims()
        _lib.check(_lib.lib().mgt_prolong(d, b, self.nv, ptr(self.P), ptr(xc), ptr(out), n, stream_ptr()),
                   "prolong")
        return out

    # reference-layout interface (multigrid.py:153-157)
    def restrict(self, x):
        host = not isinstance(x, torch.Tensor)
        xd = torch.as_tensor(np.asarray(x, dtype=np.complex128)).to(device()) if host else x
        nat = self._layout.to_native(xd.reshape(1, -1))
        xc = self.coarse_to_ref(self.restrict_native(nat)).reshape(-1)
        return xc.cpu().numpy() if host else xc

    def prolong(self, xc):
        host = not isinstance(xc, torch.Tensor)
        xd = torch.as_tensor(np.asarray(xc, dtype=np.complex128)).to(device()) if host else xc
        nat = self.coarse_from_ref(xd.reshape(1, self.n_blocks, self.nc))
        y = self._layout.from_native(self.prolong_native(nat)).reshape(-1)
        return y.cpu().numpy() if host else y

    def dense(self):
        """Dense N x Nc in reference order (oracle-scale interop only)."""
        eye = torch.eye(self.coarse_dim, dtype=torch.complex128, device=device())
        nat = self.coarse_from_ref(eye.reshape(self.coarse_dim, self.n_blocks, self.nc))
        cols = self._layout.from_native(self.prolong_native(nat))
        return cols.T.cpu().numpy()


def _block_maps(geo, blocking):
    """(b_native -> b_ref, (b_native, s) -> reference fine site) for the
    dense block layout of `Prolongator.P` (csrc/prolong.cu agg_site)."""
    L = np.array(geo.dims)
    B = np.array(blocking.block_dims)
    Cd = L // B
    m = int(np.prod(Cd))
    S = int(np.prod(B))
    bn = np.arange(m)
    c2 = bn % Cd[2]
    c1 = (bn // Cd[2]) % Cd[1]
    c0 = (bn // (Cd[2] * Cd[1])) % Cd[0]
    c3 = bn // (Cd[2] * Cd[1] * Cd[0])
    b_ref = ((c0 * Cd[1] + c1) * Cd[2] + c2) * Cd[3] + c3
    sl = np.arange(S)
    l2 = sl % B[2]
    l1 = (sl // B[2]) % B[1]
    l0 = (sl // (B[2] * B[1])) % B[0]
    l3 = sl // (B[2] * B[1] * B[0])
    x0 = c0[:, None] * B[0] + l0[None, :]
    x1 = c1[:, None] * B[1] + l1[None, :]
    x2 = c2[:, None] * B[2] + l2[None, :]
    x3 = c3[:, None] * B[3] + l3[None, :]
    site_ref = ((x0 * L[1] + x1) * L[2] + x2) * L[3] + x3
    return b_ref, site_ref


def prolongator_entries(pro):
    """Every stored entry of P in the reference's CSR terms: (col, fine row
    site, fine component, value), ordered by column then row like the
    reference's dump (multigrid.py:384-407).  Dropped columns are skipped and
    the surviving ones renumbered in the reference's column order."""
    geo, nv = pro.geometry, pro.nv
    m = pro.n_blocks
    S = int(np.prod(pro.blocking.block_dims))
    Ph = pro.P.reshape(m, 2, nv, 6, S).cpu().numpy()
    b_ref, site_ref = _block_maps(geo, pro.blocking)
    keep = pro.keep.reshape(m, 2, nv).astype(bool)
    order_b = np.argsort(b_ref)                      # native blocks in reference order
    cols, sites, comps, vals = [], [], [], []
    col = 0
    q = np.arange(6)
    for bn in order_b:
        for c in range(2):
            comp = (2 * c + q // 3) * 3 + q % 3      # (6,)
            row = site_ref[bn][None, :] * pro.fine_dof + comp[:, None]   # (6, S)
            ordr = np.argsort(row, axis=None)
            for k in range(nv):
                if not keep[bn, c, k]:
                    continue
                cols.append(np.full(6 * S, col))
                sites.append((row.reshape(-1)[ordr]) // pro.fine_dof)
                comps.append((row.reshape(-1)[ordr]) % pro.fine_dof)
                vals.append(Ph[bn, c, k].reshape(-1)[ordr])
                col += 1
    return np.concatenate(cols), np.concatenate(sites), np.concatenate(comps), np.concatenate(vals)


def prolongator_from_entries(geo, blocking, nv, col, site, comp, val, layout_op=None, fine_dof=12):
    """Inverse of `prolongator_entries` for a uniform P (every block and
    chirality keeps nv columns): the loader of multigrid.py:409-435."""
    blocking.validate(geo)
    m = blocking.block_count(geo)
    S = int(np.prod(blocking.block_dims))
    if int(np.max(col)) + 1 != 2 * nv * m:
        raise BlockingError("prolongator dump is not uniform (dropped columns); cannot place it")
    b_ref, site_ref = _block_maps(geo, blocking)
    ref_to_native_b = np.empty(m, dtype=np.int64)
    ref_to_native_b[b_ref] = np.arange(m)
    # fine reference site -> (native block, local s)
    where = np.empty((geo.site_count, 2), dtype=np.int64)
    where[site_ref.reshape(-1), 0] = np.repeat(np.arange(m), S)
    where[site_ref.reshape(-1), 1] = np.tile(np.arange(S), m)
    br = col // (2 * nv)
    c = (col % (2 * nv)) // nv
    k = col % nv
    bn = ref_to_native_b[br]
    if np.any(where[site, 0] != bn):
        raise BlockingError("prolongator dump: an entry lies outside its column's aggregate")
    spin = comp // 3
    if np.any(spin // 2 != c):
        raise BlockingError("prolongator dump: an entry has the wrong chirality for its column")
    q = (spin - 2 * c) * 3 + comp % 3
    Ph = np.zeros((m, 2, nv, 6, S), dtype=np.complex128)
    Ph[bn, c, k, q, where[site, 1]] = val
    P = torch.as_tensor(Ph.reshape(-1)).to(device())
    pro = Prolongator(P, geo, blocking, nv, fine_dof, np.ones(m * 2 * nv, dtype=np.int32))
    pro._layout = layout_op if layout_op is not None else _LayoutOnly(geo)
    return pro


def subspace_angles(prolongator, vectors):
    """sin of the principal angle between range(V) and each unit vector,
    sqrt(max(0, 1 - ||V^H v||^2)) (multigrid.py:303-313); vectors:
    reference-layout (n, N) or (N,), numpy or CUDA tensor."""
    V = torch.as_tensor(np.atleast_2d(np.asarray(vectors, dtype=np.complex128))).to(device()) \
        if not isinstance(vectors, torch.Tensor) else torch.atleast_2d(vectors)
    if hasattr(prolongator, "restrict_native"):
        c = prolongator.restrict_native(prolongator._layout.to_native(V.contiguous()))
        c2 = torch.linalg.vector_norm(c.reshape(c.shape[0], -1), dim=1) ** 2
    else:
        c2 = torch.linalg.vector_norm(prolongator.restrict(V), dim=-1) ** 2
    return np.sqrt(np.maximum(0.0, 1.0 - c2.cpu().numpy()))


def build_prolongator(null_vectors, blocking, layout_op=None):
    """Reference build_prolongator (multigrid.py:163-225) on the GPU."""
    geo = null_vectors.geometry
    blocking.validate(geo)
    nv = null_vectors.vectors.shape[0]
    m = blocking.block_count(geo)
    S = int(np.prod(blocking.block_dims))
    P = torch.empty(m * 2 * nv * 6 * S, dtype=torch.complex128, device=device())
    keep = np.zeros(m * 2 * nv, dtype=np.int32)
    _lib.check(_lib.lib().mgt_prolong_build(
        _lib.dims_arg(geo.dims), _lib.dims_arg(blocking.block_dims), nv, ptr(null_vectors.vectors.contiguous()),
        ptr(P), keep.ctypes.data_as(_lib.c_int_p), stream_ptr()), "build_prolongator")
    pro = Prolongator(P, geo, blocking, nv, null_vectors.dof, keep)
    pro._layout = layout_op if layout_op is not None else _LayoutOnly(geo)
    if pro.dropped:
        warnings.warn(f"dropped {pro.dropped} rank-deficient prolongator columns")
        for b, c in np.argwhere(pro.per_block_counts == 0):
            raise BlockingError(f"block {b} chirality {'+-'[c]} lost all columns: blocking too fine")
    return pro


class _LayoutOnly:
    """Layout conversions for a geometry without an operator handle."""

    def __init__(self, geo):
        self.geometry = geo
        self.prec = 64

    def to_native(self, x_ref):
        n = x_ref.shape[0]
        out = torch.empty((n, 12, self.geometry.site_count), dtype=torch.complex128, device=device())
        _lib.check(_lib.lib().mgt_spinor_from_ref(_lib.dims_arg(self.geometry.dims), 64, ptr(x_ref.contiguous()),
                                                   ptr(out), n, stream_ptr()))
        return out

    def from_native(self, x):
        n = x.shape[0]
        out = torch.empty((n, 12 * self.geometry.site_count), dtype=torch.complex128, device=device())
        _lib.check(_lib.lib().mgt_spinor_to_ref(_lib.dims_arg(self.geometry.dims), 64, ptr(x.contiguous()),
                                                 ptr(out), n, stream_ptr()))
        return out


# ---------------------------------------------------------------------------


def coarse_schur_blocks(C, cdims, nv, tau=0.0):
    """Even-odd factors of (C + i tau g5_c) for 9-block coarse storage C
    (flat, [b][dir][col][row]) on coarse dims `cdims` (every extent even):
    compact even / odd aggregate lists ie / io (cb index c -> aggregate),
    C_oo^-1 ([o][row][col]), D = C_oo^-1 C_o,dir (8 hops) and
    E = [C_ee, -C_e,dir] in the kernels' column-major block storage."""
    import types
    C0, C1, C2, C3 = cdims
    nb = C0 * C1 * C2 * C3
    nc = 2 * nv
    dev = C.device
    c = torch.arange(nb // 2, device=dev)
    b0 = 2 * c
    par0 = ((b0 % C2) + (b0 // C2) % C1 + (b0 // (C2 * C1)) % C0 + b0 // (C2 * C1 * C0)) & 1
    ie = b0 + (par0 != 0).long()  # compact index c -> full aggregate, even parity
    io = b0 + (par0 != 1).long()
    C4 = C.reshape(nb, 9, nc, nc)  # [b][dir][col][row]
    g5 = torch.ones(nc, dtype=torch.float64, device=dev)
    g5[nv:] = -1.0
    selfb = C4[:, 0] + torch.diag(1j * tau * g5).to(C4.dtype)  # diagonal: the same in either storage order
    Cooinv = torch.linalg.inv(selfb[io].transpose(-1, -2))      # [o][row][col]
    D = (Cooinv[:, None] @ C4[io, 1:].transpose(-1, -2)).transpose(-1, -2).contiguous()
    E = torch.cat([selfb[ie][:, None], -C4[ie, 1:]], dim=1).contiguous()
    return types.SimpleNamespace(tau=float(tau), ie=ie, io=io, Cooinv=Cooinv, D=D, E=E, D32=None, E32=None)


class CoarseOperator:
    """Galerkin V^H A V as 9 dense blocks per aggregate (multigrid.py:228-243)."""

    def __init__(self, C, prolongator, level=1):
        if not prolongator.uniform:
            raise BlockingError("coarse operator needs uniform per-block column counts "
                                "(rank-deficient blocks were dropped)")
        self.C = C
        self.prolongator = prolongator
        self.level = level
        self.geometry = prolongator.coarse_geometry
        self.dof = prolongator.nc
        self.gamma5_diag = prolongator.coarse_gamma5

    @property
    def dim(self):
        return self.prolongator.coarse_dim

    @property
    def shape(self):
        return (self.dim, self.dim)

    def apply_native(self, xc, out=None, low=False):
        """C xc for native coarse fields (n, nb, 2nv); low=True reads the
        fp32 copy of C (loose inner solves only)."""
        pr = self.prolongator
        xc = xc.contiguous()
        out = torch.empty_like(xc) if out is None else out
        d, b = pr._dims()
        if low:
            if getattr(self, "_c32", None) is None:
                self._c32 = self.C.to(torch.complex64)
            _lib.check(_lib.lib().mgt_coarse_apply_c32(d, b, pr.nv, ptr(self._c32), ptr(xc), ptr(out), xc.shape[0],
                                                        stream_ptr()), "coarse apply (fp32 C)")
            return out
        _lib.check(_lib.lib().mgt_coarse_apply(d, b, pr.nv, ptr(self.C), ptr(xc), ptr(out), xc.shape[0],
                                                stream_ptr()), "coarse apply")
        return out

    def apply(self, x):
        pr = self.prolongator
        host = not isinstance(x, torch.Tensor)
        xd = torch.as_tensor(np.asarray(x, dtype=np.complex128)).to(device()) if host else x
        if xd.shape[0] != self.dim:
            raise ValueError(f"dimension mismatch: {xd.shape[0]} != {self.dim}")
        nat = pr.coarse_from_ref(xd.reshape(1, pr.n_blocks, pr.nc))
        y = pr.coarse_to_ref(self.apply_native(nat)).reshape(-1)
        return y.cpu().numpy() if host else y

    def schur_factors(self, tau=0.0):
        """Coarse even-odd factors of (C + i tau g5_c) (every coarse extent
        even; `None` otherwise), cached per tau: the compact even / odd
        aggregate lists, C_oo^-1 per odd aggregate, the odd-side hop blocks
        D = C_oo^-1 C_o,dir and the even-side blocks E = [C_ee, -C_e,dir]
        of the Schur complement S = C_ee - C_eo C_oo^-1 C_oe
        (csrc/coarse.cu, mgt_coarse_half_apply / mgt_coarse_schur_*)."""
        key = float(tau)
        cache = getattr(self, "_schur", None)
        if cache is not None and cache.tau == key:
            return cache
        pr = self.prolongator
        cd = pr.blocking.coarse_dims(pr.geometry)
        if any(c % 2 for c in cd):
            return None
        self._schur = coarse_schur_blocks(self.C, cd, pr.nv, key)
        return self._schur

    def dense_native(self):
        """Dense Nc x Nc on the device, NATIVE coarse order (blocks of aliased
        neighbours summed)."""
        pr = self.prolongator
        nb, nc = pr.n_blocks, pr.nc
        nbr = torch.as_tensor(coarse_neighbours(pr.blocking.coarse_dims(pr.geometry)), device=device())
        blocks = self.C.reshape(nb, 9, nc, nc).transpose(-1, -2)  # -> [b][dir][row][col]
        D = torch.zeros((nb, nc, nb, nc), dtype=torch.complex128, device=device())
        rows = torch.arange(nb, device=device())
        for d in range(9):  # rows are distinct within one direction: no write conflicts
            D[rows, :, nbr[:, d], :] = D[rows, :, nbr[:, d], :] + blocks[:, d]
        return D.reshape(nb * nc, nb * nc)

    def dense_inverse_native(self):
        """C^-1 (native coarse order) by a dense fp64 LU on the device; built
        once and cached (setup of the full-prolongator deflation: Nc = 12,288
        at 16^4 is 2.4 GB)."""
        if getattr(self, "_dinv", None) is None:
            D = self.dense_native()
            self._dinv = torch.linalg.inv(D)
            del D
        return self._dinv

    def exact_inverse(self):
        """Exact C^-1 for the full-prolongator deflation (BASELINE configs[2]):
        returns an object with .t0 = tr(C^-1) and .apply_rows(H) = rows of
        H C^-T (i.e. (C^-1 h)^T for every row h), cached.  With every coarse
        extent even it is the coarse even-odd Schur factorisation
        (`CoarseSchurInverse`: ~3x fewer flops than the dense inverse), else
        the dense LU inverse."""
        if getattr(self, "_exact_inv", None) is None:
            pr = self.prolongator
            cd = pr.blocking.coarse_dims(pr.geometry)
            if all(c % 2 == 0 for c in cd):
                self._exact_inv = CoarseSchurInverse(self)
            else:
                self._exact_inv = _DenseInverse(self.dense_inverse_native())
        return self._exact_inv

    def dense(self):
        """Dense matrix in the reference coarse order (host numpy)."""
        pr = self.prolongator
        Dn = self.dense_native()
        perm = torch.as_tensor(native_to_ref_coarse(pr.blocking.coarse_dims(pr.geometry)), device=device())
        nc = pr.nc
        idx = (perm[:, None] * nc + torch.arange(nc, device=device())[None, :]).reshape(-1)
        Dr = torch.empty_like(Dn)
        Dr[idx[:, None], idx[None, :]] = Dn
        return Dr.cpu().numpy()


class _DenseInverse:
    def __init__(self, Dinv):
        self.Dinv = Dinv
        self.t0 = complex(torch.diagonal(Dinv).sum().item())

    def apply_rows(self, H):
        return H @ self.Dinv.transpose(0, 1)


class CoarseSchurInverse:
    """C^-1 through the coarse checkerboard (every coarse extent even: the
    9-point coarse stencil couples only opposite-parity aggregates, so C_oo
    and C_ee are block diagonal -- one 2nv x 2nv block per aggregate):
        S = C_ee - C_eo C_oo^-1 C_oe,   A = C_eo C_oo^-1,   B = C_oo^-1 C_oe,
        tr(C^-1) = tr(S^-1) + tr(C_oo^-1) + tr(S^-1 A B),
        y_e = S^-1 (h_e - A h_o),   y_o = C_oo^-1 h_o - B y_e.
    The reference forms tr(C^-1) by a dense factorisation of the whole
    Nc x Nc operator (trace.py:203-217); this does one dense inverse of
    half the size; S and the trace term are assembled from the 48 x 48
    blocks (the hops couple opposite parities only, so S and A B have the
    2-hop block pattern), exact in fp64 arithmetic (same t0 to rounding)."""

    def __init__(self, coarse):
        pr = coarse.prolongator
        cd = pr.blocking.coarse_dims(pr.geometry)
        C0, C1, C2, C3 = cd
        nb, nc = pr.n_blocks, pr.nc
        b = np.arange(nb)
        par = ((b % C2) + (b // C2) % C1 + (b // (C2 * C1)) % C0 + b // (C2 * C1 * C0)) & 1
        dev = device()
        cols = np.arange(nc)
        ev, od = np.flatnonzero(par == 0), np.flatnonzero(par == 1)
        iE = torch.as_tensor((ev[:, None] * nc + cols).reshape(-1), device=dev)
        iO = torch.as_tensor((od[:, None] * nc + cols).reshape(-1), device=dev)
        ne, no = len(ev), len(od)
        pos = np.empty(nb, dtype=np.int64)  # aggregate -> index within its parity
        pos[ev] = np.arange(ne)
        pos[od] = np.arange(no)
        nbr = coarse_neighbours(cd)
        # block-sparse pieces (matrix form [row][col]; C storage is column-major):
        # every hop couples opposite parities, so C_eo / C_oe have 8 blocks per
        # block row and S = C_ee - C_eo C_oo^-1 C_oe has the 2-hop pattern
        Mb = coarse.C.reshape(nb, 9, nc, nc).transpose(-1, -2)
        Mo = Mb[torch.as_tensor(od, device=dev)]                       # (no, 9, nc, nc)
        Me = Mb[torch.as_tensor(ev, device=dev)]                       # (ne, 9, nc, nc)
        self.Cooinv = torch.linalg.inv(Mo[:, 0])                       # (no, nc, nc)
        oe = torch.as_tensor(pos[nbr[ev, 1:]], device=dev)             # (ne, 8) odd neighbours of even
        eo = torch.as_tensor(pos[nbr[od, 1:]], device=dev)             # (no, 8) even neighbours of odd
        Ae = Me[:, 1:] @ self.Cooinv[oe]                               # A blocks C_e,d C_oo^-1   (ne, 8, nc, nc)
        Bo = self.Cooinv[:, None] @ Mo[:, 1:]                          # B blocks C_oo^-1 C_o,d'  (no, 8, nc, nc)
        er, orr = torch.arange(ne, device=dev), torch.arange(no, device=dev)
        S = torch.zeros((ne, nc, ne, nc), dtype=coarse.C.dtype, device=dev)
        S[er, :, er, :] = Me[:, 0]
        for d in range(8):
            o = oe[:, d]
            for d2 in range(8):
                # block (e, e2) += -C_e,d C_oo^-1 C_o,d2; e -> e2 is a translation,
                # so the targets are distinct for fixed (d, d2)
                S[er, :, eo[o, d2], :] -= Ae[:, d] @ Mo[o, 1 + d2]
        self.Sinv = torch.linalg.inv(S.reshape(ne * nc, ne * nc))
        del S
        # tr(S^-1 A B) over the 2-hop blocks (e -> e2) of A B:
        # sum <S^-1[e2, e], (A_e,d B_o,d2)^T>
        Sb = self.Sinv.reshape(ne, nc, ne, nc)
        tr_sab = torch.zeros((), dtype=coarse.C.dtype, device=dev)
        for d in range(8):
            o = oe[:, d]
            for d2 in range(8):
                P = Ae[:, d] @ Bo[o, d2]                               # block (e, e2) of A B
                tr_sab = tr_sab + torch.sum(Sb[eo[o, d2], :, er, :] * P.transpose(-1, -2))
        self.t0 = complex((torch.diagonal(self.Sinv).sum() + torch.diagonal(self.Cooinv, dim1=1, dim2=2).sum()
                           + tr_sab).item())
        # dense A = C_eo C_oo^-1 and B = C_oo^-1 C_oe for the per-probe
        # products (scatter-add: on extent-2 coarse lattices the +mu and -mu
        # neighbours coincide and add up, as in C)
        A = torch.zeros((ne, nc, no, nc), dtype=coarse.C.dtype, device=dev)
        B = torch.zeros((no, nc, ne, nc), dtype=coarse.C.dtype, device=dev)
        ar = torch.arange(nc, device=dev)
        for d in range(8):
            A.index_put_((er[:, None, None], ar[None, :, None], oe[:, d][:, None, None], ar[None, None, :]),
                         Ae[:, d], accumulate=True)
            B.index_put_((orr[:, None, None], ar[None, :, None], eo[:, d][:, None, None], ar[None, None, :]),
                         Bo[:, d], accumulate=True)
        self.A, self.B = A.reshape(ne * nc, no * nc), B.reshape(no * nc, ne * nc)
        self.iE, self.iO, self.no, self.nc = iE, iO, no, nc

    def apply_rows(self, H):
        """rows (C^-1 h)^T for the rows h of H (n, Nc), native coarse order."""
        He, Ho = H[:, self.iE], H[:, self.iO]
        Ye = (He - Ho @ self.A.transpose(0, 1)) @ self.Sinv.transpose(0, 1)
        Yo = torch.einsum("jab,njb->nja", self.Cooinv, Ho.reshape(H.shape[0], self.no, self.nc)).reshape(Ho.shape) \
            - Ye @ self.B.transpose(0, 1)
        Y = torch.empty_like(H)
        Y[:, self.iE] = Ye
        Y[:, self.iO] = Yo
        return Y


def coarse_gamma5(x, nv):
    """gamma5_c on native coarse fields (n, nb, 2nv): -1 on the nv chirality-
    columns of every aggregate (multigrid.py:213)."""
    y = x.clone()
    y[..., nv:] = -y[..., nv:]
    return y


LOW_PRECISION_TOL = 1e-5  # coarse solves at least this loose iterate with fp32 C


def _schur_bicgstab(coarse, F, b, tol, max_iter):
    """BiCGStab on the coarse Schur complement S x_e = b_e - C_eo C_oo^-1 b_o
    (coarse even-odd form), x_o = C_oo^-1 (b_o - C_oe x_e): the odd rows are
    solved exactly, so the full residual is (bh_e - S x_e, 0) and the
    stopping test is the reference's ||b - C x|| <= tol ||b||
    (krylov.py:78-85) on the explicitly recomputed Schur residual."""
    pr = coarse.prolongator
    nv = pr.nv
    low = tol >= LOW_PRECISION_TOL
    if low and F.D32 is None:
        F.D32, F.E32 = F.D.to(torch.complex64), F.E.to(torch.complex64)
    Dm, Em = (F.D32, F.E32) if low else (F.D, F.E)
    d, bk = pr._dims()
    lib = _lib.lib()
    n = b.shape[0]
    be, bo = b[:, F.ie].contiguous(), b[:, F.io].contiguous()
    uo = torch.einsum("orc,noc->nor", F.Cooinv, bo).contiguous()
    hop = torch.empty_like(be)
    _lib.check(lib.mgt_coarse_half_apply(d, bk, nv, ptr(F.E), 9, 0, 0, 1, None, ptr(uo), ptr(hop), n, stream_ptr()),
               "coarse half apply")
    bh = be + hop
    to = torch.empty_like(be)

    def S(v):  # exact (fp64) Schur apply
        y = torch.empty_like(v)
        _lib.check(lib.mgt_coarse_schur_apply(d, bk, nv, ptr(F.D), ptr(F.E), 0, ptr(v), ptr(y), ptr(to), v.shape[0],
                                              stream_ptr()), "coarse Schur apply")
        return y

    def dot(u, v):
        return torch.sum(u.conj() * v, dim=(1, 2))

    b2 = dot(b, b).real
    tol2 = (tol * tol) * b2
    x = torch.zeros_like(bh)
    r = bh.clone()
    rhat, p = r.clone(), r.clone()
    v, s_, t = torch.empty_like(r), torch.empty_like(r), torch.empty_like(r)
    rho = dot(rhat, r)
    done = (b2 == 0).cpu().numpy().copy()
    state = torch.zeros((n, 16), dtype=torch.float64, device=b.device)
    state[:, 0], state[:, 1] = rho.real, rho.imag
    state[:, 9] = torch.as_tensor(~done, device=b.device, dtype=torch.float64)
    state[:, 10] = tol2
    state[:, 13] = 1.0  # freeze: converged rhs stop themselves inside a multi-iteration call
    tol2_h = tol2.cpu().numpy()
    mv_extra = np.zeros(n, dtype=int)
    rt = None
    its = np.zeros(n, dtype=int)
    # the first call runs as many iterations as the previous solve of this
    # tolerance needed (the Davidson's inner solves repeat), then one per call:
    # few host round trips, at most a couple of surplus iterations
    hints = F.__dict__.setdefault("its_hint", {})
    k_next = max(1, hints.get(tol, 2))
    while not done.all() and its[~done].max(initial=0) < max_iter:
        k = int(min(k_next, max_iter - its[~done].max(initial=0)))
        k_next = 1
        _lib.check(lib.mgt_coarse_schur_bicgstab(d, bk, nv, ptr(Dm), ptr(Em), 1 if low else 0, n, k, ptr(x), ptr(r),
                                                 ptr(rhat), ptr(p), ptr(v), ptr(s_), ptr(t), ptr(to), ptr(state),
                                                 stream_ptr()), "coarse Schur bicgstab")
        st = state.cpu().numpy()
        its = st[:, 12].astype(int)
        newly = (st[:, 11] != 0) & (st[:, 9] == 0) & ~done
        if ((st[:, 9] == 0) & ~done & ~newly).any():
            raise RuntimeError("coarse Schur BiCGStab: a system stopped without converging")
        rt = None
        if newly.any():
            rt = bh - S(x)
            mv_extra[newly] += 1
            rt2 = dot(rt, rt).real.cpu().numpy()
            ok = newly & (rt2 <= tol2_h)
            done |= ok
            again = newly & ~ok
            if again.any():  # the recursion drifted from the true residual: restart from it
                ag = torch.as_tensor(np.flatnonzero(again), device=b.device)
                r[ag] = rt[ag]
                rhat[ag] = rt[ag]
                p[ag] = rt[ag]
                rr = dot(rt[ag], rt[ag])
                state[ag, 0], state[ag, 1] = rr.real, rr.imag
                state[ag, 9] = 1.0
                state[ag, 11] = 0.0
    hints[tol] = max(1, int(its.max(initial=1)) - 1)
    if rt is None:
        rt = bh - S(x)
    xo = torch.empty_like(uo)
    _lib.check(lib.mgt_coarse_half_apply(d, bk, nv, ptr(F.D), 8, 1, 0, 0, None, ptr(x), ptr(xo), n, stream_ptr()),
               "coarse half apply")
    xo = uo - xo
    xf = torch.empty_like(b)
    xf[:, F.ie] = x
    xf[:, F.io] = xo
    rel = (dot(rt, rt).real / torch.where(b2 > 0, b2, 1)).sqrt().cpu().numpy()
    # matvecs in full-operator units: 2 Schur applies per iteration (each ~ one C apply)
    reps = [(int(its[i]), float(rel[i]), bool(rel[i] <= tol or float(b2[i]) == 0.0), int(2 * its[i] + mv_extra[i] + 1))
            for i in range(n)]
    return xf, reps


def coarse_bicgstab(coarse, b, tol, max_iter, tau=0.0, even_odd=True):
    """BiCGStab on the coarse operator (C + i tau g5_c) for native coarse
    fields b (n, nb, 2nv), every rhs with its own scalars; zero start,
    convergence confirmed on the explicit residual (krylov.py:78-85).
    The matvec is the coarse block-stencil kernel; the short BLAS-1 runs as
    batched device tensor ops (coarse vectors are Nc = 48 x aggregates long).
    Returns (x, [(iterations, relres, converged, matvecs)]).
    even_odd (default): every coarse extent even -> BiCGStab on the coarse
    Schur complement (`_schur_bicgstab`, about half the iterations)."""
    if even_odd:
        F = coarse.schur_factors(tau)
        if F is not None:
            return _schur_bicgstab(coarse, F, b.contiguous(), tol, max_iter)
    nv = coarse.prolongator.nv
    # loose solves (the coarse Davidson's inner tol 1e-3) iterate with the
    # fp32 copy of C; the explicit-residual confirmation below uses fp64 C
    low = tol >= LOW_PRECISION_TOL

    def A(v, exact=False):
        y = coarse.apply_native(v, low=low and not exact)
        if tau != 0.0:
            y = y + 1j * tau * coarse_gamma5(v, nv)
        return y

    def dot(u, v):
        return torch.sum(u.conj() * v, dim=(1, 2))

    # the iteration itself (2 stencil applies, fused vector updates and
    # reductions, device-side scalars) is one C-ABI call per step
    pr = coarse.prolongator
    d, bk = pr._dims()
    if low and getattr(coarse, "_c32", None) is None:
        coarse._c32 = coarse.C.to(torch.complex64)
    Cm = coarse._c32 if low else coarse.C
    n = b.shape[0]
    b = b.contiguous()
    x = torch.zeros_like(b)
    r = b.clone()
    b2 = dot(b, b).real
    tol2 = (tol * tol) * b2
    rhat = r.clone()
    p = r.clone()
    v, s, t = torch.empty_like(b), torch.empty_like(b), torch.empty_like(b)
    rho = dot(rhat, r)
    its = np.zeros(n, dtype=int)
    mv = np.zeros(n, dtype=int)
    done = (b2 == 0).cpu().numpy().copy()
    state = torch.zeros((n, 16), dtype=torch.float64, device=b.device)
    state[:, 0], state[:, 1] = rho.real, rho.imag
    state[:, 9] = torch.as_tensor(~done, device=b.device, dtype=torch.float64)
    state[:, 10] = tol2
    lib = _lib.lib()
    tol2_h = tol2.cpu().numpy()
    rt = None  # explicit residual of the current x (valid until the next step)
    for it in range(max_iter):
        if done.all():
            break
        rt = None
        _lib.check(lib.mgt_coarse_bicgstab_iter(d, bk, nv, ptr(Cm), 1 if low else 0, float(tau), n, ptr(x), ptr(r),
                                                ptr(rhat), ptr(p), ptr(v), ptr(s), ptr(t), ptr(state), stream_ptr()),
                   "coarse bicgstab iteration")
        st = state.cpu().numpy()
        act = st[:, 9] != 0
        its[act] += 1
        mv[act] += 2
        conv = (st[:, 11] != 0) & act
        if conv.any():
            # confirm on the explicit residual; restart the ones that drifted
            rt = b - A(x, exact=True)
            mv[act] += 1
            rt2 = dot(rt, rt).real.cpu().numpy()
            ok = conv & (rt2 <= tol2_h)
            done |= ok
            again = conv & ~ok
            if again.any():
                ag = torch.as_tensor(np.flatnonzero(again), device=b.device)
                r[ag] = rt[ag]
                rhat[ag] = rt[ag]
                p[ag] = rt[ag]
                rr = dot(rt[ag], rt[ag])
                state[ag, 0], state[ag, 1] = rr.real, rr.imag
            state[:, 9] = torch.as_tensor(~done, device=b.device, dtype=torch.float64)
    if rt is None:  # (else: the last confirmation already holds b - A x for this x)
        rt = b - A(x, exact=True)
    rel = (dot(rt, rt).real / torch.where(b2 > 0, b2, 1)).sqrt().cpu().numpy()
    reps = [(int(its[i]), float(rel[i]), bool(rel[i] <= tol or float(b2[i]) == 0.0), int(mv[i] + 1))
            for i in range(n)]
    return x, reps


def coarse_neighbours(cdims):
    """(nb, 9) native neighbour table: dir 0 self, 1 + 2 mu + s."""
    C0, C1, C2, C3 = cdims
    nb = C0 * C1 * C2 * C3
    b = np.arange(nb)
    c2 = b % C2
    c1 = (b // C2) % C1
    c0 = (b // (C2 * C1)) % C0
    c3 = b // (C2 * C1 * C0)
    coords = [c0, c1, c2, c3]
    out = np.empty((nb, 9), dtype=np.int64)
    out[:, 0] = b
    for mu in range(4):
        for s, sgn in enumerate((1, -1)):
            cc = [c.copy() for c in coords]
            cc[mu] = (cc[mu] + sgn) % cdims[mu]
            out[:, 1 + 2 * mu + s] = ((cc[3] * C0 + cc[0]) * C1 + cc[1]) * C2 + cc[2]
    return out


def native_to_ref_coarse(cdims):
    C0, C1, C2, C3 = cdims
    nb = C0 * C1 * C2 * C3
    b = np.arange(nb)
    c2 = b % C2
    c1 = (b // C2) % C1
    c0 = (b // (C2 * C1)) % C0
    c3 = b // (C2 * C1 * C0)
    return ((c0 * C1 + c1) * C2 + c2) * C3 + c3


def build_coarse_operator(op, prolongator, level=1, check=True):
    """Reference build_coarse_operator (multigrid.py:246-259): C = P^H A P on
    the GPU, with the inherited gamma5_c-Hermiticity check to 1e-12."""
    pr = prolongator
    nb, nc = pr.n_blocks, pr.nc
    C = torch.empty(nb * 9 * nc * nc, dtype=torch.complex128, device=device())
    _lib.check(_lib.lib().mgt_coarse_build(op.handle, _lib.dims_arg(pr.blocking.block_dims), pr.nv, ptr(pr.P),
                                            ptr(C), stream_ptr()), "build_coarse_operator")
    coarse = CoarseOperator(C, pr, level=level)
    if check:
        _check_gamma5_hermitian(coarse)
    return coarse


def _check_gamma5_hermitian(coarse):
    """g5c C g5c = C^H blockwise: block (b, dir) vs (nbr, opposite)^H."""
    pr = coarse.prolongator
    nb, nc = pr.n_blocks, pr.nc
    nbr = torch.as_tensor(coarse_neighbours(pr.blocking.coarse_dims(pr.geometry)), device=device())
    B = coarse.C.reshape(nb, 9, nc, nc).transpose(-1, -2)  # [b][dir][row][col]
    g = torch.as_tensor(np.concatenate([np.ones(pr.nv), -np.ones(pr.nv)]), device=device(),
                        dtype=torch.complex128)
    opp = [0, 2, 1, 4, 3, 6, 5, 8, 7]
    scale = B.abs().max().item()
    worst = 0.0
    for d in range(9):
        lhs = g[:, None] * B[:, d] * g[None, :]
        rhs = B[nbr[:, d], opp[d]].conj().transpose(-1, -2)
        worst = max(worst, (lhs - rhs).abs().max().item())
    if worst > 1e-12 * max(scale, 1e-300):
        raise ValueError(f"coarse operator lost gamma5-Hermiticity: {worst:.3e}")
