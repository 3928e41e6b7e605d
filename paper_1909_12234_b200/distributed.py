"""Multi-GPU: probe sharding and t-slab domain decomposition.

One process per GPU (`torch.distributed`, NCCL over NVLink/NVSwitch on the
B200 box; gloo works for the host-side logic on CPU).

Probe sharding: Hutchinson probes are independent
(trace.py:100-107).  Rank r takes the contiguous probe block
[r s / W, (r+1) s / W); probe j keeps its reference seed seed0 + j
(probing.py:155), so the union of the shards is exactly the single-process
probe set.  The only collective is one all-gather of the per-probe complex
samples at the end; every rank then reduces them in GLOBAL probe order with
the reference's `_finish` arithmetic (trace.py:73-92).  A probe's solve
does not depend on the batch it was solved in (the solver's reductions are
tile-ordered, csrc/reduce.cuh; tests/test_batch_invariance_gpu.py), so a
sharded Hutchinson estimate is bitwise equal to the single-GPU one.  The
deflated estimators add per-batch projection corrections (U^H z, Y^H z)
whose summation order depends on the batch width (kernel choice and grid of
mgt_proj_vhx); their sharded samples agree with the single-GPU ones to
rounding (~1e-16 relative), not bitwise.

t-slab decomposition: see `SlabWilsonOperator`.
"""

import numpy as np
import torch
import torch.distributed as dist

from .trace import finish


def shard_range(n, rank, world):
    """Contiguous block [j0, j1) of n items owned by `rank`."""
    return rank * n // world, (rank + 1) * n // world


def gather_samples(local, n_total, group=None, device=None):
    """All-gather per-rank complex sample blocks (contiguous shards, rank
    order) into the global (n_total,) complex128 array, on every rank."""
    world = dist.get_world_size(group)
    local = np.asarray(local, dtype=np.complex128)
    counts = [shard_range(n_total, r, world)[1] - shard_range(n_total, r, world)[0] for r in range(world)]
    width = max(counts) if counts else 0
    buf = torch.zeros((width, 2), dtype=torch.float64, device=device)
    if len(local):
        buf[:len(local), 0] = torch.as_tensor(local.real)
        buf[:len(local), 1] = torch.as_tensor(local.imag)
    outs = [torch.empty_like(buf) for _ in range(world)]
    dist.all_gather(outs, buf, group=group)
    parts = []
    for r in range(world):
        o = outs[r][:counts[r]].cpu().numpy()
        parts.append(o[:, 0] + 1j * o[:, 1])
    return np.concatenate(parts) if parts else np.zeros(0, dtype=np.complex128)


def sharded_estimate(local_estimator, n_total, group=None, device=None, t0=None):
    """Run `local_estimator(j0, j1) -> TraceEstimate` on this rank's probe
    shard, gather the samples, and finish in global probe order.  t0 (the
    deterministic part) defaults to the local estimate's t0, identical on
    every rank by construction."""
    rank = dist.get_rank(group)
    world = dist.get_world_size(group)
    j0, j1 = shard_range(n_total, rank, world)
    est = local_estimator(j0, j1)
    samples = gather_samples(est.samples, n_total, group, device)
    inv = torch.tensor([int(est.inversions)], dtype=torch.int64, device=device)
    dist.all_reduce(inv, group=group)
    t0v = est.t0 if t0 is None else t0
    return finish(t0v, samples, int(inv.item()))


def _local_vhx(V, X):
    from .linalg import vhx
    return vhx(V, X)


def _local_sub(V, H, X):
    from .linalg import sub_vh
    return sub_vh(V, H, X)


def slab_vhx(V, X, group=None, local=None):
    """t-sharded H = V^H X (the deflation projection on t-slab
    fields): each rank forms its slab's k x s partial with the projection
    kernels, the partials are all-gathered and summed in rank order on every
    rank -- bitwise identical on all ranks and independent of the
    collective's own reduction order (k x s is small next to the slabs).
    V: (k, ...) and X: (s, ...) this rank's slab fields; returns (k, s)."""
    H = (local or _local_vhx)(V, X)
    world = dist.get_world_size(group)
    if world == 1:
        return H
    Hr = torch.view_as_real(H.contiguous()).contiguous()
    parts = [torch.empty_like(Hr) for _ in range(world)]
    dist.all_gather(parts, Hr, group=group)
    out = parts[0].clone()
    for p in parts[1:]:
        out += p
    return torch.view_as_complex(out)


def slab_project_out(V, X, group=None, local_vhx=None, local_sub=None):
    """t-sharded X <- X - V (V^H X) in place on this rank's slab (the
    orthogonal deflation / CGS2 step, trace.py:182-183, eigen.py:79-86);
    returns the global H = V^H X."""
    H = slab_vhx(V, X, group, local_vhx)
    (local_sub or _local_sub)(V, H, X)
    return H


def exchange_halos(to_prev, to_next, group=None):
    """Ring exchange of the two t-faces: `to_prev` (this rank's first-slice
    face) goes to rank - 1, `to_next` (last-slice face) to rank + 1.
    Returns (from_next, from_prev).  One grouped send/recv pair per
    direction (NCCL over NVLink on CUDA tensors, gloo on CPU tensors)."""
    world = dist.get_world_size(group)
    rank = dist.get_rank(group)
    if world == 1:
        return to_prev, to_next
    nxt, prv = (rank + 1) % world, (rank - 1) % world
    from_next = torch.empty_like(to_prev)
    from_prev = torch.empty_like(to_next)
    ops = [dist.P2POp(dist.isend, to_prev.contiguous(), prv, group),
           dist.P2POp(dist.irecv, from_next, nxt, group),
           dist.P2POp(dist.isend, to_next.contiguous(), nxt, group),
           dist.P2POp(dist.irecv, from_prev, prv, group)]
    for req in dist.batch_isend_irecv(ops):
        req.wait()
    return from_next, from_prev


class PeerHaloWindows:
    """Receive windows of the peer-memory halo transport.

    One device allocation per rank (`mgt_ipc_alloc`), laid out as
    [parity][face][rhs][6][S3] with face 0 = the face from rank + 1 (this
    rank's halo_next) and face 1 = the face from rank - 1 (halo_prev).  The
    64-byte CUDA IPC handles are all-gathered once; each rank maps its two
    t neighbours' windows (`mgt_ipc_open`), so `mgt_halo_pack` with
    MGT_HALO_PEER stores the projected faces straight into the neighbours'
    memory over NVLink -- the pack (spin projection + U^dag multiply) and the
    transfer are one kernel, no NCCL send/recv, no staging copy.  Parity
    alternates per apply (double buffering): pack k+1 writes the other half,
    and the barrier of apply k+1 orders pack k+2 after every neighbour's
    boundary kernel of apply k."""

    def __init__(self, S3, max_rhs, elem_bytes):
        from . import _lib
        self._lib = _lib
        self.face_bytes = int(max_rhs) * 6 * int(S3) * int(elem_bytes)
        self.max_rhs = int(max_rhs)
        self.nbytes = 4 * self.face_bytes
        p = _lib.ct.c_void_p()
        self.handle = (_lib.ct.c_char * _lib.IPC_HANDLE_BYTES)()
        _lib.check(_lib.lib().mgt_ipc_alloc(self.nbytes, _lib.ct.byref(p), self.handle), "ipc alloc")
        self.ptr = p.value
        self.prev_ptr = self.next_ptr = None
        self._opened = []

    def slot(self, base, parity, face):
        return base + (2 * parity + face) * self.face_bytes

    def connect_local(self, prev, nxt):
        """In-process wiring (single-GPU rank emulation; world == 1 wraps to
        itself): the neighbours' windows are plain device pointers."""
        self.prev_ptr, self.next_ptr = prev.ptr, nxt.ptr

    def connect(self, rank, world, group=None):
        """All-gather the IPC handles and map the t neighbours' windows."""
        if world == 1:
            return self.connect_local(self, self)
        hs = [None] * world
        dist.all_gather_object(hs, bytes(self.handle), group=group)
        prv, nxt = (rank - 1) % world, (rank + 1) % world
        mapped = {}
        for r in {prv, nxt}:
            p = self._lib.ct.c_void_p()
            buf = (self._lib.ct.c_char * self._lib.IPC_HANDLE_BYTES).from_buffer_copy(hs[r])
            self._lib.check(self._lib.lib().mgt_ipc_open(buf, self._lib.ct.byref(p)), "ipc open")
            mapped[r] = p.value
            self._opened.append(p.value)
        self.prev_ptr, self.next_ptr = mapped[prv], mapped[nxt]

    def close(self):
        lib = self._lib.lib()
        for p in self._opened:
            lib.mgt_ipc_close(self._lib.ct.c_void_p(p))
        self._opened = []
        if self.ptr:
            lib.mgt_ipc_free(self._lib.ct.c_void_p(self.ptr))
            self.ptr = None

    def __del__(self):
        try:
            self.close()
        except Exception:
            pass


def slab_links(gauge_links, dims, t_begin, t_local):
    """The slab's links in the reference layout of the LOCAL dims (t fastest)."""
    L0, L1, L2, T = dims
    U = gauge_links.reshape(L0, L1, L2, T, 4, 3, 3)[:, :, :, t_begin:t_begin + t_local]
    return U.contiguous().reshape(-1, 4, 3, 3)


class SlabWilsonOperator:
    """The Wilson operator on this rank's t-slab of a global lattice.

    Native fields are the local slab (n, 12, V_local).  `apply_native` packs
    the two spin-projected faces (`mgt_halo_pack`), starts the interior
    sites (which need no halo) on a side stream, exchanges the faces with
    rank -/+ 1 over NCCL (`exchange_halos`) and finishes the two boundary
    slices.  `exchange` may be replaced (tests emulate several ranks in one
    process by swapping faces between slab operators)."""

    def __init__(self, gauge, mass, rank, world, prec=64, recon=12, group=None, local_links=None,
                 transport="nccl", max_rhs=4, connect=True):
        """gauge: the GLOBAL GaugeField (the slab's links are cut out of it),
        or a (geometry, None) stand-in together with `local_links`, the slab's
        own links in local reference layout (when no rank holds the global
        field).  transport: "nccl" (grouped send/recv of the packed faces) or
        "p2p" (the pack kernel writes into the neighbours' IPC-mapped receive
        windows, `PeerHaloWindows`); with connect=False the p2p windows are
        wired later (`connect_local`, single-process rank emulation)."""
        from . import _lib
        from ._device import ptr, stream_ptr
        geo = gauge.geometry
        T = geo.dims[3]
        if T % world:
            raise ValueError(f"T = {T} is not divisible by {world} ranks")
        self.t_local = T // world
        if self.t_local < 2:
            raise ValueError("each t-slab needs >= 2 time slices")
        self.t_begin = rank * self.t_local
        self.global_geometry = geo
        self.rank, self.world, self.group = rank, world, group
        self.prec, self.recon, self.mass = prec, recon, float(mass)
        self.local_dims = geo.dims[:3] + (self.t_local,)
        self.volume = int(np.prod(self.local_dims))
        self.S3 = int(np.prod(geo.dims[:3]))
        links = local_links if local_links is not None else slab_links(gauge.links, geo.dims, self.t_begin,
                                                                         self.t_local)
        self._lib = _lib
        self._handle = _lib.ct.c_void_p()
        _lib.check(_lib.lib().mgt_wilson_create_slab(
            _lib.ct.byref(self._handle), _lib.dims_arg(self.local_dims), self.t_begin, T,
            1 if geo.boundary == "antiperiodic" else 0, self.mass, prec, recon, ptr(links), stream_ptr()),
            "slab operator")
        torch.cuda.current_stream().synchronize()
        self.exchange = lambda a, b: exchange_halos(a, b, self.group)
        self._side = torch.cuda.Stream()
        if transport not in ("nccl", "p2p"):
            raise ValueError(f"unknown halo transport {transport!r}")
        self.transport = transport
        self.windows = None
        self._parity = 0
        self._barrier = None
        if transport == "p2p":
            esz = 16 if prec == 64 else 8
            self.windows = PeerHaloWindows(self.S3, max_rhs, esz)
            if connect:
                self.windows.connect(rank, world, group)
                if world > 1:
                    self._barrier = torch.zeros(1, dtype=torch.int32, device="cuda")

    @staticmethod
    def connect_local(ops):
        """Wire the p2p windows of in-process slab operators (ranks 0..W-1 of
        one emulated ring) without IPC; the caller orders post/complete."""
        W = len(ops)
        for r, op in enumerate(ops):
            op.windows.connect_local(ops[(r - 1) % W].windows, ops[(r + 1) % W].windows)

    def __del__(self):
        h = getattr(self, "_handle", None)
        if h is not None and h.value:
            try:
                torch.cuda.synchronize()
                self._lib.lib().mgt_wilson_destroy(h)
            except Exception:
                pass
            self._handle = None

    @property
    def dtype(self):
        return torch.complex128 if self.prec == 64 else torch.complex64

    def pack(self, x, flags=0, tau=0.0):
        from ._device import ptr, stream_ptr
        n = x.shape[0]
        to_prev = torch.empty((n, 6, self.S3), dtype=self.dtype, device=x.device)
        to_next = torch.empty_like(to_prev)
        self._lib.check(self._lib.lib().mgt_halo_pack(self._handle, ptr(x), ptr(to_prev), ptr(to_next), n,
                                                      int(flags), float(tau), stream_ptr()), "halo pack")
        return to_prev, to_next

    def apply_part(self, x, out, halo_next, halo_prev, part, flags=0, tau=0.0):
        from ._device import ptr, stream_ptr
        self._lib.check(self._lib.lib().mgt_wilson_apply_slab(
            self._handle, ptr(x), ptr(out), ptr(halo_next) if halo_next is not None else None,
            ptr(halo_prev) if halo_prev is not None else None, x.shape[0], int(flags), float(tau), int(part),
            stream_ptr()), "slab apply")
        return out

    # -- p2p transport: post (pack into the neighbours + interior) / complete
    def post(self, x, out, flags=0, tau=0.0):
        """Pack this rank's two faces straight into the neighbours' receive
        windows (MGT_HALO_PEER) and start the interior slices on the side
        stream."""
        from ._device import ptr, stream_ptr
        n = x.shape[0]
        if n > self.windows.max_rhs:
            raise ValueError(f"n_rhs {n} exceeds the halo window capacity {self.windows.max_rhs}")
        w, par = self.windows, self._parity
        self._lib.check(self._lib.lib().mgt_halo_pack(
            self._handle, ptr(x), w.slot(w.prev_ptr, par, 0), w.slot(w.next_ptr, par, 1), n,
            int(flags) | self._lib.HALO_PEER, float(tau), stream_ptr()), "halo pack (peer)")
        main = torch.cuda.current_stream()
        if self.t_local > 2:
            self._side.wait_stream(main)
            with torch.cuda.stream(self._side):
                self.apply_part(x, out, None, None, 1, flags, tau)
        return out

    def complete(self, x, out, flags=0, tau=0.0):
        """Stream-ordered barrier (every rank's pack has landed), then the two
        boundary slices from this rank's own window; flips the parity."""
        from ._device import ptr, stream_ptr
        if self._barrier is not None:
            dist.all_reduce(self._barrier, group=self.group)
        w, par = self.windows, self._parity
        part = 2 if self.t_local > 2 else 0
        self._lib.check(self._lib.lib().mgt_wilson_apply_slab(
            self._handle, ptr(x), ptr(out), w.slot(w.ptr, par, 0), w.slot(w.ptr, par, 1), x.shape[0],
            int(flags), float(tau), part, stream_ptr()), "slab apply (peer halos)")
        if self.t_local > 2:
            torch.cuda.current_stream().wait_stream(self._side)
        self._parity ^= 1
        return out

    def apply_native(self, x, out=None, flags=0, tau=0.0, overlap=True):
        x = x.contiguous()
        out = torch.empty_like(x) if out is None else out
        if self.transport == "p2p":
            self.post(x, out, flags, tau)
            return self.complete(x, out, flags, tau)
        main = torch.cuda.current_stream()
        to_prev, to_next = self.pack(x, flags, tau)
        if overlap and self.t_local > 2:
            self._side.wait_stream(main)
            with torch.cuda.stream(self._side):
                self.apply_part(x, out, None, None, 1, flags, tau)
            halo_next, halo_prev = self.exchange(to_prev, to_next)
            self.apply_part(x, out, halo_next, halo_prev, 2, flags, tau)
            main.wait_stream(self._side)
        else:
            halo_next, halo_prev = self.exchange(to_prev, to_next)
            self.apply_part(x, out, halo_next, halo_prev, 0, flags, tau)
        return out


class Communicator:
    """NCCL communicator of the distributed solver (`mgt_comm_*`, NCCL loaded
    at run time by the native library).  Rank 0's 128-byte unique id is
    broadcast over `group`; without an initialised process group this is the
    single-rank communicator (no NCCL calls are made)."""

    def __init__(self, group=None):
        from . import _lib
        self._lib = _lib
        if dist.is_available() and dist.is_initialized():
            self.rank, self.world = dist.get_rank(group), dist.get_world_size(group)
        else:
            self.rank, self.world = 0, 1
        uid = (_lib.ct.c_char * 128)()
        if self.world > 1:
            if self.rank == 0:
                _lib.check(_lib.lib().mgt_comm_unique_id(uid), "nccl unique id")
            box = [bytes(uid)]
            src = dist.get_global_rank(group, 0) if group is not None else 0
            dist.broadcast_object_list(box, src=src, group=group)
            uid = (_lib.ct.c_char * 128).from_buffer_copy(box[0])
        self.handle = _lib.ct.c_void_p()
        _lib.check(_lib.lib().mgt_comm_create(_lib.ct.byref(self.handle), uid, self.world, self.rank),
                   "communicator")

    def allreduce_(self, t):
        """In-place sum over ranks of a float64 CUDA tensor (stream-ordered)."""
        from ._device import ptr, stream_ptr
        self._lib.check(self._lib.lib().mgt_comm_allreduce(self.handle, ptr(t), t.numel(), stream_ptr()),
                        "allreduce")
        return t

    def __del__(self):
        h = getattr(self, "handle", None)
        if h is not None and h.value:
            try:
                self._lib.lib().mgt_comm_destroy(h)
            except Exception:
                pass
            self.handle = None


class SlabBiCGStab:
    """Distributed BiCGStab on a t-slab operator (`mgt_bicgstab_solve_slab`):
    rank-local fields (n, 12, V_local), one all-reduce per reduction point,
    a face exchange before every stencil pass.  Reports, relative residuals
    and the quadratic forms z^H A^-1 z are global (identical on every rank)."""

    MAX_GROUP = 4

    def __init__(self, slab_op, comm, flags=0, tau=0.0):
        from . import _lib
        from ._device import device
        if slab_op.prec != 64:
            raise ValueError("the Krylov solver runs in complex128")
        if comm.world != slab_op.world:
            raise ValueError(f"communicator has {comm.world} ranks, slab decomposition {slab_op.world}")
        self.op, self.comm, self.flags, self.tau = slab_op, comm, int(flags), float(tau)
        self._lib = _lib
        nbytes = _lib.lib().mgt_bicgstab_slab_workspace_bytes(slab_op._handle, self.MAX_GROUP)
        self.workspace = torch.empty(int(nbytes), dtype=torch.uint8, device=device())

    def solve_native(self, b, tol, max_iter, x=None, want_dot=False):
        import ctypes as ct
        from ._device import ptr, stream_ptr
        from .krylov import REASONS, SolveReport
        n = b.shape[0]
        b = b.contiguous()
        x = torch.empty_like(b) if x is None else x
        rep = (ct.c_int64 * (4 * n))()
        rel = (ct.c_double * n)()
        dots = (ct.c_double * (2 * n))() if want_dot else None
        self._lib.check(self._lib.lib().mgt_bicgstab_solve_slab(
            self.op._handle, self.comm.handle, ptr(b), ptr(x), n, self.flags, self.tau, float(tol), int(max_iter),
            ptr(self.workspace), rep, rel, dots, stream_ptr()), "distributed bicgstab")
        reports = []
        for r in range(n):
            it, mv, conv, reason = rep[4 * r:4 * r + 4]
            reports.append(SolveReport(int(it), float(rel[r]), bool(conv), int(mv),
                                       "" if conv else REASONS.get(int(reason), "max_iter")))
        dv = np.array([complex(dots[2 * r], dots[2 * r + 1]) for r in range(n)]) if want_dot else None
        return x, reports, dv


def slab_hutchinson(solver, n_noise, kind="rademacher", seed=0, tol=1e-8, max_iter=2000):
    """Hutchinson (trace.py:122-132) with t-sharded solves: every rank holds
    its slab of each probe (`noise_native_slab`, bit-identical to the global
    probe) and `SlabBiCGStab` returns the GLOBAL quadratic forms, so the
    samples and the finished estimate are identical on every rank."""
    from .probing import noise_native_slab
    op = solver.op
    samples, inversions = [], 0
    for j0 in range(0, n_noise, SlabBiCGStab.MAX_GROUP):
        j1 = min(n_noise, j0 + SlabBiCGStab.MAX_GROUP)
        z = noise_native_slab(op.global_geometry, op.t_begin, op.t_local, [seed + j for j in range(j0, j1)], kind)
        _, reps, q = solver.solve_native(z, tol, max_iter, want_dot=True)
        samples.extend(q)
        inversions += len(reps)
    return finish(0.0, np.array(samples, dtype=np.complex128), inversions)


def distributed_hutchinson(inv_op, geometry, n_noise, kind="rademacher", seed=0, group=None):
    """Probe-sharded `hutchinson` (trace.py:122-132) over the ranks of `group`."""
    from .probing import build_probe_set
    from .trace import hutchinson

    def local(j0, j1):
        if j1 == j0:  # more ranks than probes
            return finish(0.0, np.zeros(0, dtype=np.complex128), 0)
        ps = build_probe_set(geometry, 12, j1 - j0, hp_count=1, dilution=False, kind=kind, seed=seed + j0)
        return hutchinson(inv_op, ps)

    return sharded_estimate(local, n_noise, group, device=torch.device("cuda", torch.cuda.current_device()))
