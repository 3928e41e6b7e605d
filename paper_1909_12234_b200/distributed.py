"""Multi-GPU: probe sharding and t-slab domain decomposition.

One process per GPU (`torch.distributed`, NCCL over NVLink/NVSwitch on the
B200 box; gloo works for the host-side logic on CPU).

Probe sharding: Hutchinson probes are independent
(trace.py:100-107).  Rank r takes the contiguous probe block
[r s / W, (r+1) s / W); probe j keeps its reference seed seed0 + j
(probing.py:155), so the union of the shards is exactly the single-process
probe set.  The only collective is one all-gather of the per-probe complex
samples at the end; every rank then reduces them in GLOBAL probe order with
the reference's `_finish` arithmetic (trace.py:73-92), so a sharded estimate
is bitwise equal to the single-GPU one.

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

    def __init__(self, gauge, mass, rank, world, prec=64, recon=12, group=None, local_links=None):
        """gauge: the GLOBAL GaugeField (the slab's links are cut out of it),
        or a (geometry, None) stand-in together with `local_links`, the slab's
        own links in local reference layout (when no rank holds the global
        field)."""
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

    def apply_native(self, x, out=None, flags=0, tau=0.0, overlap=True):
        x = x.contiguous()
        out = torch.empty_like(x) if out is None else out
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
