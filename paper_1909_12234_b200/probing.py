"""Probe vectors generated on the GPU, bit-exact with the reference's numpy
draws.

Mirrors `mgtrace.probing` (`/root/reference/pkg/src/mgtrace/probing.py`):
`make_noise` (`:94-107`), `ProbeGroup` / `ProbeSet` (`:120-143`) and
`build_probe_set` (`:146-165`).  Rademacher and Z4 noise come from the
`mgt_noise` kernel: numpy PCG64 (XSL-RR 128/64) streams, seeded on the host
with numpy's own SeedSequence (`PCG64(seed).state`), jumped ahead per site on
the device.  Probe j of a set uses seed `seed0 + j` (`probing.py:155`).
Gaussian noise (not a BASELINE probe kind) is drawn with numpy exactly as the
reference does.
"""

import functools
from dataclasses import dataclass

import numpy as np
import torch

from . import _lib
from ._device import device, ptr, stream_ptr

KINDS = {"rademacher": 0, "z4": 1}


@dataclass
class NoiseVector:
    kind: str
    seed: int
    values: object


@functools.lru_cache(maxsize=1 << 16)
def _seed_word(s):
    st = np.random.PCG64(s).state["state"]
    state, inc = int(st["state"]), int(st["inc"])
    m = (1 << 64) - 1
    return (state >> 64, state & m, inc >> 64, inc & m)


def seed_words(seeds):
    """(n, 4) uint64 {state_hi, state_lo, inc_hi, inc_lo} per numpy seed
    (SeedSequence hashing of each seed, cached: the probes of a sweep reuse
    their seeds)."""
    out = np.empty((len(seeds), 4), dtype=np.uint64)
    for i, s in enumerate(seeds):
        out[i] = _seed_word(int(s))
    return out


def _noise_call(dims, kind, seeds, native, out):
    words = np.ascontiguousarray(seed_words(seeds))
    wp = words.ctypes.data_as(_lib.c_u64_p)
    _lib.check(_lib.lib().mgt_noise(_lib.dims_arg(dims), KINDS[kind], wp, len(seeds), 1 if native else 0,
                                    ptr(out), stream_ptr()), "make_noise")
    return out


def noise_native(geometry, seeds, kind="rademacher", out=None):
    """Noise fields for `seeds` in the native layout, (n, 12, V) complex128."""
    if kind not in KINDS:
        raise ValueError(f"GPU noise kind must be one of {sorted(KINDS)}, got {kind!r}")
    V = geometry.site_count
    if out is None:
        out = torch.empty((len(seeds), 12, V), dtype=torch.complex128, device=device())
    return _noise_call(geometry.dims, kind, seeds, True, out)


def noise_native_slab(geometry, t_begin, t_local, seeds, kind="rademacher", out=None):
    """The global probes for `seeds` restricted to the t-slab
    [t_begin, t_begin + t_local) of `geometry`, in the slab's native layout
    (n, 12, V_slab): bit-identical to those sites of `noise_native`."""
    if kind not in KINDS:
        raise ValueError(f"GPU noise kind must be one of {sorted(KINDS)}, got {kind!r}")
    V = int(np.prod(geometry.dims[:3])) * int(t_local)
    if out is None:
        out = torch.empty((len(seeds), 12, V), dtype=torch.complex128, device=device())
    words = np.ascontiguousarray(seed_words(seeds))
    _lib.check(_lib.lib().mgt_noise_slab(_lib.dims_arg(geometry.dims), int(t_begin), int(t_local), KINDS[kind],
                                         words.ctypes.data_as(_lib.c_u64_p), len(seeds), ptr(out), stream_ptr()),
               "noise (slab)")
    return out


def noise_ref(n, seeds, kind="rademacher"):
    """Noise vectors of length n in reference order, (len(seeds), n) on device."""
    sites = -(-n // 12)
    out = torch.empty((len(seeds), sites * 12), dtype=torch.complex128, device=device())
    _noise_call((1, 1, 1, sites), kind, seeds, False, out)
    return out[:, :n]


def make_noise(n, kind="z4", seed=0):
    """Reference `make_noise` (probing.py:94-107); values is a numpy array."""
    if kind in KINDS:
        return NoiseVector(kind, seed, noise_ref(n, [seed], kind)[0].cpu().numpy())
    if kind == "gaussian":
        rng = np.random.default_rng(seed)
        values = (rng.normal(size=n) + 1j * rng.normal(size=n)) / np.sqrt(2.0)
        return NoiseVector(kind, seed, values)
    raise ValueError(f"unknown noise kind {kind!r}")


def max_hp_level(geometry):
    level = 0
    while all(L % (2 ** (level + 1)) == 0 for L in geometry.dims):
        level += 1
    return level


def _native_coords(geometry):
    """(4, V) coordinates (x0..x3) of the native site order (t slowest)."""
    L0, L1, L2, L3 = geometry.dims
    s = torch.arange(geometry.site_count, device=device(), dtype=torch.int64)
    x2 = s % L2
    x1 = (s // L2) % L1
    x0 = (s // (L2 * L1)) % L0
    x3 = s // (L2 * L1 * L0)
    return torch.stack([x0, x1, x2, x3])


def hp_level(geometry, count):
    """Level of the hierarchical-probing colouring for `count` vectors
    (probing.py:64-77), with the reference's validation."""
    if count < 1 or (count & (count - 1)) != 0:
        raise ValueError(f"hp count must be a power of two, got {count}")
    D = geometry.ndim
    level = 0
    while 2 ** (D * level) < count:
        level += 1
    if level > max_hp_level(geometry) or count > geometry.site_count:
        raise ValueError(f"hp count {count} exceeds the closing colors of {geometry.dims}")
    return level


def hp_vectors_native(geometry, count):
    """The first `count` hierarchical-probing vectors (+/-1 per site) in the
    native site order, (count, V) float64 on the device: colour(x) = Morton
    interleave of (x mod 2^level) bits (probing.py:45-61) and
    h_j(x) = (-1)^popcount(j & colour(x)) (natural-order Hadamard, :78-84)."""
    level = hp_level(geometry, count)
    D = geometry.ndim
    local = _native_coords(geometry) % (2 ** level)
    colors = torch.zeros(geometry.site_count, dtype=torch.int64, device=device())
    for b in range(level):
        for d in range(D):
            colors |= ((local[d] >> b) & 1) << (b * D + d)
    j = torch.arange(count, device=device(), dtype=torch.int64)
    anded = j[:, None] & colors[None, :]
    bits = torch.zeros_like(anded)
    for b in range(max(1, D * level)):
        bits += (anded >> b) & 1
    return torch.where(bits % 2 == 0, 1.0, -1.0).to(torch.float64)


@dataclass
class ProbeGroup:
    slots: object  # (n_slots, N) host array, materialised on demand
    weights: np.ndarray
    noise: NoiseVector = None


@dataclass(frozen=True)
class ProbingBasis:
    geometry: object
    dilution_dim: int
    hp_count: int


class ProbeSet:
    """GPU probe set: n_noise groups, each noise vector j = make_noise(N,
    kind, seed0 + j) decomposed into `dilution_dim` spin-colour slots
    (hp_count = 1).  Slots are generated on the device on demand."""

    def __init__(self, geometry, dof, n_noise, dilution=False, kind="rademacher", seed=0, hp_count=1):
        if dof != 12:
            raise ValueError("the 4D SU(3) operator has dof = 12")
        self.geometry = geometry
        self.dof = dof
        self.n_noise = int(n_noise)
        self.dilution = bool(dilution)
        self.kind = kind
        self.seed = int(seed)
        self.hp_count = int(hp_count)
        self._hp = hp_vectors_native(geometry, self.hp_count) if self.hp_count > 1 else None
        self.basis = ProbingBasis(geometry, dof if dilution else 1, self.hp_count)

    @property
    def sample_count(self):
        return self.n_noise

    @property
    def slots_per_group(self):
        return self.hp_count * (self.dof if self.dilution else 1)

    @property
    def slot_count(self):
        return self.n_noise * self.slots_per_group

    def weights(self):
        return np.full(self.slots_per_group, 1.0 / self.hp_count)

    def noise_native(self, j0, j1):
        """Noise fields of groups j0..j1-1, native layout."""
        return noise_native(self.geometry, [self.seed + j for j in range(j0, j1)], self.kind)

    def slots_native(self, j):
        """All slots of group j in the reference's slot order (hp vector
        outer, dilution pattern inner, probing.py:157-161), native layout
        (n_slots, 12, V): slot = noise (.) kron(hp_h, dilution_p), multiplied
        as complex x (mask + 0i) like numpy (signed zeros included)."""
        z = self.noise_native(j, j + 1)[0]
        V = self.geometry.site_count
        hps = self._hp if self._hp is not None else torch.ones((1, V), dtype=torch.float64, device=z.device)
        zr = torch.view_as_real(z)  # (12, V, 2)
        out = torch.empty((self.slots_per_group, 12, V, 2), dtype=torch.float64, device=z.device)
        s = 0
        for h in range(hps.shape[0]):
            for p in range(self.dof if self.dilution else 1):
                # kron(hp_h, dilution_p) as numpy computes it: hp * pattern
                # (so hp = -1 against a 0 of the pattern gives -0.0)
                pat = torch.ones(12, dtype=torch.float64, device=z.device)
                if self.dilution:
                    pat = (torch.arange(12, device=z.device) == p).to(torch.float64)
                m = hps[h][None, :] * pat[:, None]
                zero = torch.zeros_like(m)
                a, b = zr[..., 0], zr[..., 1]
                out[s, ..., 0] = a * m - b * zero
                out[s, ..., 1] = a * zero + b * m
                s += 1
        return torch.view_as_complex(out)

    @property
    def groups(self):
        """Reference-compatible host groups (materialises every slot)."""
        N = self.geometry.site_count * self.dof
        from .multigrid import _LayoutOnly
        lay = _LayoutOnly(self.geometry)
        out = []
        for j in range(self.n_noise):
            z = noise_ref(N, [self.seed + j], self.kind)[0].cpu().numpy()
            slots = lay.from_native(self.slots_native(j)).cpu().numpy()
            out.append(ProbeGroup(slots, self.weights(), NoiseVector(self.kind, self.seed + j, z)))
        return out


def build_probe_set(geometry, dof, n_noise, hp_count=1, dilution=True, kind="z4", seed=0):
    """Reference `build_probe_set` (probing.py:146-165) on the GPU: noise
    j = make_noise(N, kind, seed + j) decomposed into hp_count hierarchical-
    probing vectors x (dof if dilution else 1) spin-colour patterns, weights
    1 / hp_count."""
    return ProbeSet(geometry, dof, n_noise, dilution=dilution, kind=kind, seed=seed, hp_count=hp_count)
