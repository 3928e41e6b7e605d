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


def seed_words(seeds):
    """(n, 4) uint64 {state_hi, state_lo, inc_hi, inc_lo} per numpy seed."""
    out = np.empty((len(seeds), 4), dtype=np.uint64)
    m = (1 << 64) - 1
    for i, s in enumerate(seeds):
        st = np.random.PCG64(int(s)).state["state"]
        state, inc = int(st["state"]), int(st["inc"])
        out[i] = (state >> 64, state & m, inc >> 64, inc & m)
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

    def __init__(self, geometry, dof, n_noise, dilution=False, kind="rademacher", seed=0):
        if dof != 12:
            raise ValueError("the 4D SU(3) operator has dof = 12")
        self.geometry = geometry
        self.dof = dof
        self.n_noise = int(n_noise)
        self.dilution = bool(dilution)
        self.kind = kind
        self.seed = int(seed)
        self.basis = ProbingBasis(geometry, dof if dilution else 1, 1)

    @property
    def sample_count(self):
        return self.n_noise

    @property
    def slots_per_group(self):
        return self.dof if self.dilution else 1

    @property
    def slot_count(self):
        return self.n_noise * self.slots_per_group

    def weights(self):
        return np.ones(self.slots_per_group)

    def noise_native(self, j0, j1):
        """Noise fields of groups j0..j1-1, native layout."""
        return noise_native(self.geometry, [self.seed + j for j in range(j0, j1)], self.kind)

    def slots_native(self, j):
        """All slots of group j, native layout (n_slots, 12, V)."""
        z = self.noise_native(j, j + 1)
        if not self.dilution:
            return z
        out = torch.zeros((self.dof,) + tuple(z.shape[1:]), dtype=z.dtype, device=z.device)
        for p in range(self.dof):
            out[p, p] = z[0, p]
        return out

    @property
    def groups(self):
        """Reference-compatible host groups (materialises every slot)."""
        N = self.geometry.site_count * self.dof
        out = []
        for j in range(self.n_noise):
            z = noise_ref(N, [self.seed + j], self.kind)[0].cpu().numpy()
            if self.dilution:
                slots = np.zeros((self.dof, N), dtype=np.complex128)
                for p in range(self.dof):
                    slots[p, p::self.dof] = z[p::self.dof]
            else:
                slots = z[None, :]
            out.append(ProbeGroup(slots, self.weights(), NoiseVector(self.kind, self.seed + j, z)))
        return out


def build_probe_set(geometry, dof, n_noise, hp_count=1, dilution=True, kind="z4", seed=0):
    """Reference `build_probe_set` (probing.py:146-165) on the GPU.
    Hierarchical probing (hp_count > 1) is SURVEY.md row f2, not built yet."""
    if hp_count != 1:
        raise NotImplementedError("hierarchical probing (hp_count > 1) is not in the GPU hot path yet")
    return ProbeSet(geometry, dof, n_noise, dilution=dilution, kind=kind, seed=seed)
