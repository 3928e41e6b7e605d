"""SU(3) gauge links U_mu(x) = expm(i eps H) (BASELINE.json configs).

The reference only generates U(1) phases (`lattice.py:126-144`); the SU(3)
generator is defined here (and restated identically in `oracle/wilson4d.py`):

* draws: `rng = numpy.random.default_rng(seed)`; `rng.normal(size=(V, 4, 8))`
  over sites in REFERENCE order (t fastest), drawn in chunks of sites (the
  numpy stream is chunk-invariant);
* the 8 normals n0..n7 of link (x, mu) give the traceless Hermitian
  H01 = (n0 + i n1)/sqrt2, H02 = (n2 + i n3)/sqrt2, H12 = (n4 + i n5)/sqrt2,
  diag = (n6/sqrt2 + n7/sqrt6, -n6/sqrt2 + n7/sqrt6, -2 n7/sqrt6);
* U = expm(i eps H) is computed on the GPU (`mgt_su3_expm`, scaling and
  squaring).  The host draw is setup, like the reference's own generator.

Links are kept on the device in the reference layout (V, 4, 3, 3) complex128;
each operator handle builds its own native (SoA, t-slowest) copy.
"""

from dataclasses import dataclass

import numpy as np
import torch

from . import _lib
from ._device import device, ptr, stream_ptr


@dataclass
class GaugeField:
    geometry: object
    links: torch.Tensor  # (V, 4, 3, 3) complex128, CUDA, reference site order
    kind: str = "su3"
    eps: float = 0.0
    seed: int = 0

    def validate(self, tol=1e-8):
        U = self.links
        eye = torch.eye(3, dtype=U.dtype, device=U.device)
        err = (U @ U.conj().transpose(-1, -2) - eye).abs().max().item()
        if err > tol:
            raise ValueError(f"non-unitary link, |U U^dag - 1| = {err:.3e}")


def generate_gauge(geometry, kind="su3", eps=0.2, seed=0, chunk_sites=1 << 20):
    """'unit' (free field) or 'su3' (expm(i eps H), seeded)."""
    if geometry.ndim != 4:
        raise ValueError("SU(3) gauge fields are 4D")
    V = geometry.site_count
    dev = device()
    if kind == "unit":
        links = torch.zeros((V, 4, 3, 3), dtype=torch.complex128, device=dev)
        idx = torch.arange(3, device=dev)
        links[:, :, idx, idx] = 1.0
        return GaugeField(geometry, links, kind="unit")
    if kind != "su3":
        raise ValueError(f"unknown gauge kind {kind!r}")
    links = torch.empty((V, 4, 3, 3), dtype=torch.complex128, device=dev)
    rng = np.random.default_rng(seed)
    # standard_normal into a pinned buffer: the same stream and values as
    # rng.normal(size=(n, 4, 8)) (loc 0, scale 1), without temporaries
    buf = torch.empty(min(chunk_sites, V) * 32, dtype=torch.float64).pin_memory()
    for s0 in range(0, V, chunk_sites):
        n = min(chunk_sites, V - s0)
        hb = buf[:n * 32]
        rng.standard_normal(out=hb.numpy())
        normals = hb.to(dev, non_blocking=True)
        _lib.check(_lib.lib().mgt_su3_expm(float(eps), ptr(normals), s0, n, ptr(links), stream_ptr()),
                   "generate_gauge")
        torch.cuda.current_stream().synchronize()
    return GaugeField(geometry, links, kind="su3", eps=float(eps), seed=int(seed))


def gauge_from_array(geometry, links_ref, kind="array"):
    """Wrap host links (V, 4, 3, 3) complex (reference order) as a GaugeField."""
    arr = np.ascontiguousarray(np.asarray(links_ref, dtype=np.complex128))
    if arr.shape != (geometry.site_count, 4, 3, 3):
        raise ValueError(f"links shape {arr.shape} != {(geometry.site_count, 4, 3, 3)}")
    return GaugeField(geometry, torch.from_numpy(arr).to(device()), kind=kind)
