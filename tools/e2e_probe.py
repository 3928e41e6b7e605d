#!/usr/bin/env python
"""Host-buffer apply throughput vs chunk count (pinned buffers)."""
import os, sys, time
ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import numpy as np, torch
import paper_1909_12234_b200 as M
dims = tuple(int(v) for v in (sys.argv[1] if len(sys.argv) > 1 else "48x48x48x96").split("x"))
geo = M.LatticeGeometry(dims, "antiperiodic")
op = M.build_wilson(M.generate_gauge(geo, "su3", eps=0.2, seed=0), 0.1)
xh = torch.randn(op.dim, dtype=torch.complex128).pin_memory()
yh = torch.empty_like(xh).pin_memory()
ref = op.from_native(op.apply_native(op.to_native(xh.cuda())))[0].cpu()
for nch in (1, 4, 8, 16, 24, 48):
    op.apply_host(xh, out=yh, nchunks=nch)
    assert torch.equal(yh, ref), nch
    t0 = time.perf_counter()
    for _ in range(3):
        op.apply_host(xh, out=yh, nchunks=nch)
    el = (time.perf_counter() - t0) / 3
    print(f"nchunks={nch:3d} {el*1e3:8.2f} ms  e2e {960*geo.site_count/el/1e9:7.1f} GB/s  "
          f"PCIe {2*op.dim*16/el/1e9:6.1f} GB/s (both directions)", flush=True)
y2 = op.apply(np.asarray(xh.numpy()))
assert np.array_equal(y2, ref.numpy())
print("numpy path ok")

# raw PCIe ceilings with the same pinned buffers
dev = torch.empty(op.dim, dtype=torch.complex128, device="cuda")
dev2 = torch.empty_like(dev)
s1, s2 = torch.cuda.Stream(), torch.cuda.Stream()
nb = op.dim * 16
for name, fn in [("H2D", lambda: dev.copy_(xh, non_blocking=True)),
                 ("D2H", lambda: yh.copy_(dev2, non_blocking=True))]:
    fn(); torch.cuda.synchronize()
    t0 = time.perf_counter()
    for _ in range(3):
        fn()
    torch.cuda.synchronize()
    el = (time.perf_counter() - t0) / 3
    print(f"{name} alone: {el*1e3:7.2f} ms  {nb/el/1e9:6.1f} GB/s", flush=True)
torch.cuda.synchronize()
t0 = time.perf_counter()
for _ in range(3):
    with torch.cuda.stream(s1):
        dev.copy_(xh, non_blocking=True)
    with torch.cuda.stream(s2):
        yh.copy_(dev2, non_blocking=True)
torch.cuda.synchronize()
el = (time.perf_counter() - t0) / 3
print(f"H2D || D2H: {el*1e3:7.2f} ms  {2*nb/el/1e9:6.1f} GB/s total", flush=True)
