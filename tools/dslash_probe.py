#!/usr/bin/env python
"""Run the fp64 dslash on one lattice a few times (for ncu metric probes):
  python tools/dslash_probe.py 48x48x48x96 [recon] [n_rhs] [steps]"""
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)


def main():
    import torch
    import paper_1909_12234_b200 as M
    dims = tuple(int(v) for v in sys.argv[1].split("x"))
    recon = int(sys.argv[2]) if len(sys.argv) > 2 else 12
    nrhs = int(sys.argv[3]) if len(sys.argv) > 3 else 1
    steps = int(sys.argv[4]) if len(sys.argv) > 4 else 5
    geo = M.LatticeGeometry(dims, "antiperiodic")
    op = M.build_wilson(M.generate_gauge(geo, "su3", eps=0.2, seed=0), 0.1, recon=recon)
    x = torch.randn((nrhs, 12, geo.site_count), dtype=torch.complex128, device="cuda")
    y = torch.empty_like(x)
    for _ in range(3):
        op.apply_native(x, out=y)
    torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(True), torch.cuda.Event(True)
    e0.record()
    for _ in range(steps):
        op.apply_native(x, out=y)
    e1.record()
    torch.cuda.synchronize()
    ms = e0.elapsed_time(e1) / steps
    print(f"{sys.argv[1]} recon={recon} nrhs={nrhs} slab_mb={os.environ.get('MGT_SLAB_MB', 'default')} "
          f"ms={ms:.4f} GBps_alg={960 * geo.site_count * nrhs / ms / 1e6:.0f}")


if __name__ == "__main__":
    main()
