#!/usr/bin/env python
"""In-situ kernel timeline of one mixed even-odd BiCGStab solve (CUPTI via
torch.profiler): per-kernel time, the idle time between kernels on the
stream and the largest gaps.  python tools/solver_timeline.py 32x32x32x32 [n_rhs]"""
import collections
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)


def main():
    import torch
    from torch.profiler import ProfilerActivity, profile
    import paper_1909_12234_b200 as M
    from paper_1909_12234_b200 import krylov as K
    dims = tuple(int(v) for v in sys.argv[1].split("x"))
    g = int(sys.argv[2]) if len(sys.argv) > 2 else 4
    geo = M.LatticeGeometry(dims, "antiperiodic")
    op = M.build_wilson(M.generate_gauge(geo, "su3", eps=0.2, seed=0), 0.1)
    probes = M.build_probe_set(geo, 12, g, dilution=False, kind="rademacher", seed=0)
    z = probes.noise_native(0, g)
    solver = K.BiCGStab(op, max_rhs=max(4, g))
    for _ in range(2):
        solver.solve_native(z, 1e-8, 4000, want_dot=True, mixed=True)
    torch.cuda.synchronize()
    import time
    time.sleep(float(os.environ.get("IDLE_S", "0")))  # IDLE_S=3: start the profiled solve from an idle (cool) GPU
    with profile(activities=[ProfilerActivity.CUDA, ProfilerActivity.CPU]) as prof:
        x, reps, q = solver.solve_native(z, 1e-8, 4000, want_dot=True, mixed=True)
        torch.cuda.synchronize()
    ev = [e for e in prof.events() if e.device_type == torch.autograd.DeviceType.CUDA]
    ev.sort(key=lambda e: e.time_range.start)
    t0, t1 = ev[0].time_range.start, max(e.time_range.end for e in ev)
    busy = sum(e.time_range.end - e.time_range.start for e in ev)
    print(f"{sys.argv[1]} rhs={g} iterations={[r.iterations for r in reps]} span={(t1 - t0) / 1e3:.2f} ms "
          f"busy={busy / 1e3:.2f} ms idle={(t1 - t0 - busy) / 1e3:.2f} ms events={len(ev)}")
    agg = collections.defaultdict(lambda: [0, 0.0])
    for e in ev:
        a = agg[e.name.split("(")[0][:60]]
        a[0] += 1
        a[1] += e.time_range.end - e.time_range.start
    for name, (n, t) in sorted(agg.items(), key=lambda kv: -kv[1][1])[:16]:
        print(f"  {n:5d} x {t / n:9.1f} us = {t / 1e3:8.2f} ms  {name}")
    for key in ("bi_k1_eo", "bi_eo_first<4, 12, float", "bi_k4v"):
        seq = [round((e.time_range.end - e.time_range.start)) for e in ev if key in e.name]
        print(f"  {key} durations in launch order (us): {seq}")
    gaps = []
    for a, b in zip(ev[:-1], ev[1:]):
        gaps.append((b.time_range.start - a.time_range.end, a.name.split("(")[0][:30], b.name.split("(")[0][:30]))
    gaps.sort(reverse=True)
    print("largest gaps (us):")
    for gp, a, b in gaps[:12]:
        print(f"  {gp:8.1f}  {a} -> {b}")
    hist = collections.Counter(min(int(gp // 2) * 2, 40) for gp, _, _ in gaps)
    print("gap histogram (us bucket: count):", sorted(hist.items()))


if __name__ == "__main__":
    main()
