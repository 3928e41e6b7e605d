#!/usr/bin/env python
"""Achieved bandwidth of every hot-path kernel against the measured HBM
peak (MEASURED_PEAKS.json), CUDA-event timed after warm-up, inputs > L2
where the config allows.  Prints one JSON line per kernel; DESIGN.md §3 and
profiles/r01_kernel_rooflines.jsonl are generated from this output."""

import json
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)


def timeit(fn, steps=10, warm=3):
    import torch
    for _ in range(warm):
        fn()
    torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(True), torch.cuda.Event(True)
    e0.record()
    for _ in range(steps):
        fn()
    e1.record()
    torch.cuda.synchronize()
    return e0.elapsed_time(e1) / steps * 1e-3


def main():
    import torch
    import paper_1909_12234_b200 as M
    from paper_1909_12234_b200 import linalg as LA
    from paper_1909_12234_b200 import multigrid as MG
    from paper_1909_12234_b200.distributed import SlabWilsonOperator
    peak = json.load(open(os.path.join(ROOT, "MEASURED_PEAKS.json")))["hbm_gbs"]

    def emit(name, config, seconds, algo_bytes, flops=None):
        d = {"kernel": name, "config": config, "us": seconds * 1e6, "algorithmic_bytes": algo_bytes,
             "GBps": algo_bytes / seconds / 1e9, "frac_hbm": algo_bytes / seconds / 1e9 / peak}
        if flops:
            d["TFLOPs"] = flops / seconds / 1e12
        print(json.dumps(d), flush=True)

    # dslash at the sweep sizes, fp64/fp32, 1 and 4 rhs
    for dims in [(32, 32, 32, 32), (48, 48, 48, 96)]:
        geo = M.LatticeGeometry(dims, "antiperiodic")
        gauge = M.generate_gauge(geo, "su3", eps=0.2, seed=0)
        V = geo.site_count
        for prec in (64, 32):
            op = M.build_wilson(gauge, 0.1, prec=prec)
            w = 8 if prec == 64 else 4
            for nrhs in (1, 4):
                x = torch.randn((nrhs, 12, V), dtype=op.dtype, device="cuda")
                y = torch.empty_like(x)
                t = timeit(lambda: op.apply_native(x, out=y))
                emit(f"wilson_apply fp{prec} nrhs={nrhs}", "x".join(map(str, dims)), t,
                     V * (4 * 18 * w + nrhs * 48 * w), 1368 * V * nrhs)
                del x, y
            if prec == 64 and dims == (48, 48, 48, 96):
                # t-slab apply with halos (one rank's 12-slice slab of an 8-way split)
                import types
                sub = M.LatticeGeometry(dims[:3] + (12,), "antiperiodic")
                g2 = M.generate_gauge(sub, "su3", eps=0.2, seed=1)
                slab = SlabWilsonOperator(types.SimpleNamespace(geometry=geo), 0.1, 0, 8, local_links=g2.links)
                slab.exchange = lambda a, b: (a, b)
                xs = torch.randn((1, 12, slab.volume), dtype=torch.complex128, device="cuda")
                ys = torch.empty_like(xs)
                t = timeit(lambda: slab.apply_native(xs, out=ys))
                emit("slab apply (pack + interior||boundary), fp64", "48^3x12 slab of 48^3x96", t,
                     slab.volume * 960, 1368 * slab.volume)
                fp, fn = slab.pack(xs)
                t = timeit(lambda: slab.pack(xs))
                emit("halo_pack (2 spin-projected faces)", "48^3 faces", t, 2 * slab.S3 * (192 + 96 + 96))
                del slab, xs, ys, g2
            del op
            torch.cuda.empty_cache()
        # probes
        probes = M.build_probe_set(geo, 12, 4, dilution=False, kind="rademacher", seed=0)
        t = timeit(lambda: probes.noise_native(0, 4))
        emit("noise (PCG64 Rademacher, 4 probes)", "x".join(map(str, dims)), t, 4 * V * 192)
        del gauge
        torch.cuda.empty_cache()

    # multigrid kernels at 16^4, 4^4 aggregates, nv = 24
    geo = M.LatticeGeometry((16, 16, 16, 16), "antiperiodic")
    op = M.build_wilson(M.generate_gauge(geo, "su3", eps=0.2, seed=0), 0.1)
    nvs = MG.generate_null_vectors(op, 24, tol=1e-12, max_iter=2, seed=1)
    pro = MG.build_prolongator(nvs, MG.BlockingScheme((4, 4, 4, 4)), layout_op=op)
    N, Nc = op.dim, pro.coarse_dim
    x = torch.randn((4, 12, geo.site_count), dtype=torch.complex128, device="cuda")
    for n in (1, 4):
        t = timeit(lambda: pro.restrict_native(x[:n]))
        emit(f"restrict P^H x (n={n})", "16^4 nv=24", t, 16 * (24 * N + n * N + n * Nc))
        xc = pro.restrict_native(x[:n])
        t = timeit(lambda: pro.prolong_native(xc))
        emit(f"prolong P xc (n={n})", "16^4 nv=24", t, 16 * (24 * N + n * N + n * Nc))
    coarse = MG.build_coarse_operator(op, pro)
    xc = pro.restrict_native(x)
    t = timeit(lambda: coarse.apply_native(xc))
    emit("coarse apply (4 rhs)", "4^4 coarse, 48 dof", t, 16 * (9 * Nc * 48 + 2 * 4 * Nc), 8 * 9 * 48 * Nc * 4)
    # projections, k = 64 vectors at 16^4
    U = torch.randn((64, 12, geo.site_count), dtype=torch.complex128, device="cuda")
    for s in (1, 4, 128):
        X = torch.randn((s, 12, geo.site_count), dtype=torch.complex128, device="cuda")
        t = timeit(lambda: LA.vhx(U, X))
        emit(f"V^H X (k=64, s={s})", "16^4", t, 16 * N * (64 + s), 8 * N * 64 * s)
        H = LA.vhx(U, X)
        t = timeit(lambda: LA.sub_vh(U, H, X))
        emit(f"X - V H (k=64, s={s})", "16^4", t, 16 * N * (64 + 2 * s), 8 * N * 64 * s)
        del X
    # one BiCGStab iteration (model 4608 B/site per rhs) from a 16^4 / 32^4 solve
    from paper_1909_12234_b200 import krylov as K
    for dims in [(16, 16, 16, 16), (32, 32, 32, 32)]:
        g2 = M.LatticeGeometry(dims, "antiperiodic")
        o2 = M.build_wilson(M.generate_gauge(g2, "su3", eps=0.2, seed=0), 0.1)
        z = M.build_probe_set(g2, 12, 4, dilution=False, kind="rademacher", seed=0).noise_native(0, 4)
        solver = K.BiCGStab(o2)
        import time
        # full system: 4608 B/site/rhs per iteration; even-odd Schur system:
        # 2 x (first half 480 + second half 576) + 15 parity-field streams x 96
        # = 3552 B per full site per rhs
        # mixed: fp32 inner iterations stream half of the even-odd bytes
        # (1776 B per full site per rhs); the fp64 residual recomputations and
        # corrections are inside the whole-solve time
        for eo, mixed, model, name in [(False, False, 4608, "full"), (True, False, 3552, "even-odd Schur"),
                                       (True, True, 1776, "mixed even-odd Schur, fp32 inner")]:
            solver.solve_native(z, 1e-8, 2000, even_odd=eo, mixed=mixed)
            torch.cuda.synchronize()
            t0 = time.perf_counter()
            _, reps, _ = solver.solve_native(z, 1e-8, 2000, even_odd=eo, mixed=mixed)
            torch.cuda.synchronize()
            el = time.perf_counter() - t0
            its = sum(r.iterations for r in reps) / 4
            emit(f"BiCGStab iteration, {name} (4 rhs, whole solve / {its:g} iterations)", "x".join(map(str, dims)),
                 el / its, model * g2.site_count * 4)


if __name__ == "__main__":
    main()
