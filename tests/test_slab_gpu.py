"""t-slab decomposition of the Wilson operator on one GPU: W slab operators
(one per emulated rank) exchange their spin-projected faces through device
copies instead of NCCL, and the stitched result must equal the full-lattice
apply to 1e-13 (fp64).  The NCCL/gloo ring exchange itself is covered by
tests/test_distributed_cpu.py."""

import numpy as np
import pytest
import torch

pytestmark = pytest.mark.gpu


def _setup(dims, eps=0.3, boundary="antiperiodic"):
    import paper_1909_12234_b200 as M
    geo = M.LatticeGeometry(dims, boundary)
    gauge = M.generate_gauge(geo, "su3", eps=eps, seed=4)
    return M, geo, gauge


def _rel(a, b):
    return (torch.linalg.vector_norm(a - b) / torch.linalg.vector_norm(b)).item()


@pytest.mark.parametrize("world", [2, 4])
@pytest.mark.parametrize("recon", [18, 12])
@pytest.mark.parametrize("flags,tau", [(0, 0.0), (1, 0.0), (4, 0.3), (2, -0.2)])
def test_emulated_ranks_match_full_operator(cuda, world, recon, flags, tau):
    from paper_1909_12234_b200.distributed import SlabWilsonOperator
    dims = (4, 4, 6, 16)
    M, geo, gauge = _setup(dims)
    full = M.build_wilson(gauge, 0.1, recon=recon)
    x = torch.randn((3, 12, geo.site_count), dtype=torch.complex128, device=cuda)
    y_ref = full.apply_native(x, flags=flags, tau=tau)
    ops = [SlabWilsonOperator(gauge, 0.1, r, world, recon=recon) for r in range(world)]
    S3 = ops[0].S3
    Tl = ops[0].t_local
    xs = [x[:, :, r * Tl * S3:(r + 1) * Tl * S3].contiguous() for r in range(world)]
    faces = [op.pack(xl, flags, tau) for op, xl in zip(ops, xs)]
    ys = []
    for r, (op, xl) in enumerate(zip(ops, xs)):
        halo_next = faces[(r + 1) % world][0]
        halo_prev = faces[(r - 1) % world][1]
        out = torch.empty_like(xl)
        # interior and boundary separately, as the overlapped path does
        op.apply_part(xl, out, None, None, 1, flags, tau)
        op.apply_part(xl, out, halo_next, halo_prev, 2, flags, tau)
        ys.append(out)
    y = torch.cat(ys, dim=2)
    assert _rel(y, y_ref) < 1e-13


@pytest.mark.parametrize("boundary", ["periodic", "antiperiodic"])
def test_single_rank_slab_is_full_operator(cuda, boundary):
    import torch.distributed as dist
    from paper_1909_12234_b200.distributed import SlabWilsonOperator
    dims = (4, 6, 4, 8)
    M, geo, gauge = _setup(dims, boundary=boundary)
    full = M.build_wilson(gauge, 0.1, recon=12)
    slab = SlabWilsonOperator(gauge, 0.1, 0, 1, recon=12)
    slab.exchange = lambda a, b: (a, b)  # world = 1: my own faces come back
    x = torch.randn((2, 12, geo.site_count), dtype=torch.complex128, device=cuda)
    for overlap in (True, False):
        assert _rel(slab.apply_native(x, overlap=overlap), full.apply_native(x)) < 1e-13


def test_plain_apply_rejects_slab_handle(cuda):
    from paper_1909_12234_b200 import _lib
    from paper_1909_12234_b200._device import ptr, stream_ptr
    from paper_1909_12234_b200.distributed import SlabWilsonOperator
    M, geo, gauge = _setup((4, 4, 4, 8))
    slab = SlabWilsonOperator(gauge, 0.1, 0, 2, recon=12)
    x = torch.zeros((1, 12, slab.volume), dtype=torch.complex128, device=cuda)
    rc = _lib.lib().mgt_wilson_apply(slab._handle, ptr(x), ptr(torch.empty_like(x)), 1, 0, 0.0, stream_ptr())
    with pytest.raises(ValueError, match="slab"):
        _lib.check(rc)


@pytest.mark.parametrize("world", [1, 2, 4])
@pytest.mark.parametrize("dims", [(4, 4, 6, 16), (4, 6, 4, 8)])
def test_peer_window_transport_emulated(cuda, world, dims):
    """p2p transport (pack kernel stores the faces straight into the
    neighbours' receive windows): W in-process ranks wired without IPC,
    every rank posts (pack + interior) before any rank completes (boundary),
    as the barrier orders it across processes.  Three applies per rank with
    changing inputs exercise the parity double buffering; the stitched result
    must equal the full operator and be bitwise equal to the copy-exchange
    path."""
    from paper_1909_12234_b200.distributed import SlabWilsonOperator
    M, geo, gauge = _setup(dims)
    if dims[3] // world < 2:
        pytest.skip("slab needs >= 2 slices")
    full = M.build_wilson(gauge, 0.1, recon=12)
    ops = [SlabWilsonOperator(gauge, 0.1, r, world, recon=12, transport="p2p", max_rhs=4, connect=False)
           for r in range(world)]
    SlabWilsonOperator.connect_local(ops)
    ref = [SlabWilsonOperator(gauge, 0.1, r, world, recon=12) for r in range(world)]
    S3, Tl = ops[0].S3, ops[0].t_local
    for it, (n, flags, tau) in enumerate([(3, 0, 0.0), (1, 1, 0.0), (4, 4, 0.25)]):
        x = torch.randn((n, 12, geo.site_count), dtype=torch.complex128, device=cuda)
        xs = [x[:, :, r * Tl * S3:(r + 1) * Tl * S3].contiguous() for r in range(world)]
        outs = [torch.empty_like(xl) for xl in xs]
        for op, xl, o in zip(ops, xs, outs):
            op.post(xl, o, flags, tau)
        for op, xl, o in zip(ops, xs, outs):
            op.complete(xl, o, flags, tau)
        y = torch.cat(outs, dim=2)
        assert _rel(y, full.apply_native(x, flags=flags, tau=tau)) < 1e-13
        faces = [op.pack(xl, flags, tau) for op, xl in zip(ops, xs)]
        for r, (op, xl) in enumerate(zip(ref, xs)):
            o = torch.empty_like(xl)
            op.apply_part(xl, o, faces[(r + 1) % world][0], faces[(r - 1) % world][1], 0, flags, tau)
            assert torch.equal(o, outs[r]), (it, r)
    with pytest.raises(ValueError, match="capacity"):
        ops[0].post(torch.zeros((5, 12, ops[0].volume), dtype=torch.complex128, device=cuda),
                    torch.empty((5, 12, ops[0].volume), dtype=torch.complex128, device=cuda))


def test_peer_window_single_rank_apply_native(cuda):
    """world = 1 with the p2p transport: the window wraps to itself."""
    from paper_1909_12234_b200.distributed import SlabWilsonOperator
    M, geo, gauge = _setup((4, 4, 4, 8))
    full = M.build_wilson(gauge, 0.1, recon=12)
    slab = SlabWilsonOperator(gauge, 0.1, 0, 1, recon=12, transport="p2p")
    x = torch.randn((2, 12, geo.site_count), dtype=torch.complex128, device=cuda)
    for _ in range(3):
        assert _rel(slab.apply_native(x), full.apply_native(x)) < 1e-13


def test_distributed_solver_single_rank_matches_full_solver(cuda):
    """mgt_bicgstab_solve_slab on a one-rank communicator: every reduction
    goes through the all-reduce/finisher path and every stencil pass through
    the face exchange (the ring closes on the rank), so the distributed code
    path runs end to end; it must agree with the single-GPU full-system
    solver and meet the full-residual test against the oracle matrix."""
    from oracle import wilson4d as W
    from paper_1909_12234_b200.distributed import Communicator, SlabBiCGStab, SlabWilsonOperator
    from paper_1909_12234_b200 import krylov as K
    dims = (4, 4, 6, 8)
    M, geo, gauge = _setup(dims, eps=0.2)
    full = M.build_wilson(gauge, 0.1, recon=12)
    slab = SlabWilsonOperator(gauge, 0.1, 0, 1, recon=12)
    comm = Communicator()
    ds = SlabBiCGStab(slab, comm)
    g = torch.Generator(device="cuda").manual_seed(11)
    b = torch.randn((3, 12, geo.site_count), dtype=torch.complex128, device=cuda, generator=g)
    x, reps, q = ds.solve_native(b, 1e-10, 2000, want_dot=True)
    xf, repf, qf = K.BiCGStab(full).solve_native(b, 1e-10, 2000, want_dot=True, even_odd=False)
    A = W.build_wilson4d_csr(gauge.links.cpu().numpy(), dims, 0.1)
    X = full.from_native(x).cpu().numpy()
    B = full.from_native(b).cpu().numpy()
    for j in range(3):
        assert reps[j].converged and abs(reps[j].iterations - repf[j].iterations) <= 1
        assert np.linalg.norm(B[j] - A @ X[j]) <= 1.01e-10 * np.linalg.norm(B[j])
        assert abs(q[j] - np.vdot(B[j], X[j])) < 1e-12 * abs(q[j])
        assert abs(q[j] - qf[j]) < 1e-9 * abs(qf[j])
    assert _rel(x, xf) < 1e-8
    buf = torch.arange(5, dtype=torch.float64, device=cuda)
    assert torch.equal(comm.allreduce_(buf.clone()), buf)  # one rank: identity
    with pytest.raises(ValueError):
        SlabBiCGStab(SlabWilsonOperator(gauge, 0.1, 0, 2, recon=12), comm)


def test_slab_noise_is_the_global_probe_restricted(cuda):
    from paper_1909_12234_b200.probing import noise_native, noise_native_slab
    M, geo, gauge = _setup((4, 6, 4, 12))
    S3 = 4 * 6 * 4
    for kind in ("rademacher", "z4"):
        full = noise_native(geo, [5, 9, 123], kind)
        for t0, tl in ((0, 12), (0, 3), (3, 6), (9, 3)):
            sl = noise_native_slab(geo, t0, tl, [5, 9, 123], kind)
            assert torch.equal(torch.view_as_real(sl), torch.view_as_real(full[:, :, t0 * S3:(t0 + tl) * S3]))


def test_slab_hutchinson_single_rank(cuda):
    """t-sharded Hutchinson on one rank == the single-GPU Hutchinson (full
    system solves) within the solver tolerance; same probes bitwise."""
    from paper_1909_12234_b200.distributed import Communicator, SlabBiCGStab, SlabWilsonOperator, slab_hutchinson
    M, geo, gauge = _setup((4, 4, 4, 8), eps=0.2)
    full = M.build_wilson(gauge, 0.1, recon=12)
    slab = SlabWilsonOperator(gauge, 0.1, 0, 1, recon=12)
    est = slab_hutchinson(SlabBiCGStab(slab, Communicator()), 6, seed=40, tol=1e-10)
    ps = M.build_probe_set(geo, 12, 6, hp_count=1, dilution=False, kind="rademacher", seed=40)
    ref = M.hutchinson(M.TruncatedInverse(full, M.SolveConfig(tol=1e-10)), ps)
    assert est.inversions == 6
    assert np.max(np.abs(est.samples - ref.samples) / np.abs(ref.samples)) < 1e-8
    assert abs(est.mean - ref.mean) < 1e-9 * abs(ref.mean)
