"""GPU parity of the Wilson-Dirac stencil against the CPU oracle
(oracle/wilson4d.py, the 4D restatement of lattice.py:274-318).

Tolerance (BASELINE.json north_star): A x agrees to 1e-12 relative in fp64;
complex64 is checked against the fp64 oracle at 2e-6 relative."""

import numpy as np
import pytest
import torch

from oracle import wilson4d as W

pytestmark = pytest.mark.gpu


def _gpu():
    import paper_1909_12234_b200 as M
    return M


def _setup(dims, eps, seed=0, mass=0.1, prec=64, recon=18, boundary="antiperiodic"):
    M = _gpu()
    geo = M.LatticeGeometry(dims, boundary)
    gauge = M.generate_gauge(geo, "su3", eps=eps, seed=seed)
    op = M.build_wilson(gauge, mass, prec=prec, recon=recon)
    links = gauge.links.cpu().numpy()
    return M, geo, gauge, op, links


def _rand(n, seed, k=None):
    rng = np.random.default_rng(seed)
    shape = (n,) if k is None else (n, k)
    return (rng.normal(size=shape) + 1j * rng.normal(size=shape)) / np.sqrt(2)


def _rel(a, b):
    return np.linalg.norm(a - b) / np.linalg.norm(b)


@pytest.mark.parametrize("dims,eps", [((4, 4, 4, 4), 0.2), ((4, 6, 8, 10), 0.5), ((2, 4, 2, 6), 0.3)])
def test_links_match_oracle_generator(cuda, dims, eps):
    M, geo, gauge, op, links = _setup(dims, eps, seed=3)
    ref = W.su3_links(dims, eps, 3)
    assert np.abs(links - ref).max() < 1e-13
    gauge.validate(1e-12)


@pytest.mark.parametrize("dims,eps", [((8, 8, 8, 8), 0.2), ((8, 8, 8, 8), 0.5), ((4, 6, 8, 10), 0.2),
                                      ((2, 4, 2, 6), 0.3)])
@pytest.mark.parametrize("recon", [18, 12])
def test_apply_matches_oracle_csr(cuda, dims, eps, recon):
    M, geo, gauge, op, links = _setup(dims, eps, recon=recon)
    A = W.build_wilson4d_csr(links, dims, 0.1)
    x = _rand(op.dim, 11)
    y = op.apply(x)
    assert _rel(y, A @ x) < 1e-12


@pytest.mark.parametrize("boundary", ["periodic", "antiperiodic"])
def test_apply_variants(cuda, boundary):
    dims = (4, 4, 6, 8)
    M, geo, gauge, op, links = _setup(dims, 0.3, boundary=boundary)
    A = W.build_wilson4d_csr(links, dims, 0.1, antiperiodic=boundary == "antiperiodic")
    g5 = W.gamma5_diag(geo.site_count)
    x = _rand(op.dim, 5)
    assert _rel(op.apply(x), A @ x) < 1e-12
    assert _rel(op.apply_dagger(x), A.conj().T @ x) < 1e-12
    assert _rel(op.hermitian_form().apply(x), g5 * (A @ x)) < 1e-12
    assert _rel(op.a_gamma5().apply(x), A @ (g5 * x)) < 1e-12
    assert _rel(op.apply_shifted(0.5, x), A @ x + 0.5j * g5 * x) < 1e-12
    assert np.array_equal(op.apply_shifted(0.0, x), op.apply(x))
    assert _rel(op.shifted(-0.25).apply(x), A @ x - 0.25j * g5 * x) < 1e-12
    # gamma5-Hermiticity (SPEC.md lattice invariants)
    y = _rand(op.dim, 6)
    lhs = np.vdot(y, g5 * op.apply(g5 * x))
    rhs = np.vdot(op.apply(y), x)
    assert abs(lhs - rhs) < 1e-12 * np.linalg.norm(x) * np.linalg.norm(y) * 10


def test_multi_rhs_columns(cuda):
    dims = (4, 4, 4, 8)
    M, geo, gauge, op, links = _setup(dims, 0.2)
    A = W.build_wilson4d_csr(links, dims, 0.1)
    for k in (2, 3, 4, 5, 8):
        X = _rand(op.dim, 20 + k, k)
        Y = op.apply(X)
        assert Y.shape == X.shape
        assert _rel(Y, A @ X) < 1e-12


@pytest.mark.parametrize("prec,recon", [(64, 12), (64, 18), (32, 12)])
def test_interleaved_apply_bitwise_equals_native(cuda, prec, recon):
    """rhs-interleaved multi-rhs apply == native apply column by column,
    bitwise (same per-site arithmetic), every flag variant; interleave
    round trip exact; bad n_rhs rejected."""
    dims = (4, 6, 4, 8)
    M, geo, gauge, op, links = _setup(dims, 0.3, prec=prec, recon=recon)
    g = torch.Generator(device="cuda").manual_seed(5)
    for n in (1, 2, 4, 8, 12):
        x = torch.randn((n, 12, geo.site_count), dtype=op.dtype, device="cuda", generator=g)
        xi = op.interleave(x)
        assert torch.equal(op.deinterleave(xi), x)
        assert torch.equal(xi[:, :, n - 1], x[n - 1])
        for flags, tau in ((0, 0.0), (1, 0.0), (2, 0.0), (4, 0.3), (3, -0.7)):
            y = op.apply_native(x, flags=flags, tau=tau)
            yi = op.apply_interleaved(xi, flags=flags, tau=tau)
            assert torch.equal(op.deinterleave(yi), y)
    with pytest.raises(Exception):
        op.apply_interleaved(torch.zeros((12, geo.site_count, 3), dtype=op.dtype, device="cuda"))


def test_large_lattice_matches_stencil(cuda):
    dims = (16, 16, 16, 16)
    M, geo, gauge, op, links = _setup(dims, 0.2)
    x = _rand(op.dim, 2)
    assert _rel(op.apply(x), W.apply_stencil(links, dims, 0.1, x)) < 1e-12


def test_plane_wave_kat(cuda):
    dims = (4, 4, 6, 8)
    M = _gpu()
    geo = M.LatticeGeometry(dims, "antiperiodic")
    op = M.build_wilson(M.generate_gauge(geo, "unit"), 0.1)
    rng = np.random.default_rng(0)
    for k in [(1, 2, 3, 4), (0, 0, 0, 0), (3, 1, 5, 7)]:
        p, Mp = W.plane_wave_symbol(dims, 0.1, k)
        chi = rng.normal(size=(4, 3)) + 1j * rng.normal(size=(4, 3))
        v = W.plane_wave(dims, p, chi)
        assert _rel(op.apply(v), W.plane_wave(dims, p, Mp @ chi)) < 1e-13


def test_complex64_against_fp64_oracle(cuda):
    dims = (8, 8, 8, 8)
    for recon in (18, 12):
        M, geo, gauge, op, links = _setup(dims, 0.2, prec=32, recon=recon)
        A = W.build_wilson4d_csr(links, dims, 0.1)
        x = _rand(op.dim, 9)
        assert _rel(op.apply(x), A @ x) < 2e-6


def test_layout_roundtrip_exact(cuda):
    M, geo, gauge, op, links = _setup((4, 6, 8, 10), 0.2)
    x = torch.as_tensor(_rand(op.dim, 3, 3).T.copy(), device=cuda)
    back = op.from_native(op.to_native(x))
    assert torch.equal(back, x)


def test_dimension_mismatch_raises(cuda):
    M, geo, gauge, op, links = _setup((4, 4, 4, 4), 0.2)
    with pytest.raises(ValueError):
        op.apply(np.zeros(op.dim - 12, dtype=np.complex128))


def test_dense_guard(cuda):
    M, geo, gauge, op, links = _setup((4, 4, 8, 8), 0.2)
    with pytest.raises(M.SizeGuardError):
        op.dense()
    M2, geo2, gauge2, op2, links2 = _setup((2, 2, 2, 4), 0.2)
    D = op2.dense()
    A = W.build_wilson4d_csr(links2, (2, 2, 2, 4), 0.1).toarray()
    assert np.abs(D - A).max() < 1e-13


@pytest.mark.parametrize("recon,flags,tau", [(12, 0, 0.0), (18, 3, 0.25), (12, 4, -0.1)])
def test_apply_dot_fused(cuda, recon, flags, tau):
    """mgt_wilson_apply_dot: y bitwise equal to the plain apply, d = vdot(u, y)
    to 1e-13, deterministic, 3 rhs."""
    import torch
    import paper_1909_12234_b200 as M
    geo = M.LatticeGeometry((4, 6, 8, 10), "antiperiodic")
    op = M.build_wilson(M.generate_gauge(geo, "su3", eps=0.3, seed=2), 0.1, recon=recon)
    g = torch.Generator(device="cuda").manual_seed(3)
    x = torch.randn((3, 12, geo.site_count), dtype=torch.complex128, device="cuda", generator=g)
    u = torch.randn((3, 12, geo.site_count), dtype=torch.complex128, device="cuda", generator=g)
    y, d = op.apply_dot_native(x, u, flags=flags, tau=tau)
    y0 = op.apply_native(x, flags=flags, tau=tau)
    assert torch.equal(y, y0)
    dr = torch.sum(u.conj() * y0, dim=(1, 2))
    assert ((d - dr).abs() / dr.abs()).max().item() < 1e-13
    y2, d2 = op.apply_dot_native(x, u, flags=flags, tau=tau)
    assert torch.equal(d, d2)


@pytest.mark.parametrize("prec,recon", [(64, 12), (64, 18), (32, 12)])
def test_smem_staged_apply_matches_default(cuda, monkeypatch, prec, recon):
    """The cp.async / shared-memory staged plain apply (MGT_DSLASH_VARIANT=2,
    csrc/dslash_pipe.cuh: neighbour spinors copied DEPTH items ahead into
    shared memory, links staged in registers, pipeline running across chunk
    boundaries) performs the per-site arithmetic of the default kernel in
    the same order: equal to rounding (FMA contraction may differ by an ulp)
    on ragged lattices with a partial last chunk, both boundaries, every
    flag variant; and against the oracle CSR at 1e-12."""
    M = _gpu()
    for dims, bc in (((4, 6, 2, 10), "periodic"), ((6, 10, 6, 6), "antiperiodic"), ((8, 8, 8, 8), "antiperiodic")):
        geo = M.LatticeGeometry(dims, bc)
        gauge = M.generate_gauge(geo, "su3", eps=0.3, seed=1)
        monkeypatch.setenv("MGT_DSLASH_VARIANT", "0")
        a = M.build_wilson(gauge, 0.1, prec=prec, recon=recon)
        monkeypatch.setenv("MGT_DSLASH_VARIANT", "2")
        b = M.build_wilson(gauge, 0.1, prec=prec, recon=recon)
        monkeypatch.setenv("MGT_DSLASH_VARIANT", "0")
        g = torch.Generator(device="cuda").manual_seed(3)
        x = torch.randn((3, 12, geo.site_count), dtype=a.dtype, device="cuda", generator=g)
        tol = 4e-16 if prec == 64 else 4e-7
        for flags, tau in ((0, 0.0), (1, 0.0), (2, 0.0), (4, 0.3), (3, -0.7)):
            ya = a.apply_native(x, flags=flags, tau=tau)
            yb = b.apply_native(x, flags=flags, tau=tau)
            assert (ya - yb).abs().max().item() <= tol * ya.abs().max().item()
        if prec == 64 and dims == (8, 8, 8, 8):
            A = W.build_wilson4d_csr(gauge.links.cpu().numpy(), dims, 0.1)
            xv = _rand(b.dim, 4)
            assert _rel(b.apply(xv), A @ xv) < 1e-12


@pytest.mark.parametrize("dims,boundary", [((4, 6, 4, 8), "antiperiodic"), ((6, 4, 2, 6), "periodic"),
                                           ((8, 8, 8, 8), "antiperiodic")])
def test_host_buffer_apply_pipeline(cuda, dims, boundary):
    """The e2e path of bench.py: LatticeOperator.apply on HOST vectors in the
    reference layout through mgt_wilson_apply_host (x0-chunked H2D -> layout
    -> stencil -> layout -> D2H on three streams; lattice.py:214-217 is the
    call it stands in for).  Against the oracle CSR at 1e-12, bitwise equal
    to the device-resident apply for every chunk count (1, 2, 3, L0, more
    than L0), flag variant, row-batched input, numpy / pageable / pinned
    buffers; the chunks' periodic x0 neighbours (first and last chunk) are
    the interesting sites."""
    M, geo, gauge, op, links = _setup(dims, 0.3, seed=2, recon=12, boundary=boundary)
    A = W.build_wilson4d_csr(links, dims, 0.1, antiperiodic=boundary == "antiperiodic")
    g5 = W.gamma5_diag(geo.site_count)
    x = _rand(op.dim, 21)

    def dev(v):  # the device-resident path (to_native -> mgt_wilson_apply -> from_native)
        return op.apply(torch.from_numpy(v).cuda()).cpu().numpy()

    ref = dev(x)
    assert _rel(ref, A @ x) < 1e-12
    assert np.array_equal(op.apply(x), ref)  # 1-D numpy input takes the host pipeline
    for nch in (1, 2, 3, dims[0], dims[0] + 5):
        y = op.apply_host(x, nchunks=nch)
        assert isinstance(y, np.ndarray) and np.array_equal(y, ref), nch
    # flag variants and the shift
    assert _rel(op.apply_host(x, flags=1), A @ (g5 * x)) < 1e-12
    assert _rel(op.apply_host(x, flags=2), g5 * (A @ x)) < 1e-12
    assert _rel(op.apply_host(x, flags=4), A.conj().T @ x) < 1e-12
    assert _rel(op.apply_host(x, tau=0.4, nchunks=3), A @ x + 0.4j * g5 * x) < 1e-12
    # row-batched input, pinned tensors, caller-provided output
    X = np.stack([_rand(op.dim, 30 + j) for j in range(3)])
    xt = torch.from_numpy(X).pin_memory()
    out = torch.empty_like(xt).pin_memory()
    yt = op.apply_host(xt, out=out, nchunks=2)
    assert yt.data_ptr() == out.data_ptr()
    for j in range(3):
        assert np.array_equal(out[j].numpy(), dev(X[j]))
    with pytest.raises(ValueError):
        op.apply_host(np.zeros(op.dim + 1, dtype=np.complex128))
    # complex64 operator: host data stays complex128, the arithmetic is fp32
    op32 = M.build_wilson(gauge, 0.1, prec=32, recon=12)
    assert _rel(op32.apply_host(x, nchunks=3), A @ x) < 2e-6
