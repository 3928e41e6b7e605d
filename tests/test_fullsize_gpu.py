"""Parity at BASELINE.json's full sizes through size-independent properties
(the CPU oracle cannot materialise these lattices): spot checks of A x at
random sites against the site-local oracle stencil, gamma5-Hermiticity,
linearity, and bitwise determinism of the solver and probes."""

import numpy as np
import pytest
import torch

from oracle import pcg64 as P
from oracle import wilson4d as W

pytestmark = pytest.mark.gpu


@pytest.fixture(scope="module")
def big():
    import paper_1909_12234_b200 as M
    dims = (48, 48, 48, 96)
    geo = M.LatticeGeometry(dims, "antiperiodic")
    gauge = M.generate_gauge(geo, "su3", eps=0.2, seed=0)
    op = M.build_wilson(gauge, 0.1)  # recon 12 (generated SU(3))
    yield M, geo, gauge, op
    del op, gauge
    torch.cuda.empty_cache()


def test_spot_check_sites_48x48x48x96(big):
    M, geo, gauge, op = big
    g = torch.Generator(device="cuda").manual_seed(5)
    x = torch.randn((1, 12, geo.site_count), dtype=torch.complex128, device="cuda", generator=g)
    y = op.from_native(op.apply_native(x))[0]
    xr = op.from_native(x)[0].cpu().numpy()
    links = gauge.links.cpu().numpy()
    rng = np.random.default_rng(0)
    V = geo.site_count
    T = geo.dims[3]
    # random sites plus every kind of boundary: t wrap (antiperiodic), x wraps
    sites = list(rng.integers(0, V, 150)) + [0, V - 1, T - 1, T, V - T, 47 * T * 48 * 48]
    ref = W.apply_at_sites(links, geo.dims, 0.1, xr, sites)
    got = y.reshape(-1, 12)[torch.as_tensor(sites, device="cuda")].cpu().numpy()
    assert np.linalg.norm(got - ref) / np.linalg.norm(ref) < 1e-12


def test_gamma5_hermiticity_and_linearity_full_size(big):
    M, geo, gauge, op = big
    from paper_1909_12234_b200 import _lib
    g = torch.Generator(device="cuda").manual_seed(7)
    x = torch.randn((2, 12, geo.site_count), dtype=torch.complex128, device="cuda", generator=g)
    ax = op.apply_native(x)
    # <y, A^dag x> = <A y, x>
    adx = op.apply_native(x[:1], flags=_lib.DAGGER)
    lhs = torch.vdot(x[1].reshape(-1), adx[0].reshape(-1))
    rhs = torch.vdot(ax[1].reshape(-1), x[0].reshape(-1))
    assert abs(lhs - rhs).item() <= 1e-12 * abs(rhs).item()
    # linearity: A (a x0 + b x1) = a A x0 + b A x1
    a, b = 0.3 - 1.1j, 2.0 + 0.5j
    comb = (a * x[0] + b * x[1]).unsqueeze(0)
    lin = op.apply_native(comb)[0]
    want = a * ax[0] + b * ax[1]
    assert (torch.linalg.vector_norm(lin - want) / torch.linalg.vector_norm(want)).item() < 1e-13


def test_probe_bits_at_full_size(big):
    M, geo, gauge, op = big
    N = geo.site_count * 12
    z = M.make_noise(N, "rademacher", 123).values
    # the bit stream is sequential: check head, tail and random windows against the restatement
    st, inc = P.seed_state(123)
    head = P.rademacher(4096, 123)
    assert np.array_equal(z[:4096].view(np.uint64), head.view(np.uint64))
    for start in (N // 3 * 2 // 2 * 2, N - 1000, 123456 * 2):
        start -= start % 2
        s = P.jump(st, inc, start // 2)
        words = P.raw32(s, inc, 1000)
        want = np.array([1.0 if w >> 31 else -1.0 for w in words], dtype=np.complex128)
        assert np.array_equal(z[start:start + 1000].view(np.uint64), want.view(np.uint64))


def test_solver_bitwise_deterministic(cuda):
    import paper_1909_12234_b200 as M
    geo = M.LatticeGeometry((16, 16, 16, 16), "antiperiodic")
    op = M.build_wilson(M.generate_gauge(geo, "su3", eps=0.2, seed=1), 0.1)
    probes = M.build_probe_set(geo, 12, 8, dilution=False, kind="rademacher", seed=3)
    inv = M.TruncatedInverse(op, M.SolveConfig(tol=1e-8))
    e1 = M.hutchinson(inv, probes)
    e2 = M.hutchinson(inv, probes)
    assert np.array_equal(e1.samples, e2.samples)
    z = probes.noise_native(0, 4)
    x1, _, _ = inv.solve_native(z)
    x2, _, _ = inv.solve_native(z)
    assert torch.equal(x1, x2)
