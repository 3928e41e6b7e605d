"""Probe draws: bitwise equality with the reference's numpy draws
(probing.py:94-107, :155) -- BASELINE.json north_star: "Probe draws:
bit-exact"."""

import numpy as np
import pytest
import torch

from oracle import pcg64 as P

pytestmark = pytest.mark.gpu


def _bits_equal(a, b):
    return np.array_equal(a.view(np.uint64), b.view(np.uint64))


@pytest.mark.parametrize("seed", [0, 1, 7, 99, 12345, 2**40 + 7, 1196192930])
def test_rademacher_ref_layout_bitwise(cuda, seed):
    import paper_1909_12234_b200 as M
    for n in (12, 49152, 12 * 1000 + 7, 1):
        got = M.make_noise(n, "rademacher", seed).values
        assert _bits_equal(got, P.rademacher_numpy(n, seed))


@pytest.mark.parametrize("seed", [0, 5, 2**33 + 1])
def test_z4_bitwise_with_signed_zeros(cuda, seed):
    import paper_1909_12234_b200 as M
    n = 12 * 257
    rng = np.random.default_rng(seed)
    ref = np.exp(0.5j * np.pi * rng.integers(0, 4, size=n))
    ref = np.round(ref.real) + 1j * np.round(ref.imag)
    got = M.make_noise(n, "z4", seed).values
    assert _bits_equal(got, ref)


def test_native_layout_probe_set(cuda):
    import paper_1909_12234_b200 as M
    geo = M.LatticeGeometry((4, 6, 8, 10), "antiperiodic")
    ps = M.build_probe_set(geo, 12, 5, hp_count=1, dilution=False, kind="rademacher", seed=42)
    gauge = M.generate_gauge(geo, "unit")
    op = M.build_wilson(gauge, 0.1)
    nat = ps.noise_native(0, 5)
    ref = op.from_native(nat).cpu().numpy()
    N = geo.site_count * 12
    for j in range(5):
        assert _bits_equal(ref[j], P.rademacher_numpy(N, 42 + j))
    groups = ps.groups
    assert len(groups) == 5 and groups[2].slots.shape == (1, N)
    assert _bits_equal(groups[2].slots[0], P.rademacher_numpy(N, 44))


def test_dilution_slots_sum_to_noise(cuda):
    import paper_1909_12234_b200 as M
    geo = M.LatticeGeometry((2, 2, 2, 4), "antiperiodic")
    ps = M.build_probe_set(geo, 12, 2, dilution=True, kind="z4", seed=3)
    g = ps.groups[1]
    assert g.slots.shape == (12, geo.site_count * 12)
    assert np.array_equal(g.slots.sum(axis=0), g.noise.values)
    s = ps.slots_native(1)
    assert torch.equal(s.sum(dim=0), ps.noise_native(1, 2)[0])
