"""Parallel replay of numpy's PCG64 normal stream (paper_1909_12234_b200/rng.py)
against the sequential `rng.standard_normal` draws: bitwise, across many
chunk stitches, odd request sizes and several seeds (the null-vector starts
of generate_null_vectors, reference multigrid.py:82, :91)."""

import numpy as np
import pytest

from paper_1909_12234_b200.rng import NormalStream


@pytest.mark.parametrize("seed", [0, 7, 12345, 2**40 + 3])
def test_stream_matches_sequential_draws(seed):
    ref = np.random.default_rng(seed)
    st = NormalStream(np.random.default_rng(seed), threads=5, max_chunk=20000, min_chunk=3000)
    for n in (1, 17, 4096, 50000, 3, 123457, 99999):
        got = st.take(n)
        want = ref.standard_normal(n)
        assert np.array_equal(got.view(np.uint64), want.view(np.uint64)), n


def test_stream_reference_pair_order_and_out_buffer():
    """y0 = normal(N) + 1j normal(N): real parts first, then imaginary."""
    N = 30011
    ref = np.random.default_rng(3)
    st = NormalStream(np.random.default_rng(3), threads=3, max_chunk=8192, min_chunk=1024)
    buf = np.empty(N)
    for _ in range(4):
        re = st.take(N, out=buf).copy()
        im = st.take(N)
        assert np.array_equal(re, ref.normal(size=N))
        assert np.array_equal(im, ref.normal(size=N))
    with pytest.raises(ValueError):
        st.take(5, out=np.empty(4))


def test_stream_rejects_other_bit_generators():
    with pytest.raises(TypeError):
        NormalStream(np.random.Generator(np.random.MT19937(0)))
