"""PCG64 (XSL-RR 128/64) restatement and the reference noise draws
(TEST INFRASTRUCTURE ONLY).

The reference draws probe noise in `probing.py:94-107`:
`default_rng(seed).integers(0, 2, size=n) * 2.0 - 1.0` (Rademacher) and
`integers(0, 4)` (Z4); probe j of a probe set uses seed `seed0 + j`
(`probing.py:155`).  The arithmetic lives in numpy (third-party, not
vendored; pinned here against numpy 2.3.5, the container's version):

* PCG64 step-then-output: s <- s*M + inc (mod 2^128),
  out = rotr64(hi(s) ^ lo(s), hi(s) >> 58), M = 0x2360ED051FC65DA44385DF649FCCF645.
* `integers(0, k)` for k <= 2^32 draws buffered 32-bit words (low half of a
  64-bit output first, then the high half) and applies Lemire's
  multiply-shift: value = (u32 * k) >> 32.  For k = 2 and k = 4 the rejection
  threshold is 0, so the value is simply the top 1 (resp. 2) bits of u32.

Seeding (SeedSequence hashing) is taken from numpy itself,
`PCG64(seed).state['state']`, exactly as the product does on the host.
"""

import numpy as np

MULT = 0x2360ED051FC65DA44385DF649FCCF645
MASK128 = (1 << 128) - 1
MASK64 = (1 << 64) - 1


def seed_state(seed):
    st = np.random.PCG64(seed).state["state"]
    return int(st["state"]), int(st["inc"])


def _rotr64(v, r):
    r &= 63
    return ((v >> r) | (v << ((64 - r) & 63))) & MASK64


def raw64(state, inc, count):
    """First `count` 64-bit outputs (pure Python, small counts only)."""
    out = []
    s = state
    for _ in range(count):
        s = (s * MULT + inc) & MASK128
        hi, lo = s >> 64, s & MASK64
        out.append(_rotr64(hi ^ lo, hi >> 58))
    return out, s


def raw32(state, inc, count):
    """Buffered 32-bit stream: low half of each 64-bit output first."""
    words = []
    outs, _ = raw64(state, inc, (count + 1) // 2)
    for o in outs:
        words.append(o & 0xFFFFFFFF)
        words.append(o >> 32)
    return words[:count]


def rademacher(n, seed):
    """Restated `make_noise(n, 'rademacher', seed).values` (probing.py:97-98)."""
    st, inc = seed_state(seed)
    w = np.array(raw32(st, inc, n), dtype=np.uint64)
    bits = (w >> np.uint64(31)).astype(np.float64)
    return (bits * 2.0 - 1.0).astype(np.complex128)


def z4(n, seed):
    """Restated `make_noise(n, 'z4', seed).values` (probing.py:99-103), with
    the reference's signed zeros: k=3 maps to (-0.0 - 1j)."""
    st, inc = seed_state(seed)
    w = np.array(raw32(st, inc, n), dtype=np.uint64)
    k = (w >> np.uint64(30)).astype(np.int64)
    vals = np.exp(0.5j * np.pi * k)
    return np.round(vals.real) + 1j * np.round(vals.imag)


def rademacher_numpy(n, seed):
    """The reference's own call, for pinning the restatement."""
    rng = np.random.default_rng(seed)
    return (rng.integers(0, 2, size=n) * 2.0 - 1.0).astype(np.complex128)


def jump(state, inc, k):
    """State after k steps (affine power by squaring), for jump-ahead checks."""
    acc_mult, acc_plus = 1, 0
    cur_mult, cur_plus = MULT, inc
    while k:
        if k & 1:
            acc_mult = (acc_mult * cur_mult) & MASK128
            acc_plus = (acc_plus * cur_mult + cur_plus) & MASK128
        cur_plus = ((cur_mult + 1) * cur_plus) & MASK128
        cur_mult = (cur_mult * cur_mult) & MASK128
        k >>= 1
    return (acc_mult * state + acc_plus) & MASK128
