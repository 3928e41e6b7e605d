"""Parallel, bit-exact replay of a numpy PCG64 `standard_normal` stream.

The null-vector starts of `generate_null_vectors` (reference
multigrid.py:82, :91: `y0 = rng.normal(size=N) + 1j * rng.normal(size=N)`
from one `default_rng(seed)`) are the only host-side numbers on the
setup path; at 32^3x64 they are 1.2 G normals, ~12 s of one core.  numpy's
normal sampler (a 256-level ziggurat) consumes one 64-bit PCG64 output per
normal except on its rare rejection paths, so the stream cannot be cut at
known output positions -- but it can be cut speculatively:

* chunk j is decoded by numpy itself from a copy of the generator advanced
  by j*Q raw outputs (`PCG64.advance`), i.e. as if a normal started there;
* if that raw position lies inside a multi-output normal, the chunk's first
  few values are garbage, but its decoding re-aligns with the true one as
  soon as both start a normal at the same raw position (almost every raw
  position starts a normal), after which both produce identical values;
* chunk j-1 decodes Q + margin normals (>= Q + margin raw outputs), so it
  overlaps chunk j; the two are stitched where a run of 8 of chunk j's
  values (after its first 16) occurs in chunk j-1.

Chunks decode in parallel threads (numpy releases the GIL while filling).
The result is bitwise the sequential `rng.standard_normal` stream
(tests/test_rng_cpu.py); stitching that cannot find its overlap raises.
"""

import concurrent.futures as cf
import os
import threading

import numpy as np

_POOL = None
_POOL_LOCK = threading.Lock()


def _pool():
    global _POOL
    with _POOL_LOCK:
        if _POOL is None:
            n = max(1, min(32, os.cpu_count() or 1))
            _POOL = cf.ThreadPoolExecutor(max_workers=n, thread_name_prefix="mgt-rng")
        return _POOL


_COPY_POOL = None


def _copy_pool():
    global _COPY_POOL
    with _POOL_LOCK:
        if _COPY_POOL is None:
            _COPY_POOL = cf.ThreadPoolExecutor(max_workers=8, thread_name_prefix="mgt-rng-copy")
        return _COPY_POOL


class NormalStream:
    """Consecutive `standard_normal` draws of `rng` (a numpy Generator on
    PCG64), decoded in parallel.  `take(n, out=None)` returns the next n
    values exactly as `rng.standard_normal(n)` would have (the caller's rng is
    not advanced)."""

    SYNC_SKIP = 16   # values of a chunk that may precede its re-alignment
    SYNC_RUN = 8     # length of the matched run
    MARGIN = 4096    # extra normals decoded past a chunk's Q raw outputs

    def __init__(self, rng, threads=None, max_chunk=1 << 22, min_chunk=1 << 16):
        bg = rng.bit_generator
        if type(bg).__name__ != "PCG64":
            raise TypeError("NormalStream replays numpy PCG64 generators only")
        self._state = bg.state
        self._threads = threads or max(1, min(32, os.cpu_count() or 1))
        self._max_chunk, self._min_chunk = int(max_chunk), int(min_chunk)
        self._raw_next = 0      # raw offset (from the snapshot) of the next chunk
        self._ready = []        # trusted arrays, in order, no overlap
        self._prev = None       # the last trusted array (overlaps the next chunk)
        self._prev_raw = 0      # raw position where _prev's decoding started
        self._avail = 0         # values in _ready + _prev
        self._pending = None    # futures of the round being decoded

    def _decode(self, raw_start, count):
        bg = np.random.PCG64()
        bg.state = self._state
        if raw_start:
            bg.advance(raw_start)
        out = np.empty(count)
        np.random.Generator(bg).standard_normal(out=out)
        return out

    def _stitch(self, chunk, raw_start):
        """Append a chunk decoded from raw position raw_start (relative to
        the start of the previous one, d = raw_start - prev's start, the
        overlap begins near prev[d * (1 - rejection rate)])."""
        prev = self._prev
        d = raw_start - self._prev_raw
        for skip in (self.SYNC_SKIP, 64, 256, 1024):
            if skip + self.SYNC_RUN > len(chunk):
                break
            key = chunk[skip:skip + self.SYNC_RUN]
            windows = [(max(0, int(0.97 * d) - 64), min(len(prev), d + skip + 64)), (0, len(prev))]
            for lo, hi in windows:
                for u in lo + np.flatnonzero(prev[lo:hi] == key[0]):
                    if u + self.SYNC_RUN <= len(prev) and np.array_equal(prev[u:u + self.SYNC_RUN], key):
                        self._avail -= len(prev) - u
                        self._ready.append(prev[:u])
                        self._prev = chunk[skip:]
                        self._prev_raw = raw_start + skip  # approximately: the search window allows for it
                        self._avail += len(self._prev)
                        return
        raise RuntimeError("NormalStream: chunks did not re-align (no overlap found)")

    def _submit(self, q):
        starts = [self._raw_next + j * q for j in range(self._threads)]
        self._raw_next = starts[-1] + q
        return [(st, _pool().submit(self._decode, st, q + self.MARGIN)) for st in starts]

    def _fill(self, need):
        """Stitch the pending round of `threads` chunks (submitting one if none
        is in flight), then start decoding the next round in the background,
        so the consumer's own work overlaps the decoding."""
        q = int(min(self._max_chunk, max(self._min_chunk, -(-need // self._threads))))
        if self._pending is None:
            self._pending = self._submit(q)
        chunks = [(st, f.result()) for st, f in self._pending]
        self._pending = self._submit(q)
        for st, c in chunks:
            if self._prev is None:       # the very first chunk starts on a normal
                self._prev, self._prev_raw = c, st
                self._avail += len(c)
            else:
                self._stitch(c, st)

    def take(self, n, out=None):
        n = int(n)
        out = np.empty(n) if out is None else out
        if out.shape != (n,):
            raise ValueError("out must have shape (n,)")
        # keep one chunk beyond the request: the last trusted array may still
        # be cut back by the next stitch
        while True:
            ready = self._avail - (len(self._prev) if self._prev is not None else 0)
            if ready >= n:
                break
            self._fill(n - ready)
        pos = 0
        copies = []
        while pos < n:
            a = self._ready[0]
            m = min(len(a), n - pos)
            copies.append((pos, a[:m]))
            pos += m
            self._avail -= m
            if m == len(a):
                self._ready.pop(0)
            else:
                self._ready[0] = a[m:]
        # the copies into `out` (a pinned staging buffer: ~200 MB per half
        # vector at 32^3 x 64) are memory-bound; spread them over a few
        # threads (numpy releases the GIL while copying)
        if n >= (1 << 20) and len(copies) > 1:
            list(_copy_pool().map(lambda pa: out.__setitem__(slice(pa[0], pa[0] + len(pa[1])), pa[1]), copies))
        else:
            for p0, a in copies:
                out[p0:p0 + len(a)] = a
        return out
