"""Restated reference multigrid setup (TEST INFRASTRUCTURE ONLY).

Follows `/root/reference/pkg/src/mgtrace/multigrid.py`:
* `null_vectors` <- `generate_null_vectors` (`:74-113`): per vector
  `y0 = normal(N) + 1j normal(N)` from one `default_rng(seed)` stream
  (`:82`, `:91`), relax with GCR(max_iter, restart = max_iter) on
  A d = -A y0 (`:87`, `:93-95`), y = y0 + d, breakdown retry x3 (`:90-99`),
  degenerate fallback (`:100-110`), normalise (`:112`);
* `prolongator` <- `build_prolongator` (`:163-225`): chirality split by the
  gamma5 sign (`:180`), support = fine indices of the block and chirality in
  ascending order (`:192`), MGS run twice (`:198-200`), drop < 1e-8
  (`:202-204`), column order block-major, + chirality columns then -
  (`:189-216`);
* `coarse_operator` <- `build_coarse_operator` (`:246-259`): Galerkin
  P^H A P with the gamma5_c-Hermiticity check to 1e-12 (`:251-258`).
Blocks are the lexicographic (first coordinate slowest) coarse sites
(`BlockingScheme.block_of_site`, `:52-57`).
"""

import numpy as np
import scipy.sparse as sp

from . import krylov


def block_of_site(dims, block):
    V = int(np.prod(dims))
    coords = np.stack(np.unravel_index(np.arange(V), dims))
    bc = coords // np.array(block)[:, None]
    cdims = tuple(L // b for L, b in zip(dims, block))
    return np.ravel_multi_index(bc, cdims), cdims


def start_vectors(N, n, seed):
    """The Gaussian starts y0 in the reference's draw order (no retries)."""
    rng = np.random.default_rng(seed)
    out = np.empty((n, N), dtype=np.complex128)
    for i in range(n):
        out[i] = rng.normal(size=N) + 1j * rng.normal(size=N)
    return out


def null_vectors(matvec, N, n, tol=1e-2, max_iter=200, seed=0):
    rng = np.random.default_rng(seed)
    vecs = np.empty((n, N), dtype=np.complex128)
    for i in range(n):
        for attempt in range(3):
            y0 = rng.normal(size=N) + 1j * rng.normal(size=N)
            b = -matvec(y0)
            d, rep = krylov.gcr(matvec, b, tol, max_iter, max_iter)
            y = y0 + d
            if rep.converged or rep.reason != "breakdown":
                break
        else:
            raise RuntimeError(f"null-vector solve kept breaking down (vector {i})")
        yn = np.linalg.norm(y)
        if yn < 1e-8 * np.linalg.norm(y0):
            d1, _ = krylov.gcr(matvec, b, tol, 1, 1)
            y = y0 + d1
            yn = np.linalg.norm(y)
            if yn < 1e-8 * np.linalg.norm(y0):
                y, yn = y0, np.linalg.norm(y0)
        vecs[i] = y / yn
    return vecs


def prolongator(Y, dims, block, g5):
    """Returns (P csr (N x Nc), coarse_gamma5, per_block_counts, dropped)."""
    n, N = Y.shape
    dof = N // int(np.prod(dims))
    bos, cdims = block_of_site(dims, block)
    m = int(np.prod(cdims))
    blk = np.repeat(bos, dof)
    rows_all, vals_all, cols_all, g5c = [], [], [], []
    counts = np.zeros((m, 2), dtype=int)
    dropped = 0
    col = 0
    order = np.argsort(blk, kind="stable")  # fine indices grouped by block, ascending
    starts = np.searchsorted(blk[order], np.arange(m + 1))
    for b in range(m):
        idx = order[starts[b]:starts[b + 1]]
        for ci, sign in enumerate((1.0, -1.0)):
            support = idx[g5[idx] == sign]
            basis = []
            for i in range(n):
                v = Y[i, support].copy()
                for _ in range(2):
                    for u in basis:
                        v = v - np.vdot(u, v) * u
                nv = np.linalg.norm(v)
                if nv < 1e-8:
                    dropped += 1
                    continue
                basis.append(v / nv)
            for v in basis:
                rows_all.append(support)
                vals_all.append(v)
                cols_all.append(np.full(len(support), col))
                g5c.append(sign)
                col += 1
            counts[b, ci] = len(basis)
    P = sp.coo_matrix((np.concatenate(vals_all), (np.concatenate(rows_all), np.concatenate(cols_all))),
                      shape=(N, col)).tocsr()
    return P, np.array(g5c), counts, dropped


def coarse_operator(A, P, g5c):
    C = (P.conj().T @ (A @ P)).tocsr()
    C.eliminate_zeros()
    G = sp.diags(g5c)
    D = (G @ C @ G - C.conj().T).tocoo()
    scale = max(np.abs(C.data).max(), 1e-300)
    if D.nnz and np.abs(D.data).max() > 1e-12 * scale:
        raise ValueError("coarse operator lost gamma5-Hermiticity")
    return C
