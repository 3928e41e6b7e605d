"""Levels >= 1 of a multigrid hierarchy (3-level hierarchies, SURVEY.md 8(f)
row f1): null vectors, chirality-split prolongator and Galerkin operator of a
COARSE operator, and the recursive two-grid cycle.

Restated from the reference (`/root/reference/pkg/src/mgtrace`):
`gcr_solve` (`krylov.py:52-118`), `generate_null_vectors`
(`multigrid.py:74-113`), `build_prolongator` (`:163-225`),
`build_coarse_operator` (`:246-259`), `two_grid_solve` (`:262-300`) and the
recursion of `MultigridSolver._coarse_solver` (`:366-377`).

The fine level runs on the hand-written kernels (multigrid.py / mgsolve.py);
the coarse levels are small (the level-1 operator of a 16^4 lattice with
4^4 aggregates has 12,288 dof), so here vectors are device tensors in the
REFERENCE coarse order and the level-1 operator applies through the native
9-block coarse kernel (`mgt_coarse_apply`).  The level-2 prolongator is a
batch of dense per-(block, chirality) column groups (gather + batched
GEMV), and the level-2 Galerkin operator is formed densely on the device
from the multi-rhs coarse apply (Nc2 columns at once).
"""

import numpy as np
import torch

from ._device import device
from .krylov import SolveReport


def _vdot(a, b):
    return torch.vdot(a.reshape(-1), b.reshape(-1))


def gcr_torch(apply, b, tol, max_iter, restart):
    """Restarted GCR from x0 = 0 with the reference's control flow
    (krylov.py:52-118): explicit-residual confirmation, restart recompute,
    breakdown test 1e-14, final explicit residual.  b: 1-D device tensor."""
    bnorm = torch.linalg.vector_norm(b).item()
    if bnorm == 0.0:
        return torch.zeros_like(b), SolveReport(0, 0.0, True, 0)
    x = torch.zeros_like(b)
    r = b.clone()
    matvecs = 0
    zs, qs = [], []
    it = 0
    relres = torch.linalg.vector_norm(r).item() / bnorm
    reason = "max_iter"
    while it < max_iter:
        if relres <= tol:
            r = b - apply(x)
            matvecs += 1
            relres = torch.linalg.vector_norm(r).item() / bnorm
            if relres <= tol:
                return x, SolveReport(it, relres, True, matvecs)
            zs, qs = [], []
        z = r.clone()
        q = apply(z)
        matvecs += 1
        qn0 = torch.linalg.vector_norm(q).item()
        for zj, qj in zip(zs, qs):
            beta = _vdot(qj, q)
            q = q - beta * qj
            z = z - beta * zj
        qn = torch.linalg.vector_norm(q).item()
        if qn <= 1e-14 * max(qn0, 1e-300):
            reason = "breakdown"
            break
        q = q / qn
        z = z / qn
        alpha = _vdot(q, r)
        x = x + alpha * z
        r = r - alpha * q
        zs.append(z)
        qs.append(q)
        it += 1
        relres = torch.linalg.vector_norm(r).item() / bnorm
        if len(zs) >= restart:
            zs, qs = [], []
            r = b - apply(x)
            matvecs += 1
            relres = torch.linalg.vector_norm(r).item() / bnorm
    r = b - apply(x)
    matvecs += 1
    relres = torch.linalg.vector_norm(r).item() / bnorm
    if relres <= tol:
        return x, SolveReport(it, relres, True, matvecs)
    return x, SolveReport(it, relres, False, matvecs, reason)


class CoarseSmoother:
    """Fixed-iteration GCR from a zero start on a coarse operator
    (krylov.py:236-252)."""

    def __init__(self, op, n_iters):
        if n_iters < 1:
            raise ValueError("n_iters must be >= 1")
        self.op = op
        self.n_iters = n_iters
        self.total_matvecs = 0

    def __call__(self, b):
        x, rep = gcr_torch(self.op.apply, b, 1e-15, self.n_iters, self.n_iters)
        self.total_matvecs += rep.matvecs
        return x


def generate_null_vectors_coarse(op, n, tol=1e-2, max_iter=200, seed=0):
    """multigrid.py:74-113 on a coarse operator (same RNG stream and order:
    all N real normals, then all N imaginary ones, per start)."""
    from .multigrid import NullVectors
    if n < 1:
        raise ValueError("need n >= 1 null vectors")
    rng = np.random.default_rng(seed)
    N = op.dim
    vecs = torch.empty((n, N), dtype=torch.complex128, device=device())
    ratios = np.empty(n)
    degenerate = np.zeros(n, dtype=bool)
    for i in range(n):
        for _attempt in range(3):
            y0 = torch.from_numpy(rng.normal(size=N) + 1j * rng.normal(size=N)).to(device())
            b = -op.apply(y0)
            d, rep = gcr_torch(op.apply, b, tol, max_iter, max_iter)
            y = y0 + d
            if rep.converged or rep.reason != "breakdown":
                break
        else:
            raise RuntimeError(f"null-vector solve kept breaking down (vector {i})")
        yn = torch.linalg.vector_norm(y).item()
        y0n = torch.linalg.vector_norm(y0).item()
        if yn < 1e-8 * y0n:
            degenerate[i] = True
            d1, _ = gcr_torch(op.apply, b, tol, 1, 1)
            y = y0 + d1
            yn = torch.linalg.vector_norm(y).item()
            if yn < 1e-8 * y0n:
                y, yn = y0, y0n
        ratios[i] = torch.linalg.vector_norm(op.apply(y)).item() / max(torch.linalg.vector_norm(b).item(), 1e-300)
        vecs[i] = y / yn
    return NullVectors(vecs, ratios, seed, op.geometry, op.dof, op.gamma5_diag, degenerate)


def _block_of_site(geo, block_dims):
    """multigrid.py:52-57: coords // block, raveled C-order (reference)."""
    coords = np.stack(np.unravel_index(np.arange(geo.site_count), geo.dims), axis=1)
    cd = np.array(geo.dims) // np.array(block_dims)
    return np.ravel_multi_index(tuple((coords // np.array(block_dims)).T), tuple(cd))


class LevelProlongator:
    """Chirality-split block prolongator of a coarse level (reference order
    on both sides).  G[(b, c)] holds the nv orthonormal columns restricted to
    their support idx[(b, c)] (fine indices ascending, as multigrid.py:192)."""

    def __init__(self, G, idx, geometry, blocking, fine_dof, nv, fine_dim):
        self.G = G            # (m, 2, nv, L) complex128
        self.idx = idx        # (m, 2, L) int64 device
        self.geometry = geometry
        self.blocking = blocking
        self.fine_dof = fine_dof
        self.nv = nv
        self.fine_dim = fine_dim
        m = G.shape[0]
        self.n_blocks = m
        self.coarse_dim = m * 2 * nv
        self.coarse_gamma5 = np.tile(np.concatenate([np.ones(nv), -np.ones(nv)]), m)
        self.per_block_counts = np.full((m, 2), nv)
        self.uniform = True

    @property
    def coarse_geometry(self):
        from .lattice import LatticeGeometry
        return LatticeGeometry(self.blocking.coarse_dims(self.geometry), self.geometry.boundary)

    def restrict(self, x):
        """V^H x for x (N,) or (k, N)."""
        X = x.reshape(-1, self.fine_dim)
        g = X[:, self.idx]                                   # (k, m, 2, L)
        xc = torch.einsum("mcvl,kmcl->kmcv", self.G.conj(), g)
        return xc.reshape(x.shape[:-1] + (self.coarse_dim,)) if x.dim() > 1 else xc.reshape(-1)

    def prolong(self, xc):
        Xc = xc.reshape(-1, self.n_blocks, 2, self.nv)
        vals = torch.einsum("mcvl,kmcv->kmcl", self.G, Xc)   # (k, m, 2, L)
        out = torch.zeros((Xc.shape[0], self.fine_dim), dtype=xc.dtype, device=xc.device)
        out[:, self.idx.reshape(-1)] = vals.reshape(Xc.shape[0], -1)
        return out.reshape(xc.shape[:-1] + (self.fine_dim,)) if xc.dim() > 1 else out.reshape(-1)

    def dense(self):
        eye = torch.eye(self.coarse_dim, dtype=torch.complex128, device=device())
        return self.prolong(eye).T.cpu().numpy()


def build_level_prolongator(null_vectors, blocking):
    """multigrid.py:163-225 for coarse-level null vectors (device tensors):
    per-(block, chirality) MGS run twice, batched over all groups; columns
    below 1e-8 are dropped (a drop makes the level non-uniform -> error)."""
    from .multigrid import BlockingError
    geo = null_vectors.geometry
    dof = null_vectors.dof
    blocking.validate(geo)
    Y = null_vectors.vectors
    n = Y.shape[0]
    m = blocking.block_count(geo)
    g5 = np.asarray(null_vectors.gamma5_diag)
    block_of = np.repeat(_block_of_site(geo, blocking.block_dims), dof)
    idx = []
    for b in range(m):
        inb = block_of == b
        for cmask in (g5 > 0, g5 < 0):
            sup = np.flatnonzero(inb & cmask)
            if sup.size == 0:
                raise BlockingError(f"block {b} has no chirality sites")
            idx.append(sup)
    L = len(idx[0])
    if any(len(s) != L for s in idx):
        raise BlockingError("non-uniform block supports")
    idx_t = torch.as_tensor(np.stack(idx).reshape(m, 2, L), device=device())
    V = Y[:, idx_t].permute(1, 2, 0, 3).reshape(m * 2, n, L).clone()   # (groups, n, L)
    keep = torch.ones((m * 2, n), dtype=torch.bool, device=device())
    for i in range(n):
        v = V[:, i, :]
        for _ in range(2):
            for u in range(i):
                w = V[:, u, :]
                d = torch.einsum("gl,gl->g", w.conj(), v) * keep[:, u]
                v = v - d[:, None] * w
        nv_ = torch.linalg.vector_norm(v, dim=1)
        ok = nv_ >= 1e-8
        keep[:, i] = ok
        V[:, i, :] = torch.where(ok[:, None], v / torch.where(ok, nv_, torch.ones_like(nv_))[:, None],
                                 torch.zeros_like(v))
    if not bool(keep.all()):
        raise BlockingError("rank-deficient coarse-level blocks: uniform coarse operator impossible")
    G = V.reshape(m, 2, n, L)
    return LevelProlongator(G, idx_t, geo, blocking, dof, n, Y.shape[1])


class DenseCoarseOperator:
    """Galerkin V^H A V of a coarse operator, held dense on the device (the
    level-2 operators are small); gamma5-Hermiticity checked like
    multigrid.py:250-258."""

    def __init__(self, D, prolongator, level=2):
        self.D = D
        self.prolongator = prolongator
        self.level = level
        self.geometry = prolongator.coarse_geometry
        self.dof = 2 * prolongator.nv
        self.gamma5_diag = prolongator.coarse_gamma5
        self._inv = None

    @property
    def dim(self):
        return self.D.shape[0]

    def apply(self, x):
        return (self.D @ x.reshape(-1, self.dim).T).T.reshape(x.shape)

    def dense(self):
        return self.D.cpu().numpy()

    def solve(self, b):
        if self._inv is None:
            self._inv = torch.linalg.inv(self.D)
        return (self._inv @ b.reshape(-1, self.dim).T).T.reshape(b.shape)


def build_level_coarse_operator(op, prolongator, level=2, check=True):
    """C = V^H (A V) with A a coarse operator (reference order apply)."""
    eye = torch.eye(prolongator.coarse_dim, dtype=torch.complex128, device=device())
    cols = prolongator.prolong(eye)                    # (Nc, N) rows = columns of V
    AV = _apply_many(op, cols)                         # (Nc, N)
    D = prolongator.restrict(AV).T.contiguous()        # D[:, j] = V^H A V e_j
    if check:
        g5 = torch.as_tensor(prolongator.coarse_gamma5, device=device())
        dev = (g5[:, None] * D * g5[None, :] - D.conj().T).abs().max().item()
        scale = max(D.abs().max().item(), 1e-300)
        if dev > 1e-12 * scale:
            raise ValueError(f"coarse operator lost gamma5-Hermiticity: {dev:.3e}")
    return DenseCoarseOperator(D, prolongator, level)


def _apply_many(op, X):
    """op applied to every row of X (reference coarse order)."""
    if hasattr(op, "prolongator") and hasattr(op.prolongator, "coarse_from_ref"):
        pr = op.prolongator
        nat = pr.coarse_from_ref(X.reshape(X.shape[0], pr.n_blocks, pr.nc).contiguous())
        return pr.coarse_to_ref(op.apply_native(nat)).reshape(X.shape)
    return torch.stack([op.apply(x) for x in X])


def two_grid_solve_ref(op, prolongator, coarse_solver, smoother, b, tol, max_cycles=100):
    """multigrid.py:262-300 on a 1-D device vector of a coarse level."""
    bn = torch.linalg.vector_norm(b).item()
    if bn == 0.0:
        return torch.zeros_like(b), SolveReport(0, 0.0, True, 0)
    x = torch.zeros_like(b)
    r = b.clone()
    matvecs = 0
    sm_before = getattr(smoother, "total_matvecs", 0)
    best = torch.linalg.vector_norm(r).item() / bn
    relres = best

    def report(cycle, ok, reason=""):
        sm = getattr(smoother, "total_matvecs", sm_before) - sm_before
        return SolveReport(cycle, relres, ok, matvecs + sm, reason)

    for cycle in range(max_cycles):
        if relres <= tol:
            return x, report(cycle, True)
        xc = coarse_solver(prolongator.restrict(r))
        x = x + prolongator.prolong(xc)
        r = b - op.apply(x)
        matvecs += 1
        x = x + smoother(r)
        r = b - op.apply(x)
        matvecs += 1
        relres = torch.linalg.vector_norm(r).item() / bn
        best = min(best, relres)
        if relres > 10 * best:
            return x, report(cycle + 1, False, "divergence")
    ok = relres <= tol
    return x, report(max_cycles, ok, "" if ok else "max_cycles")
