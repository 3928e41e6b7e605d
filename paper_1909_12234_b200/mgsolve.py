"""Two-grid multigrid inverter on the GPU.

Mirrors the reference's MG-preconditioned inverter:
`krylov.Smoother` / `make_smoother` (`krylov.py:236-256`, fixed-iteration GCR
from a zero start), `multigrid.two_grid_solve` (`multigrid.py:262-300`:
coarse-grid correction, smoothing, explicit residual, divergence abort),
`Hierarchy` / `build_hierarchy` (`:315-341`, two levels) and
`MultigridSolver` (`:344-381`: coarsest level by LU or an iterative solve),
wired as a `TruncatedInverse` solver plugin exactly like
`experiments.build_inverter` (`experiments.py:50-62`).

Everything runs on device fields: the smoother is the GPU GCR(m)
(`mgt_gcr_solve`), restriction/prolongation are the P^H / P kernels, the
coarsest solve is the cached dense C^-1 (LU on the device) or the coarse
BiCGStab.  The fine prolongator kernels are specialised to the 12-component
Wilson field, so hierarchies are two-level.
"""

from dataclasses import dataclass

import numpy as np
import torch

from .krylov import SolveReport
from .multigrid import (BlockingScheme, build_coarse_operator, build_prolongator, coarse_bicgstab,
                        gcr_relax, generate_null_vectors)


class Smoother:
    """Fixed-iteration GCR from a zero start (krylov.py:236-252)."""

    def __init__(self, op, n_iters):
        if n_iters < 1:
            raise ValueError("n_iters must be >= 1")
        self.op = op
        self.n_iters = n_iters
        self.total_matvecs = 0

    def __call__(self, b):
        x, _, _, _, mv = gcr_relax(self.op, b, 1e-15, self.n_iters, self.n_iters)
        self.total_matvecs += mv
        return x


def make_smoother(op, n_iters):
    return Smoother(op, n_iters)


def two_grid_solve(op, prolongator, coarse_solver, smoother, b, tol, max_cycles=100):
    """multigrid.py:262-300 on native fields b (1, 12, V): returns
    (x, SolveReport); matvecs count fine applications incl. the smoother's."""
    bn = torch.linalg.vector_norm(b).item()
    if bn == 0.0:
        return torch.zeros_like(b), SolveReport(0, 0.0, True, 0)
    x = torch.zeros_like(b)
    r = b.clone()
    matvecs = 0
    sm_before = getattr(smoother, "total_matvecs", 0)
    best = 1.0
    relres = best

    def report(cycle, ok, reason=""):
        sm = getattr(smoother, "total_matvecs", sm_before) - sm_before
        return SolveReport(cycle, relres, ok, matvecs + sm, reason)

    for cycle in range(max_cycles):
        if relres <= tol:
            return x, report(cycle, True)
        xc = coarse_solver(prolongator.restrict_native(r))
        x = x + prolongator.prolong_native(xc)
        r = b - op.apply_native(x)
        matvecs += 1
        x = x + smoother(r)
        r = b - op.apply_native(x)
        matvecs += 1
        relres = torch.linalg.vector_norm(r).item() / bn
        best = min(best, relres)
        if relres > 10 * best:
            return x, report(cycle + 1, False, "divergence")
    ok = relres <= tol
    return x, report(max_cycles, ok, "" if ok else "max_cycles")


@dataclass
class Hierarchy:
    operators: list
    prolongators: list

    @property
    def levels(self):
        return len(self.operators)


def build_hierarchy(op, blockings, null_counts, null_tol=1e-2, null_max_iter=200, seed=0):
    """2- or 3-level hierarchy by recursive null-vector setup
    (multigrid.py:328-341; level l uses seed + 7 l).  Level 0 -> 1 runs on
    the fine kernels; level 1 -> 2 on the coarse-level pieces (mglevel.py)."""
    from .multigrid import BlockingError
    if len(blockings) != len(null_counts):
        raise BlockingError("need one null-vector count per blocking level")
    if len(blockings) not in (1, 2):
        raise NotImplementedError("hierarchies of 2 or 3 levels are supported")
    nv = generate_null_vectors(op, null_counts[0], tol=null_tol, max_iter=null_max_iter, seed=seed)
    P = build_prolongator(nv, BlockingScheme(tuple(blockings[0])), layout_op=op)
    ops, prols = [op, build_coarse_operator(op, P, level=1)], [P]
    if len(blockings) == 2:
        from .mglevel import build_level_coarse_operator, build_level_prolongator, generate_null_vectors_coarse
        nv1 = generate_null_vectors_coarse(ops[1], null_counts[1], tol=null_tol, max_iter=null_max_iter,
                                           seed=seed + 7)
        P1 = build_level_prolongator(nv1, BlockingScheme(tuple(blockings[1])))
        ops.append(build_level_coarse_operator(ops[1], P1, level=2))
        prols.append(P1)
    return Hierarchy(ops, prols)


def dump_hierarchy(hierarchy, outdir):
    """Portable dump in the reference's format (multigrid.py:384-407):
    hierarchy_manifest.csv (level, dims, block_dims, coarse_dim, fine_dof,
    columns_file) and one columns CSV per level with rows (col, site, spin,
    re, im) ordered by column then fine row, values with 17 significant
    digits (exact round trip)."""
    import csv
    import os

    from .multigrid import prolongator_entries
    os.makedirs(outdir, exist_ok=True)
    manifest = os.path.join(outdir, "hierarchy_manifest.csv")
    with open(manifest, "w", newline="") as f:
        w = csv.writer(f)
        w.writerow(["level", "dims", "block_dims", "coarse_dim", "fine_dof", "columns_file"])
        for lvl, P in enumerate(hierarchy.prolongators):
            fname = f"level{lvl}_columns.csv"
            col, site, comp, val = prolongator_entries(P) if lvl == 0 else _level_entries(P)
            w.writerow([lvl, "x".join(map(str, P.geometry.dims)), "x".join(map(str, P.blocking.block_dims)),
                        int(col.max()) + 1 if len(col) else 0, P.fine_dof, fname])
            with open(os.path.join(outdir, fname), "w", newline="") as g:
                cw = csv.writer(g)
                cw.writerow(["col", "site", "spin", "re", "im"])
                cw.writerows([int(c), int(si), int(sp), f"{v.real:.17g}", f"{v.imag:.17g}"]
                             for c, si, sp, v in zip(col, site, comp, val))
    return manifest


def load_hierarchy(fine_op, outdir):
    """Rebuild a hierarchy from a dump (multigrid.py:409-435): the
    prolongator is placed back into the device block layout and the Galerkin
    operator recomputed on the GPU."""
    import csv
    import os

    from .multigrid import prolongator_from_entries
    with open(os.path.join(outdir, "hierarchy_manifest.csv"), newline="") as f:
        recs = list(csv.DictReader(f))
    if len(recs) not in (1, 2):
        raise NotImplementedError("hierarchies of 2 or 3 levels are supported")
    rec = recs[0]
    block = tuple(int(v) for v in rec["block_dims"].split("x"))
    dims = tuple(int(v) for v in rec["dims"].split("x"))
    if dims != tuple(fine_op.geometry.dims):
        raise ValueError(f"dump is for lattice {dims}, operator is {fine_op.geometry.dims}")
    blocking = BlockingScheme(block)
    nc = int(rec["coarse_dim"])
    nv = nc // (2 * blocking.block_count(fine_op.geometry))
    cols, sites, spins, vals = [], [], [], []
    with open(os.path.join(outdir, rec["columns_file"]), newline="") as g:
        for line in csv.DictReader(g):
            cols.append(int(line["col"]))
            sites.append(int(line["site"]))
            spins.append(int(line["spin"]))
            vals.append(complex(float(line["re"]), float(line["im"])))
    P = prolongator_from_entries(fine_op.geometry, blocking, nv, np.array(cols), np.array(sites), np.array(spins),
                                 np.array(vals, dtype=np.complex128), layout_op=fine_op,
                                 fine_dof=int(rec["fine_dof"]))
    ops, prols = [fine_op, build_coarse_operator(fine_op, P, level=1)], [P]
    if len(recs) == 2:
        from .mglevel import build_level_coarse_operator
        rec = recs[1]
        cols, sites, spins, vals = _read_columns(os.path.join(outdir, rec["columns_file"]))
        P1 = _level_from_entries(ops[1], BlockingScheme(tuple(int(v) for v in rec["block_dims"].split("x"))),
                                 int(rec["coarse_dim"]), int(rec["fine_dof"]), cols, sites, spins, vals)
        ops.append(build_level_coarse_operator(ops[1], P1, level=2))
        prols.append(P1)
    return Hierarchy(ops, prols)


def _read_columns(path):
    import csv
    cols, sites, spins, vals = [], [], [], []
    with open(path, newline="") as g:
        for line in csv.DictReader(g):
            cols.append(int(line["col"]))
            sites.append(int(line["site"]))
            spins.append(int(line["spin"]))
            vals.append(complex(float(line["re"]), float(line["im"])))
    return np.array(cols), np.array(sites), np.array(spins), np.array(vals, dtype=np.complex128)


def _level_entries(P):
    """(col, site, spin, value) of a coarse-level prolongator, column then row order."""
    m, nv, L = P.n_blocks, P.nv, P.G.shape[-1]
    G = P.G.cpu().numpy()
    idx = P.idx.cpu().numpy()
    cols, rows, vals = [], [], []
    for b in range(m):
        for c in range(2):
            order = np.argsort(idx[b, c])
            for k in range(nv):
                cols.append(np.full(L, (b * 2 + c) * nv + k))
                rows.append(idx[b, c][order])
                vals.append(G[b, c, k][order])
    rows = np.concatenate(rows)
    return np.concatenate(cols), rows // P.fine_dof, rows % P.fine_dof, np.concatenate(vals)


def _level_from_entries(op, blocking, nc, dof, cols, sites, spins, vals):
    from .mglevel import LevelProlongator
    from ._device import device
    m = blocking.block_count(op.geometry)
    nv = nc // (2 * m)
    L = len(cols) // nc
    order = np.lexsort((sites * dof + spins, cols))
    rows = (sites * dof + spins)[order].reshape(m, 2, nv, L)
    if np.any(rows != rows[:, :, :1, :]):
        raise ValueError("columns of one (block, chirality) group must share their support")
    G = torch.as_tensor(vals[order].reshape(m, 2, nv, L)).to(device())
    idx = torch.as_tensor(rows[:, :, 0, :]).to(device())
    return LevelProlongator(G, idx, op.geometry, blocking, dof, nv, op.dim)


class MultigridSolver:
    """Two-grid cycles recursing through an intermediate level for 3-level
    hierarchies (multigrid.py:344-381).  Coarsest level: dense LU on the
    device ("lu"), or iterative -- coarse BiCGStab for a level-1 coarsest
    ("bicgstab"), GCR(32) for a level-2 coarsest ("gcr", as the reference)."""

    def __init__(self, hierarchy, smoother_iters=4, coarse_tol=1e-1, coarse_max_iter=200, coarsest="lu"):
        from .mglevel import CoarseSmoother
        self.hierarchy = hierarchy
        ops = hierarchy.operators
        self.smoothers = [make_smoother(ops[0], smoother_iters)] + [CoarseSmoother(o, smoother_iters)
                                                                     for o in ops[1:-1]]
        self.coarse_tol = coarse_tol
        self.coarse_max_iter = coarse_max_iter
        self.coarsest = coarsest
        coarse = ops[-1]
        if hierarchy.levels == 2:
            if coarsest == "lu":
                self._cinv = coarse.dense_inverse_native()
                self._coarse = lambda rc: (rc.reshape(rc.shape[0], -1) @ self._cinv.T).reshape(rc.shape)
            else:
                self._coarse = lambda rc: coarse_bicgstab(coarse, rc, self.coarse_tol, self.coarse_max_iter)[0]
        else:
            from .mglevel import gcr_torch, two_grid_solve_ref
            if coarsest == "lu":
                inner = coarse.solve
            else:
                inner = lambda rc: gcr_torch(coarse.apply, rc, self.coarse_tol, self.coarse_max_iter, 32)[0]  # noqa: E731
            op1, P0, P1, sm1 = ops[1], hierarchy.prolongators[0], hierarchy.prolongators[1], self.smoothers[1]

            def level1(rc):  # native coarse (n, nb, nc) -> reference order, recurse, back
                ref = P0.coarse_to_ref(rc)
                out = torch.empty_like(ref)
                for j in range(ref.shape[0]):
                    out[j] = two_grid_solve_ref(op1, P1, inner, sm1, ref[j].reshape(-1), self.coarse_tol,
                                                max_cycles=self.coarse_max_iter)[0].reshape(ref[j].shape)
                return P0.coarse_from_ref(out)
            self._coarse = level1

    def solve_native(self, b, tol, max_cycles=100):
        h = self.hierarchy
        return two_grid_solve(h.operators[0], h.prolongators[0], self._coarse, self.smoothers[0], b, tol, max_cycles)

    def solve(self, b, tol, max_cycles=100):
        """Reference-layout vector in / out (numpy or CUDA tensor)."""
        op = self.hierarchy.operators[0]
        host = not isinstance(b, torch.Tensor)
        bd = torch.as_tensor(np.asarray(b, dtype=np.complex128)).cuda() if host else b
        x, rep = self.solve_native(op.to_native(bd.reshape(1, -1)), tol, max_cycles)
        xr = op.from_native(x)[0]
        return (xr.cpu().numpy() if host else xr), rep

    def solver_plugin(self):
        """callable(op, b, config) -> (x, SolveReport) for TruncatedInverse
        (experiments.py:55-60)."""
        return lambda _op, b, cfg: self.solve(b, cfg.tol, max_cycles=cfg.max_iter)
