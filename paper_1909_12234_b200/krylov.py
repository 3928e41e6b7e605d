"""GPU Krylov solvers and the truncated inverse A^-1_xi.

Mirrors `mgtrace.krylov` (`/root/reference/pkg/src/mgtrace/krylov.py`):
`SolveConfig` (`:18-29`), `SolveReport` (`:32-38`), the solver-plugin
signature `callable(op, b, config) -> (x, SolveReport)` consumed by
`TruncatedInverse` (`:200-229`, same counters), and the contract of every
converged solve: ||b - A x|| <= tol ||b|| on the explicitly recomputed
residual (`:78-85`, `:113-118`), fresh zero initial guess per application.

The solve itself is `mgt_bicgstab_solve` (C ABI): GPU-resident BiCGStab with
fused reductions, several right-hand sides per call sharing link loads.
BASELINE.json names BiCGStab; the reference's GCR(32) minimises over the same
Krylov space family, so solutions agree to the tolerance (SURVEY.md
finding 6).
"""

import ctypes as ct
import threading
from dataclasses import dataclass

import numpy as np
import torch

from . import _lib
from ._device import device, ptr, stream_ptr, to_device_c128

REASONS = {0: "", 1: "max_iter", 2: "breakdown"}


@dataclass
class SolveConfig:
    tol: float = 1e-8
    max_iter: int = 2000
    restart: int = 32
    kind: str = "bicgstab"  # bicgstab (GPU default) | gmres (restarted GMRES(restart)) | gcr (GCR(restart))
    # BiCGStab on the even-odd Schur complement (same full-residual stopping
    # test; about half the iterations).  False solves the full system.
    even_odd: bool = True
    # mixed precision (even-odd only): fp32 inner BiCGStab cycles inside an
    # fp64 defect correction whose stopping test is the fp64 explicit
    # residual -- the same ||b - A x|| <= tol ||b|| contract, ~1.4x faster
    # per solve at 16^4.  False: fp64 throughout.
    mixed: bool = True

    def __post_init__(self):
        if not (0 < self.tol < 1):
            raise ValueError(f"tol must be in (0,1), got {self.tol}")
        if self.max_iter < 1:
            raise ValueError("max_iter must be >= 1")
        if self.kind not in ("bicgstab", "gmres", "gcr"):
            raise ValueError(f"unknown solver kind {self.kind!r}")


@dataclass
class SolveReport:
    iterations: int
    final_relres: float
    converged: bool
    matvecs: int
    reason: str = ""


def solve_options(config):
    """even_odd / mixed keywords of BiCGStab.solve_native for a config."""
    return {"even_odd": getattr(config, "even_odd", True), "mixed": getattr(config, "mixed", True)}


def _base_operator(op):
    """(WilsonOperator, flags, tau) behind an operator-like object."""
    from .lattice import FormOperator, WilsonOperator
    if isinstance(op, WilsonOperator):
        return op, 0, 0.0
    if isinstance(op, FormOperator):
        return op.op, op.flags, op.tau
    raise TypeError(f"GPU solver needs a WilsonOperator (or a form of one), got {type(op)}")


def solve_batch(volume):
    """Right-hand sides per solver call: groups of 4 rhs are batched into one
    launch per kernel (blockIdx.y) until ~8 resident waves of 148 SMs x 384
    threads are busy (even-odd: V/2 sites per group and rhs), at most 8
    groups.  MGT_SOLVE_BATCH overrides."""
    import os
    if os.environ.get("MGT_SOLVE_BATCH"):
        return max(4, 4 * (int(os.environ["MGT_SOLVE_BATCH"]) // 4))
    want = 8 * 148 * 384
    groups = -(-want // (4 * max(1, volume // 2)))
    return 4 * int(max(1, min(8, groups)))


class BiCGStab:
    """Reusable solver state (device workspace) for one operator; one call
    solves up to `max_rhs` systems (batched groups of 4)."""

    MAX_GROUP = 4

    def __init__(self, op, max_rhs=None):
        self.op, self.flags, self.tau = _base_operator(op)
        if self.op.prec != 64:
            raise ValueError("the Krylov solver runs in complex128")
        self.max_rhs = int(max_rhs) if max_rhs else solve_batch(self.op.volume)
        self.ws_bytes = int(_lib.lib().mgt_bicgstab_workspace_bytes(self.op.handle, self.max_rhs))
        self.workspace = torch.empty(self.ws_bytes, dtype=torch.uint8, device=device())

    def solve_native(self, b, tol, max_iter, x=None, want_dot=False, even_odd=True, mixed=False):
        """Solve A x_r = b_r for native fields b (n, 12, V); returns
        (x, [SolveReport], dots or None) where dots[r] = vdot(b_r, x_r).
        even_odd: solve through the even-odd Schur complement (whenever every
        extent is even); the stopping test is the full residual either way.
        tol: one relative tolerance, or one per rhs (mgt_bicgstab_solve_tols)."""
        n = b.shape[0]
        b = b.contiguous()
        x = torch.empty_like(b) if x is None else x
        rep = (ct.c_int64 * (4 * n))()
        rel = (ct.c_double * n)()
        dots = (ct.c_double * (2 * n))() if want_dot else None
        flags = int(self.flags) | (0 if even_odd else _lib.SOLVE_FULL) | (_lib.SOLVE_MIXED if mixed else 0)
        if np.ndim(tol) == 0:
            rc = _lib.lib().mgt_bicgstab_solve_ws(
                self.op.handle, ptr(b), ptr(x), n, flags, float(self.tau), float(tol), int(max_iter),
                ptr(self.workspace), self.ws_bytes, rep, rel, dots, stream_ptr())
        else:
            tols = np.ascontiguousarray(np.broadcast_to(np.asarray(tol, dtype=np.float64), (n,)))
            rc = _lib.lib().mgt_bicgstab_solve_tols(
                self.op.handle, ptr(b), ptr(x), n, flags, float(self.tau),
                tols.ctypes.data_as(ct.POINTER(ct.c_double)), int(max_iter),
                ptr(self.workspace), self.ws_bytes, rep, rel, dots, stream_ptr())
        _lib.check(rc, "bicgstab")
        reports = []
        for r in range(n):
            it, mv, conv, reason = rep[4 * r:4 * r + 4]
            reports.append(SolveReport(int(it), float(rel[r]), bool(conv), int(mv),
                                       "" if conv else REASONS.get(int(reason), "max_iter")))
        dv = None
        if want_dot:
            dv = np.array([complex(dots[2 * r], dots[2 * r + 1]) for r in range(n)])
        return x, reports, dv


_SOLVERS = {}
_SOLVERS_LOCK = threading.Lock()


def _solver_for(op):
    """One solver (device workspace) per (operator, host thread): concurrent
    solves on several streams never share a workspace."""
    key = (id(op), threading.get_ident())
    with _SOLVERS_LOCK:
        s = _SOLVERS.get(key)
        if s is None or s[0] is not op:
            s = (op, BiCGStab(op))
            _SOLVERS[key] = s
    return s[1]


def release_solvers():
    """Drop every cached solver workspace (and its operator reference);
    the next solve per (operator, thread) allocates afresh."""
    with _SOLVERS_LOCK:
        _SOLVERS.clear()


_KRYLOV_WS = {}


def restarted_solve_native(op, b, config, want_dot=False):
    """GMRES(restart) / GCR(restart) on native fields b (n, 12, V), one rhs
    at a time (C ABI `mgt_gmres_solve` / `mgt_gcr_solve`; zero start,
    explicit-residual stopping test as krylov.py:78-85, 113-118).  Returns
    (x, [SolveReport], dots or None) like BiCGStab.solve_native."""
    base, flags, tau = _base_operator(op)
    kind, m = config.kind, int(config.restart)
    if kind == "gcr" and (flags or tau):
        raise ValueError("the GPU GCR solves the plain operator only (use kind='gmres' for forms of it)")
    key = (id(base), kind, m, threading.get_ident())  # one workspace per host thread (concurrent streams)
    ws = _KRYLOV_WS.get(key)
    if ws is None or ws[0] is not base:
        fn = _lib.lib().mgt_gmres_workspace_bytes if kind == "gmres" else _lib.lib().mgt_gcr_workspace_bytes
        ws = (base, torch.empty(int(fn(base.handle, m)), dtype=torch.uint8, device=device()))
        _KRYLOV_WS[key] = ws
    b = b.contiguous()
    x = torch.empty_like(b)
    reports, dots = [], []
    for r in range(b.shape[0]):
        rep = (ct.c_int64 * 4)()
        rel = (ct.c_double * 1)()
        if kind == "gmres":
            rc = _lib.lib().mgt_gmres_solve(base.handle, ptr(b[r]), ptr(x[r]), m, int(config.max_iter),
                                            float(config.tol), int(flags), float(tau), ptr(ws[1]), rep, rel,
                                            stream_ptr())
        else:
            rc = _lib.lib().mgt_gcr_solve(base.handle, ptr(b[r]), ptr(x[r]), m, int(config.max_iter),
                                          float(config.tol), ptr(ws[1]), rep, rel, stream_ptr())
        _lib.check(rc, kind)
        it, mv, conv, reason = (int(v) for v in rep)
        reports.append(SolveReport(it, float(rel[0]), bool(conv), mv, "" if conv else REASONS.get(reason, "max_iter")))
        if want_dot:
            dots.append(complex(torch.vdot(b[r].reshape(-1), x[r].reshape(-1)).item()))
    return x, reports, (np.array(dots) if want_dot else None)


def bicgstab_solve(op, b, config):
    """Solver plugin `callable(op, b, config) -> (x, SolveReport)`
    (krylov.py:200-229).  b: reference-layout vector (numpy or CUDA tensor)."""
    base, _, _ = _base_operator(op)
    host = not isinstance(b, torch.Tensor)
    bd = to_device_c128(b)
    if bd.shape[0] != base.dim:
        raise ValueError(f"dimension mismatch: {bd.shape[0]} != {base.dim}")
    bn = base.to_native(bd.unsqueeze(0))
    if getattr(config, "kind", "bicgstab") != "bicgstab":
        x, reps, _ = restarted_solve_native(op, bn, config)
    else:
        solver = _solver_for(op)
        x, reps, _ = solver.solve_native(bn, config.tol, config.max_iter, **solve_options(config))
    xr = base.from_native(x)[0]
    return (xr.cpu().numpy() if host else xr), reps[0]


@dataclass
class TruncatedInverse:
    """A^-1_xi: fresh zero-start solve per application; counters as the
    reference's (krylov.py:200-229)."""

    op: object
    config: SolveConfig
    solver: object = None
    n_solves: int = 0
    total_iterations: int = 0
    total_matvecs: int = 0
    n_failed: int = 0
    last_report: SolveReport = None

    def _account(self, rep):
        self.n_solves += 1
        self.total_iterations += rep.iterations
        self.total_matvecs += rep.matvecs
        if not rep.converged:
            self.n_failed += 1
        self.last_report = rep

    def __call__(self, b):
        if self.solver is not None:
            x, rep = self.solver(self.op, b, self.config)
        else:
            x, rep = bicgstab_solve(self.op, b, self.config)
        self._account(rep)
        return x

    def solve_native(self, b, want_dot=False, streams=None):
        """Batched native-layout application (the estimators' fast path).
        More rhs than one solver call takes are split into calls that run
        on `streams` concurrent CUDA streams (default: trace.default_streams
        for the volume); each call's result is a pure function of its rhs,
        so the split does not change any value."""
        if getattr(self.config, "kind", "bicgstab") != "bicgstab":
            x, reps, dots = restarted_solve_native(self.op, b, self.config, want_dot=want_dot)
            for rep in reps:
                self._account(rep)
            return x, reps, dots
        base = _base_operator(self.op)[0]
        max_rhs = solve_batch(base.volume)
        n = b.shape[0]
        chunks = [(r0, min(n, r0 + max_rhs)) for r0 in range(0, n, max_rhs)]
        if streams is None:
            from .trace import default_streams
            streams = default_streams(base.volume, max_rhs)
        ns = max(1, min(int(streams), len(chunks)))
        if threading.current_thread().name.startswith("mgt-solve"):
            ns = 1  # already on a worker stream: never wait on the pool from inside it
        opts = solve_options(self.config)
        if ns == 1:
            solver = _solver_for(self.op)  # (only the calling thread's workspace is allocated)
            results = [solver.solve_native(b[r0:r1], self.config.tol, self.config.max_iter, want_dot=want_dot, **opts)
                       for r0, r1 in chunks]
            xs = [res[0] for res in results]
            x = torch.cat(xs) if len(xs) > 1 else xs[0]
        else:
            from .trace import _worker_pool
            b = b.contiguous()
            x = torch.empty_like(b)
            torch.cuda.current_stream().synchronize()  # b is ready for the worker streams
            dev = torch.cuda.current_device()
            pool, local = _worker_pool(ns)

            def run(r0, r1):
                if getattr(local, "device", None) != dev:
                    torch.cuda.set_device(dev)
                    local.device = dev
                    local.stream = torch.cuda.Stream()
                with torch.cuda.stream(local.stream):
                    res = _solver_for(self.op).solve_native(b[r0:r1], self.config.tol, self.config.max_iter,
                                                            x=x[r0:r1], want_dot=want_dot, **opts)
                    local.stream.synchronize()
                return res

            futs = [pool.submit(run, r0, r1) for r0, r1 in chunks]
            results = [f.result() for f in futs]
        reps, dots = [], []
        for _, rr, d in results:
            reps.extend(rr)
            if want_dot:
                dots.append(d)
        for rep in reps:
            self._account(rep)
        return x, reps, (np.concatenate(dots) if want_dot else None)


def truncated_inverse(op, config, solver=None):
    return TruncatedInverse(op, config, solver=solver)
