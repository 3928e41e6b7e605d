"""Restated reference Krylov solvers (TEST INFRASTRUCTURE ONLY).

Follows `/root/reference/pkg/src/mgtrace/krylov.py`:
* `gcr_solve` (`:52-118`): restarted flexible GCR with modified Gram-Schmidt
  against the stored (z_j, q_j), breakdown test `||q|| <= 1e-14 ||q0||`
  (`:95-97`), restart by explicit residual when `restart` directions are
  stored (`:107-111`), convergence confirmed on the explicit residual
  (`:78-85`, `:113-118`), matvec accounting as the reference's;
* `TruncatedInverse` counters (`:200-229`).
Pinned against the importable reference in tests/test_oracle_cpu.py.
"""

from dataclasses import dataclass

import numpy as np


@dataclass
class Report:
    iterations: int
    final_relres: float
    converged: bool
    matvecs: int
    reason: str = ""


def gcr(matvec, b, tol, max_iter, restart):
    b = np.asarray(b, dtype=np.complex128)
    bn = np.linalg.norm(b)
    if bn == 0.0:
        return np.zeros_like(b), Report(0, 0.0, True, 0)
    x = np.zeros_like(b)
    r = b.copy()
    nmv = 0
    Z, Q = [], []
    it = 0
    rel = np.linalg.norm(r) / bn
    why = "max_iter"
    while it < max_iter:
        if rel <= tol:
            r = b - matvec(x)
            nmv += 1
            rel = np.linalg.norm(r) / bn
            if rel <= tol:
                return x, Report(it, rel, True, nmv)
            Z, Q = [], []
        z = r.copy()
        q = matvec(z)
        nmv += 1
        q0 = np.linalg.norm(q)
        for zj, qj in zip(Z, Q):
            c = np.vdot(qj, q)
            q = q - c * qj
            z = z - c * zj
        qn = np.linalg.norm(q)
        if qn <= 1e-14 * max(q0, 1e-300):
            why = "breakdown"
            break
        q = q / qn
        z = z / qn
        a = np.vdot(q, r)
        x = x + a * z
        r = r - a * q
        Z.append(z)
        Q.append(q)
        it += 1
        rel = np.linalg.norm(r) / bn
        if len(Z) >= restart:
            Z, Q = [], []
            r = b - matvec(x)
            nmv += 1
            rel = np.linalg.norm(r) / bn
    r = b - matvec(x)
    nmv += 1
    rel = np.linalg.norm(r) / bn
    if rel <= tol:
        return x, Report(it, rel, True, nmv)
    return x, Report(it, rel, False, nmv, why)


class TruncatedInverse:
    def __init__(self, matvec, tol, max_iter=2000, restart=32):
        self.matvec = matvec
        self.tol = tol
        self.max_iter = max_iter
        self.restart = restart
        self.n_solves = 0
        self.total_iterations = 0
        self.n_failed = 0
        self.last_report = None

    def __call__(self, b):
        x, rep = gcr(self.matvec, b, self.tol, self.max_iter, self.restart)
        self.n_solves += 1
        self.total_iterations += rep.iterations
        self.n_failed += 0 if rep.converged else 1
        self.last_report = rep
        return x
