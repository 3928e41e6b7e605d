"""Hutchinson trace estimation of A^-1 on the GPU.

Mirrors `mgtrace.trace` (`/root/reference/pkg/src/mgtrace/trace.py`):
`TraceEstimate` (`:40-50`), `jackknife` (`:60-70`), `_finish` (`:73-92`),
per-group slot-order accumulation (`_group_samples`, `:95-113`) and
`hutchinson` (`:122-132`).  The per-slot quadratic form vdot(z, A^-1 z) is
fused into the solver (`mgt_bicgstab_solve` dot epilogue); probes are
generated on the device and solved 4 at a time as one multi-RHS BiCGStab.
Samples are then reduced on the host in the reference's slot order, so the
mean/variance/jackknife arithmetic is identical to the reference's.
"""

import warnings
from dataclasses import dataclass

import numpy as np

from .krylov import TruncatedInverse
from .probing import ProbeSet


class DeflationContractError(ValueError):
    pass


class SpuriousModeError(ValueError):
    def __init__(self, index, lam, lam_max):
        self.index = index
        super().__init__(f"spurious coarse mode {index}: |lambda| = {abs(lam):.3e} "
                         f"< 1e-12 * {lam_max:.3e}; reduce the deflation rank")


@dataclass
class TraceEstimate:
    mean: complex
    samples: np.ndarray
    s: int
    variance: float
    jackknife_err: float
    inversions: int
    t0: complex = 0.0 + 0.0j
    t1: complex = 0.0 + 0.0j
    flagged: np.ndarray = None


def _unbiased_variance(samples):
    n = len(samples)
    if n < 2:
        return 0.0
    dev = samples - samples.mean()
    return float(np.sum(np.abs(dev) ** 2) / (n - 1))


def jackknife(samples):
    """(variance, leave-one-out jackknife error) of the unbiased sample
    variance (trace.py:60-70)."""
    s = np.asarray(samples)
    n = len(s)
    if n < 2:
        raise ValueError("jackknife needs at least 2 samples")
    full = _unbiased_variance(s)
    loo = np.array([_unbiased_variance(np.delete(s, i)) for i in range(n)])
    return full, float(np.sqrt((n - 1) / n * np.sum((loo - loo.mean()) ** 2)))


def finish(t0, samples, inversions, flagged=None):
    samples = np.asarray(samples, dtype=np.complex128)
    s = len(samples)
    t1 = samples.mean() if s else 0.0 + 0.0j
    if s >= 2:
        var, err = jackknife(samples)
        var, err = var / s, err / s
    else:
        var, err = 0.0, 0.0
    return TraceEstimate(mean=complex(t0 + t1), samples=samples, s=s, variance=var, jackknife_err=err,
                         inversions=inversions, t0=complex(t0), t1=complex(t1), flagged=flagged)


def _warn_flagged(flagged):
    if flagged.any():
        warnings.warn(f"{int(flagged.sum())} sample(s) used non-converged solves (kept with TSM semantics)")


def group_samples_gpu(inv_op, probes, batch=4, correction=None):
    """Per-group samples sum_slots w * vdot(slot, A^-1 slot) with the solves
    batched on the GPU; `correction(j, slots_native, x_native)` may return a
    per-slot complex array subtracted from the quadratic forms (deflation).
    Returns (samples, flagged)."""
    ns = probes.sample_count
    samples = np.empty(ns, dtype=np.complex128)
    flagged = np.zeros(ns, dtype=bool)
    w = probes.weights()
    if probes.slots_per_group == 1:
        for j0 in range(0, ns, batch):
            j1 = min(ns, j0 + batch)
            z = probes.noise_native(j0, j1)
            x, reps, q = inv_op.solve_native(z, want_dot=True)
            if correction is not None:
                q = q - correction(j0, z, x)
            for k, j in enumerate(range(j0, j1)):
                acc = 0.0 + 0.0j
                acc = acc + w[0] * q[k]
                samples[j] = acc
                flagged[j] = not reps[k].converged
    else:
        for j in range(ns):
            z = probes.slots_native(j)
            x, reps, q = inv_op.solve_native(z, want_dot=True)
            if correction is not None:
                q = q - correction(j, z, x)
            acc = 0.0 + 0.0j
            for k in range(len(w)):
                acc = acc + w[k] * q[k]
            samples[j] = acc
            flagged[j] = not all(r.converged for r in reps)
    return samples, flagged


def _group_samples_generic(apply_fn, probes, health=None):
    """Reference-order loop for arbitrary callables (trace.py:95-113)."""
    samples = np.empty(probes.sample_count, dtype=np.complex128)
    flagged = np.zeros(probes.sample_count, dtype=bool)
    for gi, g in enumerate(probes.groups):
        acc = 0.0 + 0.0j
        for w, slot in zip(g.weights, g.slots):
            y = apply_fn(slot)
            acc = acc + w * np.vdot(slot, np.asarray(y))
            if health is not None and not health():
                flagged[gi] = True
        samples[gi] = acc
    return samples, flagged


def hutchinson(inv_op, probes):
    """Stochastic trace estimate of the operator behind inv_op
    (trace.py:122-132)."""
    if probes.sample_count == 0:
        raise ValueError("need at least one probe group")
    before = getattr(inv_op, "n_solves", None)
    if isinstance(inv_op, TruncatedInverse) and isinstance(probes, ProbeSet) and inv_op.solver is None:
        samples, flagged = group_samples_gpu(inv_op, probes)
    else:
        health = None
        if isinstance(inv_op, TruncatedInverse):
            health = lambda: inv_op.last_report is None or inv_op.last_report.converged  # noqa: E731
        samples, flagged = _group_samples_generic(inv_op, probes, health)
    _warn_flagged(flagged)
    inversions = inv_op.n_solves - before if before is not None else probes.slot_count
    return finish(0.0, samples, inversions, flagged)
