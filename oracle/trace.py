"""Restated reference estimators (TEST INFRASTRUCTURE ONLY).

Follows `/root/reference/pkg/src/mgtrace/trace.py`: `_unbiased_variance`
(`:53-57`), `jackknife` (`:60-70`), `_finish` (`:73-92`), slot-order group
accumulation (`:95-113`), `hutchinson` (`:122-132`), `deflate_orthogonal`
(`:161-188`) and the full-V coarse form of `deflate_oblique_coarse`
(`:236-274` with identity coarse triplets and rank = Nc; SURVEY.md
finding 8: t0 = tr(C^-1), sample = z^H A^-1 z - (P^H z)^H C^-1 (P^H z) when
Y = A^-1 (A P) = P).
"""

import numpy as np


def unbiased_variance(s):
    if len(s) < 2:
        return 0.0
    m = s.mean()
    return float(np.sum(np.abs(s - m) ** 2) / (len(s) - 1))


def jackknife(samples):
    s = np.asarray(samples)
    n = len(s)
    full = unbiased_variance(s)
    loo = np.array([unbiased_variance(np.delete(s, i)) for i in range(n)])
    return full, float(np.sqrt((n - 1) / n * np.sum((loo - loo.mean()) ** 2)))


def finish(t0, samples):
    samples = np.asarray(samples, dtype=np.complex128)
    s = len(samples)
    t1 = samples.mean() if s else 0j
    var, err = (0.0, 0.0)
    if s >= 2:
        var, err = jackknife(samples)
        var, err = var / s, err / s
    return {"mean": complex(t0 + t1), "samples": samples, "variance": var, "jackknife_err": err,
            "t0": complex(t0), "t1": complex(t1)}


def hutchinson(inv, probe_slots, weights=None):
    """probe_slots: list (per group) of lists of slot vectors."""
    samples = []
    for g, slots in enumerate(probe_slots):
        w = np.ones(len(slots)) if weights is None else weights
        acc = 0.0 + 0.0j
        for wk, z in zip(w, slots):
            acc = acc + wk * np.vdot(z, inv(z))
        samples.append(acc)
    return finish(0.0, samples)


def deflate_orthogonal(inv, U, probe_slots):
    k = U.shape[1]
    Y = np.column_stack([inv(U[:, i]) for i in range(k)])
    t0 = complex(np.einsum("ij,ij->", U.conj(), Y))
    samples = []
    for slots in probe_slots:
        acc = 0.0 + 0.0j
        for z in slots:
            acc = acc + 1.0 * np.vdot(z, inv(z) - Y @ (U.conj().T @ z))
        samples.append(acc)
    return finish(t0, samples)


def deflate_full_coarse(inv, P, C_dense, probe_slots):
    Cinv = np.linalg.inv(C_dense)
    t0 = complex(np.trace(Cinv))
    samples = []
    for slots in probe_slots:
        acc = 0.0 + 0.0j
        for z in slots:
            h = P.conj().T @ z
            acc = acc + 1.0 * (np.vdot(z, inv(z)) - np.vdot(h, Cinv @ h))
        samples.append(acc)
    return finish(t0, samples)
