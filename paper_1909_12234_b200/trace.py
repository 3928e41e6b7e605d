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

import threading
import warnings
from dataclasses import dataclass

import numpy as np

from .krylov import TruncatedInverse
from .probing import ProbeSet


DEFER_BYTES = 16 << 30  # probe fields regenerated at once for a deferred correction pass


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


def _solve_batches_concurrently(inv_op, probes, batches, correction, streams, guess=None):
    """Solve probe batches (one multi-rhs solve each) on `streams` CUDA streams from host
    worker threads: at small volumes one multi-rhs solve cannot fill 148 SMs,
    several independent ones can.  Returns [(reports, q)] in batch order;
    every result is bitwise reproducible; the solves are independent of the
    batching (tile-ordered reductions), the projection corrections' rounding
    depends on the batch width.
    `guess(j0, z) -> (r0, post)` solves A e = r0 = z - A x0 instead (same
    absolute residual bound tol ||z||) and post(e) gives the slots' values."""
    import torch

    import dataclasses

    from .krylov import _solver_for, restarted_solve_native, solve_options

    restarted = getattr(inv_op.config, "kind", "bicgstab") != "bicgstab"

    class _Restarted:  # SolveConfig.kind = gmres / gcr: the restarted C-ABI solvers, one rhs at a time
        @staticmethod
        def solve_native(b, tol, max_iter, want_dot=False, **_):
            cfg = dataclasses.replace(inv_op.config, tol=tol, max_iter=max_iter)
            return restarted_solve_native(inv_op.op, b, cfg, want_dot=want_dot)

    def work(j0, j1, stream):
        with torch.cuda.stream(stream):
            z = probes.noise_native(j0, j1)
            solver = _Restarted if restarted else _solver_for(inv_op.op)
            tol = inv_op.config.tol
            if guess is not None:
                r0, post = guess(j0, z)
                zn = torch.linalg.vector_norm(z.reshape(z.shape[0], -1), dim=1)
                rn = torch.linalg.vector_norm(r0.reshape(r0.shape[0], -1), dim=1)
                ratio = torch.where(rn > 0, rn / zn, torch.ones_like(rn)).cpu().numpy()
                # per rhs: ||r0_i - A e_i|| <= tol ||z_i||  <=>  relative tol ||z_i|| / ||r0_i|| on r0_i
                tols = np.minimum(0.99, tol / ratio) if not restarted else min(0.99, tol / float(ratio.max()))
                e, reps, _ = solver.solve_native(r0, tols, inv_op.config.max_iter, **solve_options(inv_op.config))
                for rep, f in zip(reps, ratio):  # residuals relative to the probe, as the reference's
                    rep.final_relres *= float(f)
                    rep.converged = rep.final_relres <= tol
                q = post(e)
            else:
                x, reps, q = solver.solve_native(z, tol, inv_op.config.max_iter, want_dot=True,
                                                 **solve_options(inv_op.config))
                if correction is not None:
                    q = q - correction(j0, z, x)
            stream.synchronize()
        return reps, q

    n = max(1, min(streams, len(batches)))
    if n == 1:
        return [work(j0, j1, torch.cuda.current_stream()) for j0, j1 in batches]
    torch.cuda.current_stream().synchronize()  # shared inputs (deflation factors) are ready
    dev = torch.cuda.current_device()
    pool, local = _worker_pool(n)

    def run(j0, j1):
        if getattr(local, "device", None) != dev:  # one stream per worker thread and device
            torch.cuda.set_device(dev)
            local.device = dev
            local.stream = torch.cuda.Stream()
        return work(j0, j1, local.stream)

    futs = [pool.submit(run, j0, j1) for j0, j1 in batches]
    return [f.result() for f in futs]


_POOL = {}


def _worker_pool(n):
    """Process-wide worker threads (stable identities, so their solver
    workspaces and cached solver graphs are reused across calls)."""
    import concurrent.futures as cf
    if n not in _POOL:
        _POOL[n] = (cf.ThreadPoolExecutor(max_workers=n, thread_name_prefix="mgt-solve"), threading.local())
    return _POOL[n]


def default_streams(volume, batch=4):
    """Concurrent multi-rhs solves: one even-odd solve of `batch` rhs on V
    sites exposes batch V/2 stencil threads per kernel; ~32 resident waves
    of 148 SMs x 384 threads in flight hide the per-kernel launch/tail gaps
    and the host-side status polls (measured on B200, tools/batch_sweep.sh:
    16^4 best at 16 rhs x 4 streams, 8^4 at 32 rhs x 1).  Where one solve
    already fills the GPU (32^4, 32^3 x 64) two solves still pay: one's
    latency-bound stencil kernels overlap the other's HBM-bound vector
    kernels (tools/streams_probe.py: +17-18 % probes/s); above 2^22 sites
    the second workspace is not worth its memory."""
    import os
    if os.environ.get("MGT_SOLVE_STREAMS"):
        return max(1, int(os.environ["MGT_SOLVE_STREAMS"]))
    want = 32 * 148 * 384
    n = int(max(1, min(8, -(-want // (batch * max(1, volume // 2))))))
    if n == 1 and volume <= (1 << 22):
        n = 2
    return n


def group_samples_gpu(inv_op, probes, batch=None, correction=None, streams=None, deferred=None, guess=None):
    """Per-group samples sum_slots w * vdot(slot, A^-1 slot) with the solves
    batched on the GPU; `correction(j, slots_native, x_native)` may return a
    per-slot complex array subtracted from the quadratic forms (deflation).
    `deferred = (collect, finish)` instead calls collect(j, slots, x) per
    batch and finish() once -> per-slot corrections in slot order (one large
    product instead of one per batch).  The samples are accumulated exactly
    as the reference's slot loop (trace.py:100-107).  Returns (samples,
    flagged)."""
    ns = probes.sample_count
    flagged = np.zeros(ns, dtype=bool)
    w = probes.weights()
    per_group = []  # (reports, q) per group, q per slot
    if deferred is not None:
        correction = lambda j0, z, x: deferred[0](j0, z, x) or 0.0  # noqa: E731
    if probes.slots_per_group == 1:
        if batch is None:
            from .krylov import solve_batch
            batch = solve_batch(probes.geometry.site_count)
        batches = [(j0, min(ns, j0 + batch)) for j0 in range(0, ns, batch)]
        if streams is None:
            streams = default_streams(probes.geometry.site_count, batch)
        results = _solve_batches_concurrently(inv_op, probes, batches, correction, streams, guess)
        for (j0, j1), (reps, q) in zip(batches, results):
            for k in range(j1 - j0):
                per_group.append(([reps[k]], np.atleast_1d(q[k])))
    else:
        for j in range(ns):
            z = probes.slots_native(j)
            x, reps, q = inv_op.solve_native(z, want_dot=True)
            if correction is not None:
                q = q - correction(j, z, x)
            per_group.append((reps, q))
    if deferred is not None:
        corr = deferred[1]()
        pos = 0
        for g, (reps, q) in enumerate(per_group):
            per_group[g] = (reps, q - corr[pos:pos + len(q)])
            pos += len(q)
    samples = np.empty(ns, dtype=np.complex128)
    for j, (reps, q) in enumerate(per_group):
        if probes.slots_per_group == 1:
            for rep in reps:  # counters in probe order, as the reference's
                inv_op._account(rep)
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


def deflate_orthogonal(inv_op, U, probes, op=None, guess=False):
    """Algorithm-1 trace estimate with the orthogonal projector of U
    (trace.py:161-188): t0 = sum_i u_i^H A^-1 u_i and per slot
    z^H (A^-1 z - Y U^H z) = q - (Y^H z)^H (U^H z), Y = A^-1 U solved once.

    guess=True (single-slot probe groups; off by default, the reference
    solves from zero): every probe solve starts from the deflated guess
    x0 = Y (U^H z), i.e. solves A e = z - A x0 to the same residual bound
    tol ||z|| per probe (per-rhs tolerance tol ||z_i|| / ||r0_i||), and the
    slot value is z^H e -- the same quantity (z^H (x - Y U^H z) with
    x = x0 + e), O(xi) apart from the zero-start form; the low modes of the
    start residual are gone, ~11 % fewer iterations at 16^4 with k = 64.

    U: native fields (k, 12, V) CUDA tensor, or reference-layout (N, k)
    array/tensor (then `op` or inv_op.op converts the layout)."""
    import torch
    from .linalg import vhx
    before = getattr(inv_op, "n_solves", 0)
    base = op if op is not None else inv_op.op
    if not (isinstance(U, torch.Tensor) and U.dim() == 3):
        Ut = torch.as_tensor(np.ascontiguousarray(np.asarray(U).T)) if not isinstance(U, torch.Tensor) \
            else U.transpose(0, 1).contiguous()
        U = base.to_native(Ut.to(torch.complex128).cuda()) if Ut.numel() else None
    k = 0 if U is None else U.shape[0]
    if k == 0:
        samples, flagged = group_samples_gpu(inv_op, probes)
        _warn_flagged(flagged)
        return finish(0.0, samples, (inv_op.n_solves - before) or probes.slot_count, flagged)
    gram = vhx(U, U) - torch.eye(k, dtype=torch.complex128, device=U.device)
    gmax = gram.abs().max().item()
    if gmax > 1e-6:
        raise DeflationContractError(f"U not orthonormal: ||U^dag U - I||_max = {gmax:.3e}")
    Y, _, _ = inv_op.solve_native(U)
    t0 = complex(torch.diagonal(vhx(U, Y)).sum().item())

    def correction(j0, z, x):
        a = vhx(U, z)  # (k, n)  U^H z
        h = vhx(Y, z)  # (k, n)  Y^H z
        return torch.sum(h.conj() * a, dim=0).cpu().numpy()

    use_guess = guess and probes.slots_per_group == 1 and isinstance(inv_op, TruncatedInverse) \
        and inv_op.solver is None
    if use_guess:
        from .krylov import _base_operator
        bop, flags, tau = _base_operator(inv_op.op)

        def start(j0, z):
            x0 = torch.einsum("kn,kcv->ncv", vhx(U, z), Y)  # Y (U^H z)
            r0 = (z - bop.apply_native(x0, flags=flags, tau=tau)).contiguous()

            def post(e):
                return torch.sum(z.conj() * e, dim=(1, 2)).cpu().numpy()
            return r0, post

        samples, flagged = group_samples_gpu(inv_op, probes, guess=start)
        _warn_flagged(flagged)
        return finish(t0, samples, inv_op.n_solves - before, flagged)
    if probes.slots_per_group == 1:
        # the corrections need only the probes: regenerate them from their
        # seeds after the solves and project them in a few wide products
        # (cuBLAS ZGEMM for s >= 32) instead of two skinny projections per
        # solve batch inside the concurrent solve streams
        def finish_corr():
            n = probes.sample_count
            out = np.empty(n, dtype=np.complex128)
            per = max(1, int(DEFER_BYTES // max(1, 16 * base.dim)))
            for j0 in range(0, n, per):
                j1 = min(n, j0 + per)
                out[j0:j1] = correction(j0, probes.noise_native(j0, j1), None)
            return out

        samples, flagged = group_samples_gpu(inv_op, probes, deferred=(lambda j0, z, x: None, finish_corr))
    else:
        samples, flagged = group_samples_gpu(inv_op, probes, correction=correction)
    _warn_flagged(flagged)
    return finish(t0, samples, inv_op.n_solves - before, flagged)


@dataclass
class ObliqueFactors:
    """Small factors of the coarse oblique deflation (trace.py:191-204)."""

    rank: int
    lam: np.ndarray
    uhat: np.ndarray
    s_small: np.ndarray
    t_small: np.ndarray
    t0: complex

    def minv(self):
        return self.uhat @ np.diag(1.0 / self.lam) @ self.uhat.conj().T


def factorize_small(s_small, t_small):
    """trace.py:207-217: eigh of the Hermitian part, |lambda| ascending,
    spurious-mode guard, t0 = tr(Uhat^H T Uhat Lam^-1)."""
    k = s_small.shape[0]
    lam, uhat = np.linalg.eigh(0.5 * (s_small + s_small.conj().T))
    order = np.argsort(np.abs(lam), kind="stable")
    lam, uhat = lam[order], uhat[:, order]
    lam_max = np.abs(lam).max() if k else 0.0
    for i, l in enumerate(lam):
        if abs(l) < 1e-12 * lam_max:
            raise SpuriousModeError(i, l, lam_max)
    t0 = complex(np.trace(uhat.conj().T @ t_small @ uhat @ np.diag(1.0 / lam))) if k else 0j
    return lam, uhat, t0


class IdentityTriplets:
    """Full coarse space: Ubar = I (rank = Nc), i.e. deflation with V = P
    (SURVEY.md finding 8)."""

    def __init__(self, n):
        self.count = n


def _full_coarse_deflation(op, inv_op, prolongator, probes, coarse_op):
    """rank = Nc, Ubar = I: t0 = tr(C^-1); per slot
    z^H A^-1 z - (P^H z)^H C^-1 (P^H z)  (Y = A^-1 (A P) = P)."""
    import torch
    from .multigrid import build_coarse_operator
    coarse = coarse_op if coarse_op is not None else build_coarse_operator(op, prolongator)
    cinv = coarse.exact_inverse()  # setup, cached on the coarse operator (coarse Schur or dense LU)
    t0 = cinv.t0
    Nc = prolongator.coarse_dim
    store = {}

    def restrict(j0, z, x):  # per batch: keep P^H z (Nc complex per probe)
        store[j0] = prolongator.restrict_native(z).reshape(z.shape[0], Nc)

    def corrections():
        # one (s x Nc) x (Nc x Nc) product for all probes: C^-1 is read once
        keys = sorted(store)
        H = torch.cat([store[k] for k in keys])
        CH = cinv.apply_rows(H)
        return torch.sum(H.conj() * CH, dim=1).cpu().numpy()

    return t0, (restrict, corrections)


def coarse_deflation_triplets(coarse_op, k, tol=1e-2, tau=0.0, inner_tol=1e-2, max_iter=2000, max_basis=0, block=1):
    """Algorithm-2 line 2 (experiments.py:65-74): inexact Davidson on the
    coarse operator (GPU coarse BiCGStab inner solves), converted to singular
    triplets whose vectors are native coarse fields.  block > 1 runs the
    block Davidson (batched coarse solves)."""
    from . import eigen as E
    from .krylov import SolveConfig
    conf = E.EigenConfig(k=k, tol=tol, tau=tau, max_basis=max_basis, block=block,
                         inner=SolveConfig(tol=inner_tol, max_iter=max_iter))
    res = E.inexact_eigensolve(coarse_op, coarse_op.gamma5_diag, conf, E.shift_inverter_factory(coarse_op, conf.inner))
    return E.to_singular_triplets(res), res


def deflate_oblique_coarse(op, inv_op, prolongator, coarse_triplets, rank, probes, coarse_op=None):
    """Algorithm-2 trace estimate (trace.py:236-274) on the GPU.

    rank = Nc with identity triplets (`IdentityTriplets`, or None) is the
    full-prolongator deflation of BASELINE configs 3/5; otherwise the
    reference's rank-r decoupled form with Y = A^-1_xi (A W Ubar) solved
    once (r fine solves)."""
    import torch
    before = getattr(inv_op, "n_solves", 0)
    if rank == 0:
        samples, flagged = group_samples_gpu(inv_op, probes)
        _warn_flagged(flagged)
        return finish(0.0, samples, inv_op.n_solves - before, flagged)
    if coarse_triplets is None or isinstance(coarse_triplets, IdentityTriplets):
        if rank != prolongator.coarse_dim:
            raise ValueError("identity coarse triplets need rank = Nc")
        t0, corr = _full_coarse_deflation(op, inv_op, prolongator, probes, coarse_op)
        samples, flagged = group_samples_gpu(inv_op, probes, deferred=corr)
        _warn_flagged(flagged)
        return finish(t0, samples, inv_op.n_solves - before, flagged)
    if rank > coarse_triplets.count:
        raise ValueError(f"rank {rank} exceeds the {coarse_triplets.count} available triplets")
    # rank-r form (trace.py:220-233, :251-271)
    fac, ubn, Y = _oblique_setup(op, inv_op, prolongator, coarse_triplets, rank)
    minv = torch.as_tensor(fac.minv(), device=Y.device)
    pr = prolongator

    def correction(j0, z, x):
        g, h = _oblique_gh(pr, ubn, Y, z)
        return torch.sum(h.conj() * (g @ minv.T), dim=1).cpu().numpy()

    if probes.slots_per_group == 1:
        # the corrections need only the probes, which are regenerated from
        # their seeds: one pass over Y (r fine fields, 25.7 GB at 32^3 x 64,
        # r = 64) and P per DEFER_BATCH probes instead of per solve batch
        done = []

        def collect(j0, z, x):
            done.append((j0, z.shape[0]))

        def finish_corr():
            n = probes.sample_count
            out = np.empty(n, dtype=np.complex128)
            per = max(1, int(DEFER_BYTES // max(1, 16 * op.dim)))
            for j0 in range(0, n, per):
                j1 = min(n, j0 + per)
                out[j0:j1] = correction(j0, probes.noise_native(j0, j1), None)
            return out

        samples, flagged = group_samples_gpu(inv_op, probes, deferred=(collect, finish_corr))
    else:
        samples, flagged = group_samples_gpu(inv_op, probes, correction=correction)
    _warn_flagged(flagged)
    return finish(fac.t0, samples, inv_op.n_solves - before, flagged)


def _oblique_setup(op, inv_op, pr, coarse_triplets, rank):
    """oblique_factors (trace.py:220-233) + Y = A^-1_xi (A W Ubar) (:252):
    returns (ObliqueFactors, Ubar as native coarse fields (r, nb, 2nv), Y)."""
    import torch
    dev = pr.P.device
    left = coarse_triplets.left
    if isinstance(left, torch.Tensor):  # GPU triplets: native coarse fields (r, nb, 2nv)
        ubn = left[:rank].contiguous()
        ubar = pr.coarse_to_ref(ubn).reshape(rank, -1).T.cpu().numpy()
    else:  # reference triplets: (Nc, r) in the reference coarse order
        ubar = np.asarray(left)[:, :rank]
        ub = torch.as_tensor(np.ascontiguousarray(ubar.T), device=dev)
        ubn = pr.coarse_from_ref(ub.reshape(rank, pr.n_blocks, pr.nc))
    wu = pr.prolong_native(ubn)  # W Ubar, (r, 12, V)
    g_cols = op.apply_native(wu)  # A W Ubar
    # S = (W Ubar)^H g5 (A W Ubar) with the projection kernel; g5 flips the
    # sign of comps 6..11 in place (exact) and back, so no r-field temporary
    from .linalg import vhx
    g_cols[:, 6:].neg_()
    s_small = vhx(wu, g_cols).cpu().numpy()
    g_cols[:, 6:].neg_()
    del wu  # r fine fields (25.8 GB at 32^3 x 64, r = 64): not needed past S
    g5c = pr.coarse_gamma5
    t_small = ubar.conj().T @ (g5c[:, None] * ubar)
    lam, uhat, t0 = factorize_small(s_small, t_small)
    Y, _, _ = inv_op.solve_native(g_cols)
    return ObliqueFactors(rank, lam, uhat, s_small, t_small, t0), ubn, Y


def _oblique_gh(pr, ubn, Y, z):
    """Per slot g = Ubar^H (W^H (g5 z)) and h = Y^H z (trace.py:266-267), (n, r) each."""
    n, r = z.shape[0], ubn.shape[0]
    g = pr.restrict_native(z, gamma5_in=True).reshape(n, -1) @ ubn.reshape(r, -1).conj().T
    h = z.reshape(n, -1) @ Y.reshape(r, -1).conj().T
    return g, h


@dataclass
class PosteriorAnalysis:
    """Small products of one expensive solve pass (trace.py:277-331): per
    slot q = z^H A^-1 z, H = Y^H Z, G = Ubar^H W^H g5 Z and the k_max x k_max
    small matrices; the deflated estimate at any rank <= k_max follows by
    small dense algebra."""

    rank_grid: list
    k_max: int
    weights: list
    q: list
    h: list
    g: list
    s_small: np.ndarray
    t_small: np.ndarray
    inversions: int
    variances: dict = None
    estimates: dict = None
    errors: dict = None

    def __post_init__(self):
        self.variances = {} if self.variances is None else self.variances
        self.estimates = {} if self.estimates is None else self.estimates
        self.errors = {} if self.errors is None else self.errors

    def storage_entries(self):
        n = self.s_small.size + self.t_small.size
        for qs, hs, gs, ws in zip(self.q, self.h, self.g, self.weights):
            n += qs.size + hs.size + gs.size + ws.size
        return n

    def factors_at(self, rank):
        lam, uhat, t0 = factorize_small(self.s_small[:rank, :rank], self.t_small[:rank, :rank])
        return ObliqueFactors(rank, lam, uhat, self.s_small[:rank, :rank], self.t_small[:rank, :rank], t0)

    def samples_at(self, rank):
        minv = None if rank == 0 else self.factors_at(rank).minv()
        out = np.empty(len(self.q), dtype=np.complex128)
        for gi, (qs, hs, gs, ws) in enumerate(zip(self.q, self.h, self.g, self.weights)):
            acc = 0.0 + 0.0j
            for si in range(len(qs)):
                if rank == 0:
                    acc = acc + ws[si] * qs[si]
                else:
                    acc = acc + ws[si] * (qs[si] - np.vdot(hs[si, :rank], minv @ gs[si, :rank]))
            out[gi] = acc
        return out

    def estimate_at(self, rank):
        t0 = self.factors_at(rank).t0 if rank else 0.0 + 0.0j
        return finish(t0, self.samples_at(rank), self.inversions)


def posterior_rank_sweep(op, inv_op, prolongator, coarse_triplets, probes, rank_grid):
    """One pass of expensive solves, then the deflated estimate at every rank
    of rank_grid (trace.py:334-385)."""
    rank_grid = sorted(set(int(r) for r in rank_grid))
    if any(r < 0 for r in rank_grid):
        raise ValueError("ranks must be >= 0")
    k_max = max(rank_grid)
    if k_max > coarse_triplets.count:
        raise ValueError(f"rank grid up to {k_max} exceeds the {coarse_triplets.count} stored triplets")
    before = getattr(inv_op, "n_solves", 0)
    if k_max > 0:
        fac, ubn, Y = _oblique_setup(op, inv_op, prolongator, coarse_triplets, k_max)
        s_small, t_small = fac.s_small, fac.t_small
    else:
        s_small = t_small = np.zeros((0, 0), dtype=np.complex128)
    store = {}

    def collect(j0, z, x):
        if k_max > 0:
            g, h = _oblique_gh(prolongator, ubn, Y, z)
            store[j0] = (h.cpu().numpy(), g.cpu().numpy())
        return None

    ns = probes.sample_count
    w = probes.weights()
    qs, hs, gs, ws = [], [], [], []
    if probes.slots_per_group == 1:
        batches = [(j0, min(ns, j0 + 4)) for j0 in range(0, ns, 4)]
        results = _solve_batches_concurrently(inv_op, probes, batches, lambda j0, z, x: collect(j0, z, x) or 0.0,
                                              default_streams(probes.geometry.site_count))
        for (j0, j1), (reps, q) in zip(batches, results):
            for rep in reps:
                inv_op._account(rep)
            for k in range(j1 - j0):
                qs.append(np.array([q[k]]))
                if k_max > 0:
                    hs.append(store[j0][0][k:k + 1])
                    gs.append(store[j0][1][k:k + 1])
                else:
                    hs.append(np.zeros((1, 0), dtype=np.complex128))
                    gs.append(np.zeros((1, 0), dtype=np.complex128))
                ws.append(np.array(w))
    else:
        for j in range(ns):
            z = probes.slots_native(j)
            x, reps, q = inv_op.solve_native(z, want_dot=True)
            collect(j, z, x)
            qs.append(np.asarray(q))
            hs.append(store[j][0] if k_max > 0 else np.zeros((len(q), 0), dtype=np.complex128))
            gs.append(store[j][1] if k_max > 0 else np.zeros((len(q), 0), dtype=np.complex128))
            ws.append(np.array(w))
    inversions = inv_op.n_solves - before
    post = PosteriorAnalysis(rank_grid, k_max, ws, qs, hs, gs, s_small, t_small, inversions)
    for r in rank_grid:
        est = post.estimate_at(r)
        post.variances[r] = est.variance
        post.estimates[r] = est.mean
        post.errors[r] = est.jackknife_err
    return post


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


def tsm_correction(op, xi_low, xi_high, s_corr, seed, kind="z4", solver=None, max_iter=5000):
    """Truncated-solver bias correction (trace.py:388-407): the mean over
    s_corr noise vectors (seeds seed .. seed+s_corr-1) of
    z^H (A^-1_{xi_high} z - A^-1_{xi_low} z).  Both solves run on the GPU in
    batches with the quadratic forms fused into the solver; the solver is
    deterministic, so xi_high == xi_low returns exactly 0."""
    if xi_high > xi_low:
        raise ValueError("expected xi_high <= xi_low (xi_high is the tighter tolerance)")
    from .krylov import SolveConfig
    from .probing import build_probe_set
    if solver is not None:
        raise NotImplementedError("tsm_correction runs the GPU BiCGStab; custom solver plugins are not supported")
    inv_hi = TruncatedInverse(op, SolveConfig(tol=xi_high, max_iter=max_iter))
    inv_lo = TruncatedInverse(op, SolveConfig(tol=xi_low, max_iter=max_iter))
    probes = build_probe_set(op.geometry, 12, s_corr, hp_count=1, dilution=False, kind=kind, seed=seed)
    qs = []
    for j0 in range(0, s_corr, 4):
        j1 = min(s_corr, j0 + 4)
        z = probes.noise_native(j0, j1)
        _, _, q_hi = inv_hi.solve_native(z, want_dot=True)
        _, _, q_lo = inv_lo.solve_native(z, want_dot=True)
        qs.append(np.asarray(q_hi) - np.asarray(q_lo))
    samples = np.concatenate(qs) if qs else np.zeros(0, dtype=np.complex128)
    return finish(0.0, samples, inv_hi.n_solves + inv_lo.n_solves).mean


def orthogonal_rank_sweep(inv_op, U, lefts_inv, probes, rank_grid, op=None):
    """Per-rank orthogonally deflated estimates from ONE set of undeflated
    probe solves (experiments.py:205-243): U (k columns, ascending singular
    value) and lefts_inv = A^-1_xi U as reference-layout (N, k) arrays or
    native (k, 12, V) tensors.  Per slot the GPU solve returns q = z^H A^-1 z
    (fused), and a = U^H z, ybar = lefts^H z come from the projection kernel;
    rank r uses q - sum_{i<r} conj(ybar_i) a_i and t0 = sum_{i<r} u_i^H l_i.
    Returns {rank: TraceEstimate}."""
    import torch
    from .linalg import vhx
    base = op if op is not None else inv_op.op
    rank_grid = sorted(set(int(r) for r in rank_grid))
    k_max = max(rank_grid)

    def native(M):
        if isinstance(M, torch.Tensor) and M.dim() == 3:
            return M
        Mt = torch.as_tensor(np.ascontiguousarray(np.asarray(M).T)) if not isinstance(M, torch.Tensor) \
            else M.transpose(0, 1).contiguous()
        return base.to_native(Mt.to(torch.complex128).cuda())

    U, L = native(U), native(lefts_inv)
    if k_max > U.shape[0]:
        raise ValueError("rank grid exceeds available vectors")
    U, L = U[:k_max], L[:k_max]
    t0_terms = torch.diagonal(vhx(U, L)).cpu().numpy() if k_max else np.zeros(0, dtype=np.complex128)
    per_group = []
    w = probes.weights()

    def collect(z, n_groups):
        _, _, q = inv_op.solve_native(z, want_dot=True)
        a = vhx(U, z).cpu().numpy() if k_max else np.zeros((0, z.shape[0]), dtype=np.complex128)
        yb = vhx(L, z).cpu().numpy() if k_max else np.zeros((0, z.shape[0]), dtype=np.complex128)
        per = z.shape[0] // n_groups
        for gidx in range(n_groups):
            sl = slice(gidx * per, (gidx + 1) * per)
            per_group.append((np.asarray(q)[sl], a[:, sl].T, yb[:, sl].T))

    ns = probes.sample_count
    if probes.slots_per_group == 1:
        for j0 in range(0, ns, 4):
            j1 = min(ns, j0 + 4)
            collect(probes.noise_native(j0, j1), j1 - j0)
    else:
        for j in range(ns):
            collect(probes.slots_native(j), 1)
    out = {}
    for r in rank_grid:
        samples = np.empty(len(per_group), dtype=np.complex128)
        for gi, (q, a, yb) in enumerate(per_group):
            acc = 0.0 + 0.0j
            for si in range(len(q)):
                if r == 0:
                    acc = acc + w[si] * q[si]
                else:
                    acc = acc + w[si] * (q[si] - np.sum(np.conj(yb[si, :r]) * a[si, :r]))
            samples[gi] = acc
        t0 = complex(np.sum(t0_terms[:r])) if r else 0.0 + 0.0j
        out[r] = finish(t0, samples, probes.slot_count + r)
    return out

