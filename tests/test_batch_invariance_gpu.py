"""A probe's solve does not depend on the batch it is solved in.

The solver's reductions are tile-ordered (csrc/reduce.cuh): every sum over
sites is defined by the ordered-site index alone, not by how many rhs share a
launch (NR = 1, 2, 4), how many groups are batched (blockIdx.y) or the grid
size.  So the same probe solved alone, in a pair, in a group of 4 or in a
batch of 8 + 1 gives bitwise the same solution and quadratic form -- which is
what makes a probe-sharded estimate (distributed.sharded_estimate) bitwise
equal to the single-GPU one.
"""

import numpy as np
import pytest

from oracle import pcg64 as P

pytestmark = pytest.mark.gpu


def _solve_in_batches(M, op, z, sizes, mode):
    import torch
    from paper_1909_12234_b200.krylov import BiCGStab
    solver = BiCGStab(op, max_rhs=max(sizes))
    xs, qs, its = [], [], []
    j = 0
    for n in sizes:
        b = z[j:j + n]
        x, reps, q = solver.solve_native(b, 1e-9, 500, want_dot=True, **mode)
        assert all(r.converged for r in reps)
        xs.append(x.clone())
        qs.extend(q)
        its.extend(r.iterations for r in reps)
        j += n
    torch.cuda.synchronize()
    return torch.cat(xs), np.array(qs), its


@pytest.mark.parametrize("dims", [(4, 6, 6, 10), (8, 8, 8, 8)])
@pytest.mark.parametrize("mode", [dict(even_odd=True, mixed=True), dict(even_odd=True, mixed=False),
                                  dict(even_odd=False, mixed=False)], ids=["mixed", "eo64", "full64"])
def test_probe_result_independent_of_batch(cuda, dims, mode):
    import torch
    import paper_1909_12234_b200 as M
    geo = M.LatticeGeometry(dims, "antiperiodic")
    op = M.build_wilson(M.generate_gauge(geo, "su3", eps=0.3, seed=3), 0.1)
    N = op.dim
    s = 9
    z = op.to_native(torch.as_tensor(np.stack([P.rademacher_numpy(N, 40 + j) for j in range(s)])).cuda())
    ref_x, ref_q, ref_it = _solve_in_batches(M, op, z, [9], mode)          # 2 groups of 4 + 1
    for sizes in ([1] * 9, [2, 2, 2, 2, 1], [4, 4, 1], [4, 3, 2], [8, 1]):
        x, q, it = _solve_in_batches(M, op, z, sizes, mode)
        assert it == ref_it, sizes
        assert torch.equal(x, ref_x), sizes
        assert np.array_equal(q.view(np.float64), ref_q.view(np.float64)), sizes


def test_sharded_hutchinson_bitwise_equals_single(cuda):
    """Probe shards of different sizes (the bench's probe sharding) give the
    per-probe samples of the single-GPU run bitwise."""
    import paper_1909_12234_b200 as M
    dims = (8, 8, 8, 8)
    geo = M.LatticeGeometry(dims, "antiperiodic")
    op = M.build_wilson(M.generate_gauge(geo, "su3", eps=0.2, seed=0), 0.1)
    inv = M.TruncatedInverse(op, M.SolveConfig(tol=1e-8))
    full = M.hutchinson(inv, M.build_probe_set(geo, 12, 12, hp_count=1, dilution=False, kind="rademacher", seed=5))
    parts = []
    for j0, j1 in ((0, 5), (5, 6), (6, 12)):
        est = M.hutchinson(inv, M.build_probe_set(geo, 12, j1 - j0, hp_count=1, dilution=False,
                                                  kind="rademacher", seed=5 + j0))
        parts.append(est.samples)
    got = np.concatenate(parts)
    assert np.array_equal(got.view(np.float64), np.asarray(full.samples).view(np.float64))


@pytest.mark.parametrize("mixed", [True, False], ids=["mixed", "eo64"])
def test_per_rhs_tolerances(cuda, mixed):
    """mgt_bicgstab_solve_tols: rhs r stops at its own tolerance, bitwise as
    if it had been solved alone with that scalar tolerance."""
    import torch
    import paper_1909_12234_b200 as M
    from paper_1909_12234_b200.krylov import BiCGStab
    geo = M.LatticeGeometry((4, 6, 6, 10), "antiperiodic")
    op = M.build_wilson(M.generate_gauge(geo, "su3", eps=0.3, seed=3), 0.1)
    N = op.dim
    tols = np.array([1e-4, 1e-8, 1e-6, 1e-10, 1e-5, 1e-9])
    z = op.to_native(torch.as_tensor(np.stack([P.rademacher_numpy(N, 60 + j) for j in range(len(tols))])).cuda())
    solver = BiCGStab(op, max_rhs=8)
    x, reps, q = solver.solve_native(z, tols, 800, want_dot=True, mixed=mixed)
    assert all(r.converged for r in reps)
    assert all(r.final_relres <= t for r, t in zip(reps, tols))
    its = [r.iterations for r in reps]
    assert its[3] > its[1] > its[2] >= its[4] >= its[0] and its[3] >= its[5] >= its[1]
    for j, t in enumerate(tols):
        xj, rj, qj = solver.solve_native(z[j:j + 1], float(t), 800, want_dot=True, mixed=mixed)
        assert rj[0].iterations == its[j]
        assert torch.equal(xj[0], x[j])
        assert qj[0] == q[j]
    with pytest.raises(ValueError):  # MGT_ERR_INVALID: a tolerance outside (0, 1)
        solver.solve_native(z[:2], np.array([1e-8, 1.5]), 10)
