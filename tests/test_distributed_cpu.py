"""World-size-2 (and 3) gloo tests of the multi-GPU host logic on CPU:
probe sharding + global-order sample gathering (bitwise equal to the
single-process estimate) and the t-slab halo exchange plumbing."""

import os
import socket

import numpy as np
import pytest
import torch
import torch.distributed as dist
import torch.multiprocessing as mp


def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    p = s.getsockname()[1]
    s.close()
    return p


def _run(rank, world, port, fn, q):
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        q.put((rank, fn(rank, world)))
    finally:
        dist.destroy_process_group()


def spawn(world, fn):
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_run, args=(r, world, port, fn, q)) for r in range(world)]
    for p in procs:
        p.start()
    out = dict(q.get(timeout=120) for _ in range(world))
    for p in procs:
        p.join(timeout=60)
        assert p.exitcode == 0
    return [out[r] for r in range(world)]


def _small_problem():
    from oracle import wilson4d as W
    dims = (2, 2, 2, 4)
    A = W.build_wilson4d_csr(W.su3_links(dims, 0.3, 1), dims, 0.2)
    return A


def _local_estimate(j0, j1, s_seed=5):
    from oracle import krylov as OK
    from oracle import pcg64 as OP
    from paper_1909_12234_b200.trace import finish
    A = _small_problem()
    inv = OK.TruncatedInverse(lambda v: A @ v, 1e-10)
    samples = []
    for j in range(j0, j1):
        z = OP.rademacher(A.shape[0], s_seed + j)
        acc = 0.0 + 0.0j
        acc = acc + 1.0 * np.vdot(z, inv(z))
        samples.append(acc)
    return finish(0.0, np.array(samples, dtype=np.complex128), j1 - j0)


def _sharded(rank, world):
    from paper_1909_12234_b200.distributed import sharded_estimate
    est = sharded_estimate(_local_estimate, 7)
    return est.mean, est.samples, est.variance, est.jackknife_err, est.inversions


@pytest.mark.parametrize("world", [2, 3])
def test_probe_sharding_bitwise_equal_single_process(world):
    single = _local_estimate(0, 7)
    res = spawn(world, _sharded)
    for mean, samples, var, jk, inv in res:
        assert np.array_equal(samples, single.samples)
        assert mean == single.mean and var == single.variance and jk == single.jackknife_err
        assert inv == 7


def test_shard_ranges_cover_exactly():
    from paper_1909_12234_b200.distributed import shard_range
    for n in (0, 1, 5, 32, 33):
        for w in (1, 2, 3, 8):
            blocks = [shard_range(n, r, w) for r in range(w)]
            assert blocks[0][0] == 0 and blocks[-1][1] == n
            assert all(blocks[i][1] == blocks[i + 1][0] for i in range(w - 1))


def _halo(rank, world):
    from paper_1909_12234_b200.distributed import exchange_halos
    # each rank sends its id-tagged faces; forward face goes to rank-1, backward to rank+1
    fwd = torch.full((3, 5), float(10 * rank + 1), dtype=torch.float64)
    bwd = torch.full((3, 5), float(10 * rank + 2), dtype=torch.float64)
    from_next, from_prev = exchange_halos(fwd, bwd)
    return float(from_next[0, 0]), float(from_prev[0, 0])


@pytest.mark.parametrize("world", [2, 3])
def test_halo_exchange_ring(world):
    res = spawn(world, _halo)
    for r, (from_next, from_prev) in enumerate(res):
        assert from_next == 10 * ((r + 1) % world) + 1  # next rank's first-slice face
        assert from_prev == 10 * ((r - 1) % world) + 2  # previous rank's last-slice face


def _slab_proj(rank, world):
    from paper_1909_12234_b200.distributed import shard_range, slab_project_out, slab_vhx
    rng = np.random.default_rng(21)
    k, s, n = 5, 3, 61
    V = rng.normal(size=(k, n)) + 1j * rng.normal(size=(k, n))
    X = rng.normal(size=(s, n)) + 1j * rng.normal(size=(s, n))
    j0, j1 = shard_range(n, rank, world)
    Vl = torch.as_tensor(V[:, j0:j1].copy())
    Xl = torch.as_tensor(X[:, j0:j1].copy())

    def local_vhx(a, b):
        return a.conj() @ b.T

    def local_sub(a, h, x):
        x -= (a.T @ h).T
        return x
    H = slab_vhx(Vl, Xl, local=local_vhx)
    H2 = slab_project_out(Vl, Xl, local_vhx=local_vhx, local_sub=local_sub)
    return H.numpy(), H2.numpy(), Xl.numpy(), (j0, j1)


@pytest.mark.parametrize("world", [2, 3])
def test_slab_projection_matches_global(world):
    """t-sharded V^H X and X - V (V^H X): rank-ordered sum of slab partials
    == the global product (1e-14), bitwise identical on every rank."""
    rng = np.random.default_rng(21)
    k, s, n = 5, 3, 61
    V = rng.normal(size=(k, n)) + 1j * rng.normal(size=(k, n))
    X = rng.normal(size=(s, n)) + 1j * rng.normal(size=(s, n))
    Hg = V.conj() @ X.T
    Xg = X - (V.T @ Hg).T
    res = spawn(world, _slab_proj)
    for H, H2, Xl, (j0, j1) in res:
        assert np.abs(H - Hg).max() <= 1e-14 * np.abs(Hg).max()
        assert np.array_equal(H, res[0][0]) and np.array_equal(H2, H)
        assert np.abs(Xl - Xg[:, j0:j1]).max() <= 1e-13 * np.abs(Xg).max()
