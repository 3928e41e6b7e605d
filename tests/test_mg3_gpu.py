"""3-level hierarchy (`build_hierarchy` with two blockings,
`MultigridSolver` recursing through level 1) against the reference's golden
run on 8^4 (tests/golden/make_golden_mg3.py).  Level 0 -> 1 runs on the fine
kernels, level 1 -> 2 on mglevel.py; the level-1 null vectors follow the
reference's RNG stream, so everything is compared value by value."""

import os

import numpy as np
import pytest
import scipy.sparse as sp
import torch

from oracle import wilson4d as W

pytestmark = pytest.mark.gpu
GOLD = os.path.join(os.path.dirname(__file__), "golden", "golden_mg3_8x8x8x8.npz")


@pytest.fixture(scope="module")
def mg3():
    import paper_1909_12234_b200 as M
    g = dict(np.load(GOLD))
    dims = tuple(int(v) for v in g["dims"])
    geo = M.LatticeGeometry(dims, "antiperiodic")
    links = W.su3_links(dims, float(g["eps"]), int(g["links_seed"]))
    op = M.build_wilson(M.gauge_from_array(geo, links), float(g["mass"]))
    hier = M.build_hierarchy(op, [tuple(b) for b in g["blockings"]], [int(c) for c in g["counts"]],
                             null_tol=1e-12, null_max_iter=8, seed=int(g["seed"]))
    return M, g, op, hier


def _rel(a, b):
    return np.linalg.norm(a - b) / np.linalg.norm(b)


def test_level1_null_vectors_prolongator_and_level2_operator(cuda, mg3):
    M, g, op, hier = mg3
    assert hier.levels == 3
    P1 = hier.prolongators[1]
    Pg = sp.coo_matrix((g["P1_val"], (g["P1_row"], g["P1_col"])), shape=tuple(g["P1_shape"])).toarray()
    assert np.abs(P1.dense() - Pg).max() < 1e-9
    G = hier.prolongators[1].G
    gram = torch.einsum("mcvl,mcwl->mcvw", G.conj(), G)
    eye = torch.eye(G.shape[2], dtype=G.dtype, device=G.device)
    assert (gram - eye).abs().max().item() < 1e-13
    C2 = hier.operators[2].dense()
    assert np.abs(C2 - g["C2_dense"]).max() < 1e-9 * np.abs(g["C2_dense"]).max()


@pytest.mark.parametrize("coarsest", ["lu", "gcr"])
def test_three_level_inverter_matches_reference(cuda, mg3, coarsest):
    M, g, op, hier = mg3
    mg = M.MultigridSolver(hier, smoother_iters=4, coarse_tol=1e-1, coarsest=coarsest)
    x, rep = mg.solve(g["b"], 1e-10, max_cycles=100)
    assert rep.converged and bool(g[f"converged_{coarsest}"])
    assert abs(rep.iterations - int(g[f"cycles_{coarsest}"])) <= 1
    assert _rel(x, g[f"x_{coarsest}"]) < 1e-8
    A = W.build_wilson4d_csr(W.su3_links(tuple(int(v) for v in g["dims"]), float(g["eps"]),
                                         int(g["links_seed"])), tuple(int(v) for v in g["dims"]), float(g["mass"]))
    assert np.linalg.norm(g["b"] - A @ x) <= 1.01e-10 * np.linalg.norm(g["b"])


def test_three_level_dump_load_roundtrip(cuda, mg3, tmp_path):
    M, g, op, hier = mg3
    M.dump_hierarchy(hier, str(tmp_path))
    back = M.load_hierarchy(op, str(tmp_path))
    assert back.levels == 3
    assert np.array_equal(back.prolongators[0].dense(), hier.prolongators[0].dense())
    assert np.array_equal(back.prolongators[1].dense(), hier.prolongators[1].dense())
    assert np.abs(back.operators[2].dense() - hier.operators[2].dense()).max() < 1e-14 * np.abs(
        hier.operators[2].dense()).max()
    with open(tmp_path / "hierarchy_manifest.csv") as f:
        lines = f.read().splitlines()
    assert lines[2].split(",")[:5] == ["1", "4x4x4x4", "2x2x2x2", "128", "12"]
