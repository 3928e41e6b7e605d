"""CPU tests of the drop-in boundary: the C-ABI library loads without a GPU
and exports every function `include/mgtrace_b200.h` declares; the ctypes
binding covers the same set; argument validation fails with the mapped
error before touching the device."""

import ctypes as ct
import os
import re

import numpy as np
import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
HEADER = os.path.join(ROOT, "include", "mgtrace_b200.h")


def declared_functions():
    src = open(HEADER).read()
    src = re.sub(r"/\*.*?\*/", "", src, flags=re.S)
    names = re.findall(r"^\s*(?:const\s+)?[a-z_0-9]+\s*\*?\s*(mgt_[a-z_0-9]+)\s*\(", src, flags=re.M)
    return sorted(set(names))


@pytest.fixture(scope="module")
def lib():
    from paper_1909_12234_b200 import _lib
    if not os.path.exists(_lib.LIB_PATH):
        pytest.skip("native library not built")
    return _lib.lib()


def test_header_declares_the_boundary():
    names = declared_functions()
    for n in ("mgt_wilson_create", "mgt_wilson_apply", "mgt_bicgstab_solve", "mgt_noise", "mgt_prolong",
              "mgt_restrict", "mgt_coarse_build", "mgt_proj_vhx", "mgt_proj_sub", "mgt_last_error"):
        assert n in names
    assert len(names) >= 20


def test_library_exports_every_declared_symbol(lib):
    missing = [n for n in declared_functions() if not hasattr(lib, n)]
    assert not missing, missing


def test_ctypes_binding_matches_header(lib):
    from paper_1909_12234_b200 import _lib
    assert set(_lib.exported_symbols()) == set(declared_functions())


def test_no_cpu_fallback_and_error_mapping(lib):
    from paper_1909_12234_b200 import _lib
    assert lib.mgt_version() >= 1
    # argument validation happens before any CUDA call
    h = ct.c_void_p()
    rc = lib.mgt_wilson_create(ct.byref(h), _lib.dims_arg((4, 4, 4, 1)), 1, 0.1, 64, 18, ct.c_void_p(1), None)
    assert rc == _lib.MGT_ERR_INVALID
    with pytest.raises(ValueError, match="extent"):
        _lib.check(rc)
    rc = lib.mgt_wilson_create(ct.byref(h), _lib.dims_arg((4, 4, 4, 4)), 1, 0.1, 48, 18, ct.c_void_p(1), None)
    with pytest.raises(ValueError, match="prec"):
        _lib.check(rc)
    rc = lib.mgt_prolong(_lib.dims_arg((4, 4, 4, 6)), _lib.dims_arg((4, 4, 4, 4)), 8, ct.c_void_p(1),
                         ct.c_void_p(1), ct.c_void_p(1), 1, None)
    from paper_1909_12234_b200.multigrid import BlockingError
    with pytest.raises(BlockingError):
        _lib.check(rc)
    rc = lib.mgt_noise(_lib.dims_arg((2, 2, 2, 2)), 7, (ct.c_uint64 * 4)(), 1, 1, ct.c_void_p(1), None)
    with pytest.raises(ValueError, match="kind"):
        _lib.check(rc)


def test_operator_requires_cuda_no_fallback():
    import torch
    if torch.cuda.is_available():
        pytest.skip("GPU present")
    import paper_1909_12234_b200 as M
    geo = M.LatticeGeometry((4, 4, 4, 4), "antiperiodic")
    with pytest.raises(RuntimeError, match="CUDA"):
        M.generate_gauge(geo, "unit")


def test_geometry_and_blocking_validation():
    import paper_1909_12234_b200 as M
    from paper_1909_12234_b200 import multigrid as MG
    with pytest.raises(M.GeometryError):
        M.LatticeGeometry((4, 1, 4, 4))
    with pytest.raises(M.GeometryError):
        M.LatticeGeometry((4, 4, 4, 4), "twisted")
    geo = M.LatticeGeometry((8, 8, 8, 16), "antiperiodic")
    assert geo.site_count == 8192 and geo.neighbor(geo.site_index((0, 0, 0, 15)), 3, +1) == 0
    MG.BlockingScheme((4, 4, 4, 4)).validate(geo)
    with pytest.raises(MG.BlockingError):
        MG.BlockingScheme((3, 4, 4, 4)).validate(geo)
    with pytest.raises(MG.BlockingError):
        MG.BlockingScheme((0, 4, 4, 4))
    assert MG.BlockingScheme((4, 4, 4, 4)).coarse_dims(geo) == (2, 2, 2, 4)


def test_coarse_tables_host_logic():
    import numpy as np
    from paper_1909_12234_b200 import multigrid as MG
    cd = (2, 3, 4, 5)
    nbr = MG.coarse_neighbours(cd)
    perm = MG.native_to_ref_coarse(cd)
    assert sorted(perm) == list(range(int(np.prod(cd))))
    # forward then backward returns to self, in every direction
    for mu in range(4):
        f, b = nbr[:, 1 + 2 * mu], nbr[:, 2 + 2 * mu]
        assert np.array_equal(nbr[f, 2 + 2 * mu], np.arange(len(perm)))
        assert np.array_equal(nbr[b, 1 + 2 * mu], np.arange(len(perm)))


def test_estimator_statistics_match_reference_formulas():
    import numpy as np
    from oracle import trace as OT
    from paper_1909_12234_b200 import trace as TR
    s = np.random.default_rng(0).normal(size=9) + 1j * np.random.default_rng(1).normal(size=9)
    a = TR.finish(0.5 + 0.25j, s, 9)
    b = OT.finish(0.5 + 0.25j, s)
    assert a.mean == b["mean"] and a.variance == b["variance"] and a.jackknife_err == b["jackknife_err"]
    one = TR.finish(0.0, s[:1], 1)
    assert one.variance == 0.0 and one.jackknife_err == 0.0
    with pytest.raises(ValueError):
        TR.jackknife(s[:1])
    lam, uhat, t0 = TR.factorize_small(np.diag([3.0, -1.0, 2.0]).astype(complex), np.eye(3, dtype=complex))
    assert np.allclose(np.abs(lam), [1, 2, 3]) and abs(t0 - (1 / 3 - 1 + 1 / 2)) < 1e-14
    with pytest.raises(TR.SpuriousModeError):
        TR.factorize_small(np.diag([1.0, 1e-14]).astype(complex), np.eye(2, dtype=complex))


def test_default_streams_rule():
    from paper_1909_12234_b200.trace import default_streams
    from paper_1909_12234_b200.krylov import solve_batch
    assert solve_batch(8 ** 4) == 32 and solve_batch(16 ** 4) == 16 and solve_batch(32 ** 4) == 4
    assert default_streams(8 ** 4, 32) == 8
    assert default_streams(16 ** 4, 16) == 4
    assert default_streams(32 ** 4, 4) == 2          # two overlapping solves (tools/streams_probe.py)
    assert default_streams(32 ** 3 * 64, 4) == 2
    assert default_streams(48 ** 3 * 96, 4) == 1


@pytest.mark.parametrize("restart,max_iter,tol", [(8, 8, 1e-12), (4, 30, 1e-10), (32, 200, 1e-9)])
def test_coarse_level_gcr_follows_the_reference_control_flow(restart, max_iter, tol):
    """mglevel.gcr_torch (the coarse-level GCR of 3-level hierarchies and
    smoothers) against the oracle's restatement of krylov.py:52-118 on a
    CPU tensor: same iterations, matvec count, convergence flag and x."""
    import torch
    from oracle import krylov as OK
    from paper_1909_12234_b200.mglevel import gcr_torch
    rng = np.random.default_rng(restart + max_iter)
    n = 60
    A = np.eye(n) * 3 + (rng.normal(size=(n, n)) + 1j * rng.normal(size=(n, n))) / np.sqrt(n)
    b = rng.normal(size=n) + 1j * rng.normal(size=n)
    At, bt = torch.as_tensor(A), torch.as_tensor(b)
    x, rep = gcr_torch(lambda v: At @ v, bt, tol, max_iter, restart)
    xo, ro = OK.gcr(lambda v: A @ v, b, tol, max_iter, restart)
    assert rep.iterations == ro.iterations and rep.matvecs == ro.matvecs and rep.converged == ro.converged
    assert np.linalg.norm(x.numpy() - xo) <= 1e-12 * np.linalg.norm(xo)
