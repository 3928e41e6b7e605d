"""Result-file formats against the reference's own output
(tests/golden/golden_io.npz, written by tests/golden/make_golden_io.py with
the reference's experiments.write_results_csv / write_angles_csv /
write_manifest): byte-identical files, exact read-back, manifest checks."""

import os

import numpy as np
import pytest

from paper_1909_12234_b200 import experiments as E

GOLD_IO = os.path.join(os.path.dirname(__file__), "golden", "golden_io.npz")


def _rows(g):
    gold = np.load(os.path.join(os.path.dirname(GOLD_IO), "golden_4x4x4x4.npz"))
    return [{"rank": r, "hp_count": 1, "variance": float(v), "jackknife_err": float(v) / 3,
             "t0_re": 1.0 / 3, "t0_im": -2.0 / 7, "estimate_re": float(e), "estimate_im": 1e-17 * r,
             "inversions": 10 + r}
            for r, (e, v) in enumerate(zip(gold["post_estimates"].real, gold["post_variances"]))]


def test_results_and_angles_csv_bytes(tmp_path):
    g = np.load(GOLD_IO)
    rows = _rows(g)
    E.write_results_csv(tmp_path / "results.csv", rows)
    E.write_angles_csv(tmp_path / "angles.csv", [0.0, 1e-3 / 3, 0.5, 1.0])
    assert (tmp_path / "results.csv").read_bytes() == g["results_csv"].tobytes()
    assert (tmp_path / "angles.csv").read_bytes() == g["angles_csv"].tobytes()
    back = E.read_results_csv(tmp_path / "results.csv")
    assert back == rows
    assert E.read_angles_csv(tmp_path / "angles.csv") == [(0, 0.0), (1, 1e-3 / 3), (2, 0.5), (3, 1.0)]


def test_manifest_bytes_verify_and_tamper(tmp_path):
    g = np.load(GOLD_IO)
    run = E.RunDirectory(str(tmp_path))
    E.write_results_csv(run.add("results.csv"), _rows(g))
    E.write_angles_csv(run.add("angles.csv"), [0.0, 1e-3 / 3, 0.5, 1.0])
    run.finish("ok")
    assert (tmp_path / "MANIFEST.csv").read_bytes() == g["MANIFEST_csv"].tobytes()
    assert E.verify_manifest(str(tmp_path)) == "ok"
    with open(tmp_path / "angles.csv", "a") as f:
        f.write("4,0.25\n")
    with pytest.raises(E.NumericalFailure, match="angles.csv"):
        E.verify_manifest(str(tmp_path))
    run.finish("failed: solver")
    assert E.verify_manifest(str(tmp_path)) == "failed: solver"


def test_result_row_from_estimate():
    from paper_1909_12234_b200.trace import finish
    est = finish(1.5 - 0.5j, np.array([1 + 1j, 2 - 1j, 3 + 0.5j]), 12)
    r = E.result_row(4, 16, est)
    assert r["rank"] == 4 and r["hp_count"] == 16 and r["inversions"] == 12
    assert r["estimate_re"] == est.mean.real and r["t0_im"] == -0.5 and r["variance"] == est.variance
