"""Result files of the reference's experiment drivers.

Only the file formats are rebuilt -- the experiment drivers themselves (CLI,
config, variance sweeps) are out of scope.  Restated from
`mgtrace.experiments` (`/root/reference/pkg/src/mgtrace/experiments.py`):
results CSV (`RESULT_COLUMNS`, `write_results_csv` / `read_results_csv`,
`:93-133`), principal-angle CSV (`:136-146`), SHA-256 MANIFEST with a
trailing status row (`:149-180`) and `RunDirectory` (`:183-199`).  Floats
are written with 17 significant digits, so a read-back is exact.
"""

import csv
import hashlib
import os


class NumericalFailure(RuntimeError):
    """experiments.py:19 -- raised on manifest mismatches."""


RESULT_COLUMNS = ["rank", "hp_count", "variance", "jackknife_err",
                  "t0_re", "t0_im", "estimate_re", "estimate_im", "inversions"]

_INT_COLUMNS = ("rank", "hp_count", "inversions")


def _fmt(x):
    return f"{x:.17g}"


def result_row(rank, hp_count, estimate):
    """One results row from a TraceEstimate (rank = deflation rank)."""
    return {"rank": int(rank), "hp_count": int(hp_count), "variance": float(estimate.variance),
            "jackknife_err": float(estimate.jackknife_err), "t0_re": complex(estimate.t0).real,
            "t0_im": complex(estimate.t0).imag, "estimate_re": complex(estimate.mean).real,
            "estimate_im": complex(estimate.mean).imag, "inversions": int(estimate.inversions)}


def write_results_csv(path, rows):
    """rows: dicts with the RESULT_COLUMNS keys."""
    with open(path, "w", newline="") as f:
        w = csv.writer(f)
        w.writerow(RESULT_COLUMNS)
        for r in rows:
            w.writerow([r[c] if c in _INT_COLUMNS else _fmt(r[c]) for c in RESULT_COLUMNS])
    return path


def read_results_csv(path):
    with open(path, newline="") as f:
        return [{c: (int(rec[c]) if c in _INT_COLUMNS else float(rec[c])) for c in RESULT_COLUMNS}
                for rec in csv.DictReader(f)]


def write_angles_csv(path, sines):
    with open(path, "w", newline="") as f:
        w = csv.writer(f)
        w.writerow(["i", "sine"])
        w.writerows([i, _fmt(s)] for i, s in enumerate(sines))
    return path


def read_angles_csv(path):
    with open(path, newline="") as f:
        return [(int(r["i"]), float(r["sine"])) for r in csv.DictReader(f)]


def sha256_file(path, block=1 << 16):
    h = hashlib.sha256()
    with open(path, "rb") as f:
        while True:
            chunk = f.read(block)
            if not chunk:
                break
            h.update(chunk)
    return h.hexdigest()


def write_manifest(outdir, files, status="ok"):
    """MANIFEST.csv: (file, sha256) sorted by name, then ("_status", status)."""
    path = os.path.join(outdir, "MANIFEST.csv")
    rows = [[name, sha256_file(os.path.join(outdir, name))] for name in sorted(files)]
    with open(path, "w", newline="") as f:
        w = csv.writer(f)
        w.writerow(["file", "sha256"])
        w.writerows(rows)
        w.writerow(["_status", status])
    return path


def verify_manifest(outdir):
    """Re-hash every listed file; returns the recorded status, raises
    NumericalFailure on a mismatch."""
    status = None
    with open(os.path.join(outdir, "MANIFEST.csv"), newline="") as f:
        for rec in csv.DictReader(f):
            if rec["file"] == "_status":
                status = rec["sha256"]
            elif sha256_file(os.path.join(outdir, rec["file"])) != rec["sha256"]:
                raise NumericalFailure(f"manifest mismatch for {rec['file']}")
    return status


class RunDirectory:
    """Collects a run's output files; `finish` writes the MANIFEST (also on
    failure, with the failure status)."""

    def __init__(self, outdir):
        self.outdir = outdir
        os.makedirs(outdir, exist_ok=True)
        self.files = []

    def path(self, name):
        return os.path.join(self.outdir, name)

    def add(self, name):
        self.files.append(name)
        return self.path(name)

    def finish(self, status="ok"):
        return write_manifest(self.outdir, self.files, status=status)
