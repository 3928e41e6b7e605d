#!/usr/bin/env python
"""Summarise an ncu report: key raw metrics per kernel (run here, no GPU)."""
import csv
import subprocess
import sys

KEYS = ["gpu__time_duration.sum", "dram__bytes_read.sum", "dram__bytes_write.sum",
        "dram__throughput.avg.pct_of_peak_sustained_elapsed", "lts__t_sector_hit_rate.pct",
        "l1tex__t_sector_hit_rate.pct", "launch__registers_per_thread", "launch__grid_size",
        "launch__block_size", "sm__warps_active.avg.pct_of_peak_sustained_active",
        "smsp__inst_executed.sum", "sm__pipe_fp64_cycles_active.avg.pct_of_peak_sustained_active",
        "sm__inst_executed_pipe_fp64.avg.pct_of_peak_sustained_active",
        "local_load_bytes", "smsp__average_warp_latency_issue_stalled_long_scoreboard",
        "l1tex__data_bank_conflicts_pipe_lsu.sum", "lts__t_bytes.sum"]


def main(path):
    out = subprocess.run(["ncu", "-i", path, "--page", "raw", "--csv"], capture_output=True, text=True).stdout
    rows = list(csv.reader(out.splitlines()))
    h, u = rows[0], rows[1]
    for r in rows[2:]:
        print("kernel:", r[h.index("Kernel Name")][:110])
        for k in KEYS:
            if k in h:
                i = h.index(k)
                print(f"  {k:70s} {r[i]:>16s} {u[i]}")
        # tensor-pipe metrics (DMMA kernels): whatever this ncu names them
        for i, k in enumerate(h):
            if k not in KEYS and ("dmma" in k or "pipe_tensor" in k or "pipe_fp64" in k) and r[i] not in ("", "0", "n/a"):
                print(f"  {k:70s} {r[i]:>16s} {u[i]}")


if __name__ == "__main__":
    main(sys.argv[1])
