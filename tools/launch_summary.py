#!/usr/bin/env python
"""Summarise an ncu `--metrics gpu__time_duration.sum --csv` launch list:
launches, mean duration and share of summed kernel time per kernel."""
import csv
import sys
from collections import defaultdict


def main(path, top=40):
    lines = [l for l in open(path) if l.startswith('"')]
    rows = list(csv.reader(lines))
    h = rows[0]
    ki, vi, ui = h.index("Kernel Name"), h.index("Metric Value"), h.index("Metric Unit")
    tot = defaultdict(float)
    cnt = defaultdict(int)
    for r in rows[1:]:
        scale = {"ns": 1e-3, "us": 1.0, "usecond": 1.0, "ms": 1e3, "nsecond": 1e-3}.get(r[ui], 1e-3)
        name = r[ki].split("(")[0] if not r[ki].startswith("void ") else r[ki][5:].split("(")[0]
        tot[name] += float(r[vi].replace(",", "")) * scale
        cnt[name] += 1
    s = sum(tot.values())
    print(f"{len(rows) - 1} launches, {s / 1e3:.1f} ms summed kernel time (cold-cache, serialised)")
    print(f"{'launches':>9} {'mean_us':>10} {'share':>6}  kernel")
    for name, t in sorted(tot.items(), key=lambda kv: -kv[1])[:top]:
        print(f"{cnt[name]:9d} {t / cnt[name]:10.2f} {100 * t / s:5.1f}%  {name[:110]}")


if __name__ == "__main__":
    main(sys.argv[1])
