#!/bin/bash
# Per-kernel time and DRAM bytes of the mixed even-odd solver on one lattice
# (ncu, serialised launches; a 4-rhs solve, a few iterations):
#   tools/solver_kernel_profile.sh 32x32x32x32 out_prefix
D=${1:-32x32x32x32}
O=${2:-gpurun_out/solver_kernels}
ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum --clock-control none \
    -k regex:'bi_|mx_' -c 400 --csv --log-file ${O}.csv \
    python tools/solver_bench.py --dims $D --groups 4 --nprobe 4 --mixed 1 > ${O}.log 2>&1
python - "${O}.csv" <<'PY' > ${O}.txt
import csv, sys, collections
rows = list(csv.reader([l for l in open(sys.argv[1]) if l.startswith('"')]))
h = rows[0]; ki, mi, vi, ui = h.index("Kernel Name"), h.index("Metric Name"), h.index("Metric Value"), h.index("Metric Unit")
idi = h.index("ID")
per = collections.defaultdict(dict)
for r in rows[1:]:
    v = float(r[vi].replace(",", ""))
    u = r[ui]
    if r[mi] == "gpu__time_duration.sum":
        v *= {"ns": 1e-3, "us": 1.0, "ms": 1e3}.get(u, 1e-3)
    else:
        v *= {"byte": 1, "Kbyte": 1e3, "Mbyte": 1e6, "Gbyte": 1e9}.get(u, 1)
    per[(r[idi], r[ki])][r[mi]] = v
agg = collections.defaultdict(lambda: [0, 0.0, 0.0, 0.0])
for (i, k), m in per.items():
    name = k.split("(")[0].replace("void ", "")
    a = agg[name]; a[0] += 1; a[1] += m.get("gpu__time_duration.sum", 0)
    a[2] += m.get("dram__bytes_read.sum", 0); a[3] += m.get("dram__bytes_write.sum", 0)
tot = sum(a[1] for a in agg.values())
print(f"{'n':>4} {'us':>9} {'share':>6} {'MB_rd':>8} {'MB_wr':>8} {'GB/s':>7}  kernel")
for name, a in sorted(agg.items(), key=lambda kv: -kv[1][1]):
    n, t, rd, wr = a
    print(f"{n:4d} {t/n:9.1f} {100*t/tot:5.1f}% {rd/n/1e6:8.1f} {wr/n/1e6:8.1f} {(rd+wr)/t/1e3:7.0f}  {name}")
PY
