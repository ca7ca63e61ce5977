"""Summarise an ncu --csv launch list: per kernel name, launches, mean time and
share of the total, DRAM bytes per launch.
    python scripts/launch_summary.py gpurun_out/launches.csv"""
import csv
import sys
from collections import defaultdict

rows = list(csv.reader(open(sys.argv[1])))
hdr = next(i for i, r in enumerate(rows) if "Kernel Name" in r)
h = rows[hdr]
ki, mi, vi, ii = h.index("Kernel Name"), h.index("Metric Name"), h.index("Metric Value"), h.index("ID")
per = defaultdict(dict)
for r in rows[hdr + 1:]:
    if len(r) > vi:
        per[int(r[ii])]["name"] = r[ki]
        per[int(r[ii])][r[mi]] = float(r[vi].replace(",", ""))
agg = defaultdict(lambda: [0, 0.0, 0.0])
for d in per.values():
    n = d["name"].split("(")[0].replace("void ", "")
    a = agg[n]
    a[0] += 1
    a[1] += d.get("gpu__time_duration.sum", 0.0)
    a[2] += d.get("dram__bytes_read.sum", 0.0) + d.get("dram__bytes_write.sum", 0.0)
tot = sum(a[1] for a in agg.values())
print(f"{'kernel':60s} {'n':>4s} {'mean_us':>10s} {'share':>7s} {'dram_MB/launch':>15s}")
for n, (c, t, b) in sorted(agg.items(), key=lambda kv: -kv[1][1]):
    print(f"{n[:60]:60s} {c:4d} {t / c / 1e3:10.1f} {100 * t / tot:6.1f}% {b / c / 1e6:15.1f}")
