"""Attribute ncu per-SASS-instruction counters (a `--page source --print-source
sass` CSV of one launch) to CUDA source lines using the -lineinfo of the same
cubin (nvdisasm -g), for kernels whose ncu source view is unavailable.

    python scripts/sass_line_map.py dis.txt function_substring sass.csv [top]
"""
import csv
import re
import sys
from collections import defaultdict

dis, fn, sass = sys.argv[1], sys.argv[2], sys.argv[3]
top = int(sys.argv[4]) if len(sys.argv) > 4 else 60
amap = {}
inside = False
cur = ("?", 0)
for l in open(dis):
    if l.startswith("//----") and ".text." in l:
        inside = fn in l
        continue
    if not inside:
        continue
    m = re.search(r'//## File "([^"]+)", line (\d+)', l)
    if m:
        cur = (m.group(1).split("/")[-1], int(m.group(2)))
        continue
    m = re.match(r"\s+/\*([0-9a-f]{4,})\*/", l)
    if m:
        amap[int(m.group(1), 16)] = cur
rows = list(csv.reader(open(sass)))
h = rows[1]
ia, ii, it, iw = (h.index(k) for k in ("Address", "Instructions Executed",
                                       "Predicated-On Thread Instructions Executed",
                                       "Warp Stall Sampling (All Samples)"))
base = None
acc = defaultdict(lambda: [0, 0, 0])
tot = [0, 0, 0]
for r in rows[2:]:
    if len(r) <= max(ia, ii, it, iw) or not r[ia].startswith("0x"):
        continue
    a = int(r[ia], 16)
    if base is None:
        base = a
    key = amap.get(a - base, ("?", -1))
    v = (int(r[ii]), int(r[it]), int(r[iw]))
    for k in range(3):
        acc[key][k] += v[k]
        tot[k] += v[k]
print(f"total warp inst {tot[0]}, thread inst {tot[1]}, samples {tot[2]}")
for key, v in sorted(acc.items(), key=lambda kv: -kv[1][0])[:top]:
    print(f"{key[0]:>16}:{key[1]:<5} inst {100 * v[0] / tot[0]:5.2f}%  samp {100 * v[2] / max(tot[2], 1):5.2f}%  thr/inst {v[1] / max(v[0], 1):5.1f}")
