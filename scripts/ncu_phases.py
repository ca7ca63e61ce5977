"""Instructions executed per collision-kernel phase (source line ranges between
VAPR_PHASE markers) from an ncu report captured with --import-source.
    python scripts/ncu_phases.py report.ncu-rep"""
import csv
import io
import re
import subprocess
import sys

rep = sys.argv[1]
src = open("paper_2310_07854_b200/csrc/collision.cu").read().splitlines()
marks = [(i + 1, int(m.group(1))) for i, l in enumerate(src) if (m := re.search(r"VAPR_PHASE\((\d+)\);", l))]
kernel_start = next(i + 1 for i, l in enumerate(src) if "collision_kernel(const __grid_constant__" in l)
out = subprocess.run(["ncu", "-i", rep, "--page", "source", "--csv", "-k", "regex:collision",
                      "--print-source", "cuda,sass"], capture_output=True, text=True).stdout
lines = out.splitlines()
start = next(i for i, l in enumerate(lines) if l.startswith('"Line No"'))
rows = list(csv.reader(io.StringIO("\n".join(lines[start:]))))
h = rows[0]
ii = h.index("Instructions Executed")
iw = h.index("Warp Stall Sampling (All Samples)")
agg = {}
for r in rows[1:]:
    if len(r) <= ii or not r[0].isdigit():
        continue
    ln = int(r[0])
    try:
        n, w = int(r[ii]), int(r[iw])
    except ValueError:
        continue
    if ln < kernel_start:
        key = "helpers (inlined)"
    else:
        key = "tail"
        prev = kernel_start
        for mline, ph in marks:
            if prev <= ln < mline:
                key = f"phase {ph}"
                break
            prev = mline
    a = agg.setdefault(key, [0, 0])
    a[0] += n
    a[1] += w
ti = sum(a[0] for a in agg.values())
tw = sum(a[1] for a in agg.values())
for k, (n, w) in sorted(agg.items()):
    print(f"{k:20s} inst {100 * n / ti:5.1f}%  stall-samples {100 * w / tw:5.1f}%")
