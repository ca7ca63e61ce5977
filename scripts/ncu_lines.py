"""Per-CUDA-source-line hotspots of one kernel in an ncu report.

    python scripts/ncu_lines.py report.ncu-rep kernel_regex [top]
"""
import csv
import os
import io
import subprocess
import sys

rep, k = sys.argv[1], sys.argv[2]
# NCU_LAUNCH=i picks the i-th matching launch of the report
EXTRA = ["--launch-skip", os.environ["NCU_LAUNCH"], "--launch-count", "1"] if os.environ.get("NCU_LAUNCH") else []
top = int(sys.argv[3]) if len(sys.argv) > 3 else 25
out = subprocess.run(["ncu", "-i", rep, "--page", "source", "--csv", "-k", f"regex:{k}", *EXTRA,
                      "--print-source", "cuda,sass"], capture_output=True, text=True).stdout
lines = out.splitlines()
start = next(i for i, l in enumerate(lines) if l.startswith('"Line No"'))
rows = list(csv.reader(io.StringIO("\n".join(lines[start:]))))
h = rows[0]
iL, iS = 0, 1
iw = h.index("Warp Stall Sampling (All Samples)")
ii = h.index("Instructions Executed")
res = []
tot_w = tot_i = 0
for r in rows[1:]:
    if len(r) <= ii or not r[0].isdigit():
        continue
    try:
        w = int(r[iw]); n = int(r[ii])
    except ValueError:
        continue
    tot_w += w; tot_i += n
    res.append((w, n, int(r[0]), r[1][:90]))
res.sort(reverse=True, key=(lambda t: t[1]) if os.environ.get("BY_INST") else None)
print(f"total stall samples {tot_w}, warp instructions {tot_i}")
for w, n, ln, src in res[:top]:
    print(f"{100*w/tot_w:5.1f}% samp {100*n/tot_i:5.1f}% inst  L{ln:4d}  {src}")
