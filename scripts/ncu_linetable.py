"""Per-source-line table (warp instructions, thread instructions, threads per
instruction, stall samples) of one kernel for a line range.

    python scripts/ncu_linetable.py report.ncu-rep kernel_regex lo hi
"""
import csv
import io
import subprocess
import sys

rep, k, lo, hi = sys.argv[1], sys.argv[2], int(sys.argv[3]), int(sys.argv[4])
out = subprocess.run(["ncu", "-i", rep, "--page", "source", "--csv", "-k", f"regex:{k}",
                      "--print-source", "cuda,sass"], capture_output=True, text=True).stdout
lines = out.splitlines()
start = next(i for i, l in enumerate(lines) if l.startswith('"Line No"'))
rows = list(csv.reader(io.StringIO("\n".join(lines[start:]))))
h = rows[0]
iw, ii = h.index("Warp Stall Sampling (All Samples)"), h.index("Instructions Executed")
it = h.index("Predicated-On Thread Instructions Executed")
P = 2.56e6
for r in rows[1:]:
    if len(r) <= it or not r[0].isdigit():
        continue
    ln = int(r[0])
    if lo <= ln <= hi:
        n, th, w = int(r[ii] or 0), int(r[it] or 0), int(r[iw] or 0)
        if n:
            print(f"L{ln:4d} {n / P:8.1f} w/pose {th / P:9.1f} t/pose {th / max(n, 1):5.1f} thr  {w:7d} samp  {r[1][:70]}")
