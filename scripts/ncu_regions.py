"""Instructions executed and stall samples of one kernel in an ncu report,
summed over source-line ranges (a region table for the collision kernel).

    python scripts/ncu_regions.py report.ncu-rep kernel_regex file.cu name:lo-hi ...
"""
import csv
import io
import subprocess
import sys

rep, k, src = sys.argv[1], sys.argv[2], sys.argv[3]
regions = []
for a in sys.argv[4:]:
    name, rng = a.split(":")
    lo, hi = (int(x) for x in rng.split("-"))
    regions.append((name, lo, hi))
import os as _os
# NCU_LAUNCH=i picks the i-th matching launch of the report
EXTRA = (["--launch-skip", _os.environ["NCU_LAUNCH"], "--launch-count", "1"]
         if _os.environ.get("NCU_LAUNCH") else [])
out = subprocess.run(["ncu", "-i", rep, "--page", "source", "--csv", "-k", f"regex:{k}", *EXTRA,
                      "--print-source", "cuda,sass"], capture_output=True, text=True).stdout
lines = out.splitlines()
rows = []
cur_file = ""
start = None
for i, l in enumerate(lines):
    if l.startswith('"Line No"'):
        start = i
        break
rows = list(csv.reader(io.StringIO("\n".join(lines[start:]))))
h = rows[0]
iw = h.index("Warp Stall Sampling (All Samples)")
ii = h.index("Instructions Executed")
it = h.index("Predicated-On Thread Instructions Executed")
tot = {n: [0, 0, 0] for n, _, _ in regions}
ti = tw = tt = 0
for r in rows[1:]:
    if len(r) <= ii or not r[0].isdigit():
        continue
    try:
        ln, w, n, th = int(r[0]), int(r[iw]), int(r[ii]), int(r[it])
    except ValueError:
        continue
    ti += n
    tw += w
    tt += th
    for name, lo, hi in regions:
        if lo <= ln <= hi:
            tot[name][0] += n
            tot[name][1] += w
            tot[name][2] += th
import os
P = float(os.environ.get("POSES", "2560000"))
print(f"total warp instructions {ti}, thread instructions (pred-on) {tt}, stall samples {tw}")
print(f"{'region':>14s}  warp-inst%  samples%  warp-inst/pose  thread-inst/pose  threads/inst")
for name, (n, w, th) in tot.items():
    print(f"{name:>14s}: {100 * n / max(ti, 1):8.1f}  {100 * w / max(tw, 1):8.1f}  {n / P:12.1f}  {th / P:14.1f}  {th / max(n, 1):8.1f}")
