"""Sum ncu source-page stall samples / executed instructions over line ranges.

    python scripts/ncu_ranges.py report.ncu-rep kernel_regex name:lo-hi [name:lo-hi ...]
"""
import csv
import os
import io
import subprocess
import sys

rep, k = sys.argv[1], sys.argv[2]
# NCU_LAUNCH=i picks the i-th matching launch of the report
EXTRA = ["--launch-skip", os.environ["NCU_LAUNCH"], "--launch-count", "1"] if os.environ.get("NCU_LAUNCH") else []
ranges = []
for a in sys.argv[3:]:
    name, r = a.split(":")
    lo, hi = r.split("-")
    ranges.append((name, int(lo), int(hi)))
out = subprocess.run(["ncu", "-i", rep, "--page", "source", "--csv", "-k", f"regex:{k}", *EXTRA,
                      "--print-source", "cuda,sass"], capture_output=True, text=True).stdout
lines = out.splitlines()
start = next(i for i, l in enumerate(lines) if l.startswith('"Line No"'))
rows = list(csv.reader(io.StringIO("\n".join(lines))))
h = rows[start]
iw = h.index("Warp Stall Sampling (All Samples)")
ii = h.index("Instructions Executed")
acc = {n: [0, 0] for n, _, _ in ranges}
acc["other"] = [0, 0]
tw = ti = 0
MAIN = os.environ.get("NCU_MAIN_FILE", "collision.cu")
cur = ""
for r in rows:
    if r and r[0] in ("File Name", "File Path"):
        cur = r[1]
        continue
    if len(r) <= ii or not r[0].isdigit():
        continue
    try:
        w = int(r[iw]); n = int(r[ii])
    except ValueError:
        continue
    ln = int(r[0])
    tw += w; ti += n
    if not cur.endswith(MAIN):
        key = "file:" + os.path.basename(cur)
        acc.setdefault(key, [0, 0])
        acc[key][0] += w; acc[key][1] += n
        continue
    for name, lo, hi in ranges:
        if lo <= ln <= hi:
            acc[name][0] += w; acc[name][1] += n
            break
    else:
        acc["other"][0] += w; acc["other"][1] += n
for name, (w, n) in acc.items():
    print(f"{name:16s} samples {100*w/max(tw,1):5.1f}%  inst {100*n/max(ti,1):5.1f}%  ({n/1e6:.0f}M)")
