"""Dump per-CUDA-source-line counters of one kernel launch in an ncu report as
a compact CSV (line, file, warp instructions, predicated-on thread
instructions, stall samples), for offline region analysis.

    NCU_LAUNCH=i python scripts/ncu_dump_lines.py report.ncu-rep kernel_regex > out.csv
"""
import csv
import io
import os
import subprocess
import sys

rep, k = sys.argv[1], sys.argv[2]
EXTRA = ["--launch-skip", os.environ["NCU_LAUNCH"], "--launch-count", "1"] if os.environ.get("NCU_LAUNCH") else []
out = subprocess.run(["ncu", "-i", rep, "--page", "source", "--csv", "-k", f"regex:{k}", *EXTRA,
                      "--print-source", "cuda"], capture_output=True, text=True).stdout
lines = out.splitlines()
fname = ""
w = csv.writer(sys.stdout)
w.writerow(["file", "line", "warp_inst", "thread_inst", "samples", "source"])
hdr = None
for l in lines:
    if l.startswith('"File Path"') or l.startswith("File Path") or l.startswith('"Source File"'):
        continue
    if l.startswith('"Line No"'):
        hdr = next(csv.reader([l]))
        continue
    if hdr is None:
        if l.strip():
            fname = l.strip().strip('"')
        continue
    r = next(csv.reader([l]))
    if not r or not r[0].isdigit():
        if l.strip() and not r[0].isdigit():
            fname = l.strip().strip('"')
            hdr = None
        continue
    try:
        row = [fname, int(r[0]), int(r[hdr.index("Instructions Executed")]),
               int(r[hdr.index("Predicated-On Thread Instructions Executed")]),
               int(r[hdr.index("Warp Stall Sampling (All Samples)")]), r[1][:90]]
    except (ValueError, IndexError):
        continue
    if row[2] or row[4]:
        w.writerow(row)
