"""Per-phase stall-reason breakdown (source lines between VAPR_PHASE markers)
of the collision kernel.  python scripts/ncu_stalls.py report.ncu-rep"""
import csv
import io
import re
import subprocess
import sys

rep = sys.argv[1]
src = open("paper_2310_07854_b200/csrc/collision.cu").read().splitlines()
marks = [(i + 1, int(m.group(1))) for i, l in enumerate(src) if (m := re.search(r"VAPR_PHASE\((\d+)\);", l))]
kstart = next(i + 1 for i, l in enumerate(src) if "collision_kernel(const __grid_constant__" in l)
out = subprocess.run(["ncu", "-i", rep, "--page", "source", "--csv", "-k", "regex:collision",
                      "--print-source", "cuda,sass"], capture_output=True, text=True).stdout
lines = out.splitlines()
start = next(i for i, l in enumerate(lines) if l.startswith('"Line No"'))
rows = list(csv.reader(io.StringIO("\n".join(lines[start:]))))
h = rows[0]
reasons = [c for c in h if c.startswith("stall_") and "Not Issued" not in c]
idx = {c: h.index(c) for c in reasons}
ii = h.index("Instructions Executed")
agg = {}
for r in rows[1:]:
    if len(r) <= ii or not r[0].isdigit():
        continue
    ln = int(r[0])
    key = "helpers"
    if ln >= kstart:
        key = "tail"
        prev = kstart
        for ml, ph in marks:
            if prev <= ln < ml:
                key = f"phase {ph}"
                break
            prev = ml
    a = agg.setdefault(key, {c: 0 for c in reasons + ["inst"]})
    for c in reasons:
        try:
            a[c] += int(r[idx[c]] or 0)
        except ValueError:
            pass
    try:
        a["inst"] += int(r[ii])
    except ValueError:
        pass
tot = sum(sum(v for k, v in a.items() if k != "inst") for a in agg.values())
for k in sorted(agg):
    a = agg[k]
    s = sum(v for c, v in a.items() if c != "inst")
    top = sorted(((v, c) for c, v in a.items() if c != "inst"), reverse=True)[:4]
    print(f"{k:8s} {100 * s / tot:5.1f}% of samples  inst {a['inst'] / 1e6:8.1f}M  " +
          "  ".join(f"{c[6:]}={100 * v / max(s, 1):.0f}%" for v, c in top))
