"""Per-opcode and per-source-line instruction counts from an ncu
`--page source --csv --print-source cuda,sass` dump.
    python scripts/ncu_sass_ops.py dump.csv [opcode ...]"""
import csv
import sys
from collections import Counter, defaultdict

rows = list(csv.reader(open(sys.argv[1])))
want = sys.argv[2:] or ["IMAD", "LDS", "LOP3", "ISETP", "BRA"]
cur, hdr, line = "", None, None
byline, tot, src_of = defaultdict(Counter), Counter(), {}
for r in rows:
    if r and r[0] in ("File Path", "File Name"):
        cur = r[1].split("/")[-1]
        continue
    if r and r[0] == "Line No":
        hdr = r
        ie = hdr.index("Instructions Executed")
        continue
    if hdr is None or not r:
        continue
    if r[0].isdigit():
        line = (cur, int(r[0]))
        src_of[line] = r[1][:80]
        continue
    if r[0] == "" and len(r) > ie and line:
        try:
            n = int(r[ie])
        except ValueError:
            continue
        sass = r[3].strip()
        if sass.startswith("@"):
            sass = sass.split(None, 1)[1] if " " in sass else sass
        opc = sass.split()[0].split(".")[0] if sass else "?"
        byline[line][opc] += n
        tot[opc] += n
allt = sum(tot.values())
print("total %.0fM" % (allt / 1e6), " ".join("%s %.1f%%" % (k, 100 * v / allt) for k, v in tot.most_common(12)))
for opc in want:
    lst = sorted(((c[opc], k) for k, c in byline.items() if c[opc] > 0), reverse=True)[:6]
    print("==", opc, "%.0fM" % (tot[opc] / 1e6))
    for n, k in lst:
        print("   %6.1fM %s:%d  %s" % (n / 1e6, k[0], k[1], src_of.get(k, "")))
