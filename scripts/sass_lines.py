"""Static SASS instruction count of one kernel per source file:line range
(code size; instruction-cache footprint), from `nvdisasm -g` output.

    python scripts/sass_lines.py all.sass kernel_substring [name:file:lo-hi ...]
"""
import re
import sys
from collections import Counter

path, kname = sys.argv[1], sys.argv[2]
regions = []
for a in sys.argv[3:]:
    name, f, rng = a.split(":")
    lo, hi = (int(x) for x in rng.split("-"))
    regions.append((name, f, lo, hi))
inside = False
cur = ("?", 0)
per = Counter()
n = 0
for line in open(path):
    if line.startswith("//--------------------- .text."):
        inside = kname in line
        continue
    if not inside:
        continue
    m = re.search(r'//## File "([^"]+)", line (\d+)', line)
    if m:
        cur = (m.group(1).split("/")[-1], int(m.group(2)))
        continue
    if re.match(r"\s+/\*[0-9a-f]{4,}\*/", line):
        per[cur] += 1
        n += 1
print("total", n)
if regions:
    for name, f, lo, hi in regions:
        c = sum(v for (ff, ln), v in per.items() if ff == f and lo <= ln <= hi)
        print(f"{name:>12s}: {c}")
else:
    byfile = Counter()
    for (f, ln), v in per.items():
        byfile[f] += v
    print(byfile.most_common())
    for (f, ln), v in per.most_common(40):
        print(v, f, ln)
