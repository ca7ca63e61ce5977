"""Region table (warp instructions, stall samples, threads per instruction)
of a collision pass from the per-line output of scripts/sass_line_map.py,
over the source-line ranges of csrc/collision.cu at the measured tree.

    python scripts/sass_regions.py lines.txt
"""
import re
import sys
from collections import defaultdict

REGIONS = [("world_term", 72, 136), ("sparse_row", 137, 199), ("or_code3", 200, 224),
           ("row reads (RowView)", 225, 250), ("self_pair", 251, 296), ("warp_queue", 482, 547),
           ("kernel head", 633, 778), ("tile stage+decode", 779, 961), ("margin+zero", 962, 983),
           ("world broadphase", 984, 1075), ("world items", 1076, 1167), ("self broadphase", 1168, 1215),
           ("self narrowphase", 1216, 1310), ("self touched", 1311, 1327), ("self gradients", 1328, 1401),
           ("tile tail", 1402, 1440)]
acc = defaultdict(lambda: [0.0, 0.0, 0.0])
head = ""
for l in open(sys.argv[1]):
    if l.startswith("total"):
        head = l.strip()
    m = re.match(r"\s*(\S+):(-?\d+)\s+inst\s+([\d.]+)%\s+samp\s+([\d.]+)%\s+thr/inst\s+([\d.]+)", l)
    if not m:
        continue
    f, ln, ip, sp, thr = m.group(1), int(m.group(2)), float(m.group(3)), float(m.group(4)), float(m.group(5))
    name = "(other) " + f
    if f == "collision.cu":
        name = "(other) collision.cu"
        for n, a, b in REGIONS:
            if a <= ln <= b:
                name = n
    acc[name][0] += ip
    acc[name][1] += sp
    acc[name][2] += ip * thr
print(head)
print(f"{'region':>28} {'warp-inst %':>11} {'samples %':>10} {'threads/inst':>12}")
for k, v in sorted(acc.items(), key=lambda kv: -kv[1][0]):
    if v[0] >= 0.3:
        print(f"{k:>28} {v[0]:11.2f} {v[1]:10.2f} {v[2] / max(v[0], 1e-9):12.1f}")
