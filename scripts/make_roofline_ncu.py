"""profiles/r2/roofline_ncu.json from the raw CSV of one full ncu capture of
the bench step's kernels (scripts/r2_measure.sh: step_sparse43.raw.csv):
per stage of vapr_cost_grad the DRAM bytes per launch, duration, issue and
occupancy figures and the measured limiter.  bench.py reads it for the
roofline's `traffic` / `limiter` / `issue` fields.

    python scripts/make_roofline_ncu.py gpurun_out/r2/step_sparse43.raw.csv 43bit 2560000
"""
import csv
import json
import sys

src, formats, poses = sys.argv[1], sys.argv[2], int(sys.argv[3])
rows = list(csv.reader(open(src)))
h = rows[0]
recs = [dict(zip(h, r)) for r in rows[2:]]


def f(d, k):
    try:
        return float(d[k])
    except (KeyError, ValueError):
        return None


def stage(name):
    n = name
    if "fk_" in n:
        return "fk"
    if "collision_kernel" in n or "Geo, WorldsDev" in n:
        return "collision"
    if "traj_reduce" in n:
        return "reduce"
    if "aggregate" in n:
        return "aggregate"
    if "bk_kernel" in n:
        return "bk"
    return n[:40]


STALLS = ["long_scoreboard", "short_scoreboard", "barrier", "wait", "math_pipe_throttle",
          "no_instructions", "not_selected", "selected", "mio_throttle", "lg_throttle"]
out = {"formats": formats, "poses": poses, "source": src.split("/")[-1],
       "note": "ncu --set full --clock-control none, one vapr_cost_grad of config 4 (sparse "
               "storage); per-launch values; collision = the self pass + the world pass",
       "kernels": {}}
for d in recs:
    st = stage(d.get("Kernel Name", ""))
    MB = 1e6
    dram = (f(d, "dram__bytes_read.sum") or 0) + (f(d, "dram__bytes_write.sum") or 0)
    unit = d.get("dram__bytes_read.sum")
    # the raw page reports bytes in the unit of its header row (MB here)
    launch = {
        "kernel": d.get("Kernel Name", "")[:80],
        "ms": f(d, "gpu__time_duration.sum"),
        "dram_MB": round(dram, 3),
        "issue_active_pct": f(d, "smsp__issue_active.avg.pct_of_peak_sustained_active"),
        "warps_active_pct": f(d, "sm__warps_active.avg.pct_of_peak_sustained_active"),
        "warp_instructions": f(d, "smsp__inst_executed.sum"),
        "threads_per_instruction": f(d, "smsp__thread_inst_executed_per_inst_executed.ratio"),
        "registers": f(d, "launch__registers_per_thread"),
        "shared_bank_conflicts": f(d, "l1tex__data_bank_conflicts_pipe_lsu_mem_shared.sum"),
        "stall_samples": {s: f(d, "smsp__pcsamp_warps_issue_stalled_" + s) for s in STALLS},
    }
    e = out["kernels"].setdefault(st, {"launches": []})
    e["launches"].append(launch)
units = rows[1]
u = dict(zip(h, units)).get("dram__bytes_read.sum", "")
scale = {"Mbyte": 1e6, "Gbyte": 1e9, "Kbyte": 1e3, "byte": 1.0}.get(u, 1e6)
for st, e in out["kernels"].items():
    L = e["launches"]
    e["dram_bytes"] = sum(l["dram_MB"] for l in L) * scale
    e["ms"] = sum(l["ms"] or 0 for l in L)
    e["issue"] = {"issue_active_pct": [l["issue_active_pct"] for l in L],
                  "warps_active_pct": [l["warps_active_pct"] for l in L],
                  "warp_instructions": [l["warp_instructions"] for l in L],
                  "threads_per_instruction": [l["threads_per_instruction"] for l in L]}
LIMITER = {
    "collision": "two passes, each its own kernel, one CTA per SM, both with 16-bit tile rows "
                 "(E5M10 out_spheres): self pass 2 CTAs x 11 warps per SM, 80 registers, world pass 24 "
                 "warps, 78 registers; both ~75 % issue-active (instruction issue; the occupancy "
                 "sweeps: self 12 -> 16 -> 26 warps 1.64 -> 1.37 -> 1.14 ms, world 16 -> 24 "
                 "1.22 -> 1.03 ms); 21-23 of 32 threads per instruction; DRAM traffic = "
                 "out_spheres read by both passes + the sparse outputs "
                 "(profiles/r2/collision_regions_*.txt)",
    "fk": "instruction issue: ~88 % issue-active at 40 warps per SM, 31.6 of 32 threads per "
          "instruction",
    "aggregate": "divergence: a thread per row over the set spheres (10.7 of 32 threads per "
                 "instruction), 67 % issue-active",
    "bk": "latency / occupancy: 36 % issue-active, 18 % warps active, top stalls long "
          "scoreboard and the CTA barrier (compaction of the poses with a gradient), 16.7 of "
          "32 threads per instruction",
    "reduce": "memory latency (a thread per trajectory)",
}
for st, e in out["kernels"].items():
    e["limiter"] = LIMITER.get(st, "")
json.dump(out, open("profiles/r2/roofline_ncu.json", "w"), indent=1)
print({k: (round(v["dram_bytes"] / 1e9, 3), round(v["ms"], 3)) for k, v in out["kernels"].items()})
