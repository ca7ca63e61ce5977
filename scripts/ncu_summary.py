"""Summarise an ncu report: key metrics per kernel (+ optional hot source lines).

    python scripts/ncu_summary.py gpurun_out/prof.ncu-rep [--source collision_kernel]
"""
import csv
import io
import subprocess
import sys

WANT = ["gpu__time_duration.sum", "dram__bytes_read.sum", "dram__bytes_write.sum",
        "gpu__dram_throughput.avg.pct_of_peak_sustained_elapsed",
        "sm__throughput.avg.pct_of_peak_sustained_elapsed",
        "smsp__issue_active.avg.pct_of_peak_sustained_active",
        "sm__warps_active.avg.pct_of_peak_sustained_active",
        "smsp__inst_executed.sum", "smsp__thread_inst_executed_per_inst_executed.ratio",
        "launch__registers_per_thread", "launch__occupancy_limit_shared_mem",
        "launch__occupancy_limit_registers", "l1tex__data_bank_conflicts_pipe_lsu_mem_shared.sum",
        "smsp__pcsamp_warps_issue_stalled_long_scoreboard",
        "smsp__pcsamp_warps_issue_stalled_short_scoreboard",
        "smsp__pcsamp_warps_issue_stalled_barrier", "smsp__pcsamp_warps_issue_stalled_wait",
        "smsp__pcsamp_warps_issue_stalled_math_pipe_throttle",
        "smsp__pcsamp_warps_issue_stalled_lg_throttle",
        "smsp__pcsamp_warps_issue_stalled_mio_throttle",
        "smsp__pcsamp_warps_issue_stalled_no_instructions",
        "smsp__pcsamp_warps_issue_stalled_not_selected",
        "smsp__pcsamp_warps_issue_stalled_selected"]


def raw(rep):
    out = subprocess.run(["ncu", "-i", rep, "--page", "raw", "--csv"], capture_output=True,
                         text=True).stdout
    rows = list(csv.reader(io.StringIO(out)))
    h = rows[0]
    res = []
    for r in rows[2:]:
        d = dict(zip(h, r))
        res.append(d)
    return res


def main():
    rep = sys.argv[1]
    for d in raw(rep):
        name = d.get("Kernel Name", "?")
        name = name.split("::")[-1].split("(")[0] if "::" in name else name[:40]
        print(f"== {name}")
        for w in WANT:
            if w in d:
                print(f"   {w:70s} {d[w]}")
    if "--source" in sys.argv:
        k = sys.argv[sys.argv.index("--source") + 1]
        out = subprocess.run(["ncu", "-i", rep, "--page", "source", "--csv", "-k", k,
                              "--print-source", "cuda"], capture_output=True, text=True).stdout
        print(out[:200])


if __name__ == "__main__":
    main()
