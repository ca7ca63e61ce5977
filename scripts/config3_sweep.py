"""BASELINE config 3, cost path: on the bookshelf workload
(1.024M poses), for each slot each of the 21 canonical formats with the other
four slots at E8M23 (105 runs, the Phase-1 shape of P:249) plus the 21
uniform runs (every slot the same format): vapr_cost_grad ms, G sphere-evals/s
and algorithmic GB/s, in dense and in sparse storage.  One JSON line per run.

    python scripts/config3_sweep.py [--reps 10] [--storage dense,sparse]
"""
import argparse
import json
import os
import sys

sys.path.insert(0, os.path.join(os.path.dirname(os.path.abspath(__file__)), ".."))
import torch  # noqa: E402

from paper_2310_07854_b200.rollout import Rollout  # noqa: E402
from paper_2310_07854_b200.search import enumerate_formats  # noqa: E402
from workloads import config3  # noqa: E402

ap = argparse.ArgumentParser()
ap.add_argument("--reps", type=int, default=10)
ap.add_argument("--storage", default="dense,sparse")
a = ap.parse_args()
S, FP32 = 52, (8, 23)
SLOTS = ("out_spheres", "grad_out_spheres", "out_vec", "closest_pt", "closest_pt_swept")
wl = config3()
P = wl.poses


def v_alg(f):
    return 4.0 * 3 * S / (32 // (1 + f[0] + f[1]))


def a_min(fm):
    # q twice, grad_q, two pose costs, each live tensor written + read once (swept)
    return 28 * 3 + 8 + 2 * (v_alg(fm[0]) + v_alg(fm[1]) + v_alg(fm[2]) + v_alg(fm[4]))


def time_run(r):
    for _ in range(3):
        r.run()
    torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record()
    for _ in range(a.reps):
        r.run()
    e1.record()
    torch.cuda.synchronize()
    return e0.elapsed_time(e1) / a.reps


fmts = enumerate_formats()
for storage in a.storage.split(","):
    r = Rollout(wl, sparse=(storage == "sparse"))
    runs = [("uniform", None, (f,) * 5) for f in fmts]
    for slot in (0, 1, 2, 4):           # closest_pt (slot 3) is not live in swept TO
        for f in fmts:
            fm = [FP32] * 5
            fm[slot] = f
            runs.append(("slot", SLOTS[slot], tuple(fm)))
    runs.append(("uniform", None, (FP32,) * 5))
    for mode, slot, fm in runs:
        r.set_formats(fm)
        ms = time_run(r)
        print(json.dumps({"storage": storage, "mode": mode, "slot": slot,
                          "formats": ["E%dM%d" % f for f in fm], "ms": round(ms, 4),
                          "G_sphere_evals_s": round(P * S / (ms * 1e-3) / 1e9, 3),
                          "alg_GB_s": round(a_min(fm) * P / (ms * 1e-3) / 1e9, 1),
                          "poses": P}), flush=True)
    del r
    torch.cuda.empty_cache()
