"""Success rates of the N4 pipeline evaluator for a few format tuples.
    python scripts/pipeline_rates.py [--ppe 4]"""
import argparse
import json
import os
import sys
import time

sys.path.insert(0, os.path.join(os.path.dirname(os.path.abspath(__file__)), ".."))
from paper_2310_07854_b200.pipeline import PipelineEvaluator  # noqa: E402
from workloads.configs import FORMAT_SETS  # noqa: E402

ap = argparse.ArgumentParser()
ap.add_argument("--ppe", type=int, default=4)
a = ap.parse_args()
ev = PipelineEvaluator(problems_per_env=a.ppe)
cfgs = {"fp32": FORMAT_SETS["fp32"], "43bit": FORMAT_SETS["43bit"], "fp16": FORMAT_SETS["fp16"],
        "e2m1_all": ((2, 1),) * 5, "e3m2_os_rest_e2m1": ((3, 2),) + ((2, 1),) * 4}
out = {}
for name, c in cfgs.items():
    t0 = time.perf_counter()
    rates = ev.evaluate(c)
    dt = time.perf_counter() - t0
    L = ev.last
    out[name] = {"mean_rate": round(float(sum(rates.values()) / len(rates)), 4),
                 "ik_ok": int(L["ik_ok"].sum()), "success": int(L["success"].sum()),
                 "problems": int(len(L["success"])), "seconds": round(dt, 3), "rates": rates}
    print(name, json.dumps(out[name]), flush=True)
print(json.dumps(out))
