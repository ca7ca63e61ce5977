"""Step time and per-stage times (stage events) of vapr_cost_grad on the bench
workload: python scripts/time_step.py [formats] [sparse|dense|fused]
(VAPR_SO selects a variant library)."""
import os
import sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch
from paper_2310_07854_b200 import binding as vb
from paper_2310_07854_b200.rollout import Rollout
from workloads import config4
from workloads.configs import FORMAT_SETS

fs = sys.argv[1] if len(sys.argv) > 1 else "43bit"
mode = sys.argv[2] if len(sys.argv) > 2 else "sparse"
wl = config4(formats=FORMAT_SETS[fs])
r = Rollout(wl, sparse=(mode == "sparse"), fused=(mode == "fused"))
for _ in range(3):
    r.run()
torch.cuda.synchronize()
e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
e0.record()
for _ in range(10):
    r.run()
e1.record()
torch.cuda.synchronize()
step = e0.elapsed_time(e1) / 10
ev = [torch.cuda.Event(enable_timing=True) for _ in range(6)]
vb.vapr_set_stage_events(r.ctx.h, ev)
acc = [0.0] * 5
for _ in range(5):
    r.run()
    torch.cuda.synchronize()
    for i in range(5):
        acc[i] += ev[i].elapsed_time(ev[i + 1]) / 5
vb.vapr_set_stage_events(r.ctx.h, None)
print(f"{os.environ.get('VAPR_SO', 'release')} {fs} {mode} step {step:.3f} ms  "
      + " ".join(f"{n} {v:.3f}" for n, v in zip(["fk", "coll", "red", "agg", "bk"], acc)), flush=True)
