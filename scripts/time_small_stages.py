"""Per-stage latency of vapr_cost_grad on configs 1 / 2 from the call's own
stage events (vapr_set_stage_events), eager, warm."""
import os
import sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch
from paper_2310_07854_b200 import binding as vb
from paper_2310_07854_b200.rollout import Rollout
from workloads import config1, config2

for name, wl in (("config1", config1()), ("config2", config2())):
    for sparse in (False, True):
        r = Rollout(wl, sparse=sparse)
        ev = [torch.cuda.Event(enable_timing=True) for _ in range(6)]
        vb.vapr_set_stage_events(r.ctx.h, ev)
        acc = [0.0] * 5
        n = 50
        for i in range(n + 10):
            r.run()
            torch.cuda.synchronize()
            if i >= 10:
                for k in range(5):
                    acc[k] += 1e3 * ev[k].elapsed_time(ev[k + 1]) / n
        print(f"{name} sparse={int(sparse)}: " + " ".join(
            f"{s} {v:.1f}" for s, v in zip(["fk", "coll", "red", "agg", "bk"], acc)) +
            f"  sum {sum(acc):.1f} us", flush=True)
