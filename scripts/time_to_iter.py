"""Time a full TO iteration (N1) on the bench workload: candidates +
vapr_cost_grad over the N x B line-search batch + select/history/direction.
    python scripts/time_to_iter.py [--ppe 100] [--seeds 100] [--iters 5]"""
import argparse
import json
import os
import sys

sys.path.insert(0, os.path.join(os.path.dirname(os.path.abspath(__file__)), ".."))
import torch  # noqa: E402

from paper_2310_07854_b200 import binding as vb  # noqa: E402
from paper_2310_07854_b200.optimize import TrajOpt  # noqa: E402
from workloads import config4, config_iko  # noqa: E402

ap = argparse.ArgumentParser()
ap.add_argument("--ppe", type=int, default=100)
ap.add_argument("--seeds", type=int, default=100)
ap.add_argument("--iters", type=int, default=5)
ap.add_argument("--formats", default="43bit")
ap.add_argument("--iko", action="store_true", help="the N2 IKO workload (H=1, --seeds per problem)")
a = ap.parse_args()
wl = (config_iko(problems_per_env=a.ppe, seeds=a.seeds, formats=a.formats) if a.iko else
      config4(problems_per_env=a.ppe, seeds=a.seeds, H=32, formats=a.formats))
opt = TrajOpt(wl)
opt.reset()
for _ in range(2):
    opt.step()
torch.cuda.synchronize()
ev = [torch.cuda.Event(enable_timing=True) for _ in range(4)]
acc = [0.0, 0.0, 0.0]
for _ in range(a.iters):
    ev[0].record()
    vb.vapr_lbfgs_candidates(opt.x, opt.d, opt.B, opt.D, opt.scales, opt.lines.q.view(-1))
    ev[1].record()
    opt.lines.run()
    ev[2].record()
    vb.vapr_lbfgs_step(opt.B, opt.D, opt.scales, opt.lines.cost_traj, opt.lines.grad_q.view(-1),
                       opt.x, opt.g, opt.cost, opt.d, opt.hist_s, opt.hist_y, opt.hist_rho,
                       opt.hist_count, opt.hist_head, opt.chosen, opt.m, opt.eps)
    ev[3].record()
    torch.cuda.synchronize()
    for i in range(3):
        acc[i] += ev[i].elapsed_time(ev[i + 1])
ms = [v / a.iters for v in acc]
print(json.dumps({"B": opt.B, "N": opt.N, "D": opt.D, "poses_per_iter": opt.N * wl.poses,
                  "candidates_ms": round(ms[0], 4), "cost_grad_ms": round(ms[1], 4),
                  "lbfgs_step_ms": round(ms[2], 4), "iter_ms": round(sum(ms), 4),
                  "mean_cost": float(opt.cost.mean()),
                  "hist_count_mean": float(opt.hist_count.float().mean())}))
