"""Time each libvapr stage separately on the bench workload (CUDA events).

    python scripts/time_stages.py [--formats 43bit] [--ppe 100]
"""
import argparse
import os
import sys

sys.path.insert(0, os.path.join(os.path.dirname(os.path.abspath(__file__)), ".."))
import torch  # noqa: E402

from paper_2310_07854_b200 import binding as vb  # noqa: E402
from paper_2310_07854_b200.rollout import Rollout  # noqa: E402
from workloads import config4  # noqa: E402

ap = argparse.ArgumentParser()
ap.add_argument("--formats", default="43bit")
ap.add_argument("--ppe", type=int, default=100)
ap.add_argument("--reps", type=int, default=5)
a = ap.parse_args()
wl = config4(problems_per_env=a.ppe, formats=a.formats)
r = Rollout(wl)
P = wl.poses
B, H = wl.B, wl.H
p = wl.params
lay = vb.vapr_cost_grad_workspace_layout(r.ctx.h, B, H, 1)
fm = r.ctx.formats
W = {i: vb.vapr_packed_row_words(fm[i], 156) for i in range(5)}
ws = r.workspace


def slot(i):
    return ws[lay[i]:lay[i] + 4 * W[i] * P]


def t(fn, name):
    for _ in range(2):
        fn()
    torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record()
    for _ in range(a.reps):
        fn()
    e1.record()
    torch.cuda.synchronize()
    print(f"{name:28s} {e0.elapsed_time(e1) / a.reps:8.3f} ms", flush=True)


t(lambda: vb.vapr_fk_spheres(r.ctx.h, r.q, B, H, slot(0)), "fk")
for cull in (1, 0):
    r.ctx.set_cull(cull)
    t(lambda: vb.vapr_world_collision(r.ctx.h, slot(0), r.world_idx, B, H, 1, 1, 0.025, 1.0,
                                      r.cost_pose, slot(4)), f"world swept cull={cull}")
    t(lambda: vb.vapr_world_collision(r.ctx.h, slot(0), r.world_idx, B, H, 0, 0, 0.025, 1.0,
                                      r.cost_pose, slot(4)), f"world discrete cull={cull}")
    t(lambda: vb.vapr_self_collision(r.ctx.h, slot(0), B, H, 0.01, 1.0, r.cost_pose, slot(2)),
      f"self cull={cull}")
    t(lambda: vb.vapr_collision(r.ctx.h, slot(0), r.world_idx, B, H, p, r.cost_pose, r.cost_traj,
                                slot(4), slot(2)), f"collision fused cull={cull}")
r.ctx.set_cull(1)
t(lambda: vb.vapr_aggregate(r.ctx.h, slot(4), 1, slot(2), P, slot(1)), "aggregate")
t(lambda: vb.vapr_backward_kinematics(r.ctx.h, r.q, B, H, slot(1), r.grad_q), "bk")
t(lambda: r.run(), "cost_grad")
