"""Run one libvapr stage a few times on the bench workload (for ncu).
    python scripts/prof_stage.py {world_discrete,world_swept,self,fused} [--cull 1]"""
import argparse
import os
import sys

sys.path.insert(0, os.path.join(os.path.dirname(os.path.abspath(__file__)), ".."))
import torch  # noqa: E402

from paper_2310_07854_b200 import binding as vb  # noqa: E402
from paper_2310_07854_b200.rollout import Rollout  # noqa: E402
from workloads import config4  # noqa: E402

ap = argparse.ArgumentParser()
ap.add_argument("stage")
ap.add_argument("--cull", type=int, default=1)
ap.add_argument("--reps", type=int, default=2)
a = ap.parse_args()
wl = config4(formats="43bit")
r = Rollout(wl)
B, H, P = wl.B, wl.H, wl.poses
lay = vb.vapr_cost_grad_workspace_layout(r.ctx.h, B, H, 1)
W = {i: vb.vapr_packed_row_words(r.ctx.formats[i], 156) for i in range(5)}
ws = r.workspace


def slot(i):
    return ws[lay[i]:lay[i] + 4 * W[i] * P]


r.ctx.set_cull(a.cull)
vb.vapr_fk_spheres(r.ctx.h, r.q, B, H, slot(0))
for _ in range(a.reps):
    if a.stage == "world_discrete":
        vb.vapr_world_collision(r.ctx.h, slot(0), r.world_idx, B, H, 0, 0, 0.025, 1.0, r.cost_pose, slot(4))
    elif a.stage == "world_swept":
        vb.vapr_world_collision(r.ctx.h, slot(0), r.world_idx, B, H, 1, 1, 0.025, 1.0, r.cost_pose, slot(4))
    elif a.stage == "self":
        vb.vapr_self_collision(r.ctx.h, slot(0), B, H, 0.01, 1.0, r.cost_pose, slot(2))
    else:
        vb.vapr_collision(r.ctx.h, slot(0), r.world_idx, B, H, wl.params, r.cost_pose, r.cost_traj,
                          slot(4), slot(2))
torch.cuda.synchronize()
print("ok")
