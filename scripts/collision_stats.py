"""Work counters of the collision kernel on the bench workload (needs the
variant build: python -m paper_2310_07854_b200.build --variant stats -DVAPR_STATS;
run with VAPR_SO=paper_2310_07854_b200/variants/libvapr_stats.so)."""
import ctypes
import os
import sys

sys.path.insert(0, os.path.join(os.path.dirname(os.path.abspath(__file__)), ".."))
import torch  # noqa: E402

from paper_2310_07854_b200 import binding as vb  # noqa: E402
from paper_2310_07854_b200.rollout import Rollout  # noqa: E402
from workloads import config4  # noqa: E402

wl = config4(formats="43bit")
r = Rollout(wl)
B, H, P = wl.B, wl.H, wl.poses
lay = vb.vapr_cost_grad_workspace_layout(r.ctx.h, B, H, 1)
W = {i: vb.vapr_packed_row_words(r.ctx.formats[i], 156) for i in range(5)}
ws = r.workspace
lib = ctypes.CDLL(vb.SO_PATH)
buf = (ctypes.c_ulonglong * 8)()


def slot(i):
    return ws[lay[i]:lay[i] + 4 * W[i] * P]


def stats(tag):
    torch.cuda.synchronize()
    lib.vapr_debug_stats(buf, 1)
    v = list(buf)
    poses = max(v[7], 1)
    names = ["world items", "world terms", "live group pairs", "chunks", "candidate pairs",
             "touched spheres", "active pmask words", "poses"]
    print(tag, {n: round(x / poses, 3) for n, x in zip(names, v)})


vb.vapr_fk_spheres(r.ctx.h, r.q, B, H, slot(0))
torch.cuda.synchronize()
lib.vapr_debug_stats(buf, 1)
vb.vapr_world_collision(r.ctx.h, slot(0), r.world_idx, B, H, 1, 1, 0.025, 1.0, r.cost_pose, slot(4))
stats("world swept")
vb.vapr_world_collision(r.ctx.h, slot(0), r.world_idx, B, H, 0, 0, 0.025, 1.0, r.cost_pose, slot(4))
stats("world discrete")
vb.vapr_self_collision(r.ctx.h, slot(0), B, H, 0.01, 1.0, r.cost_pose, slot(2))
stats("self")
