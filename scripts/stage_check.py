"""Run each libvapr stage on its own for a format set and report errors
(debugging aid): python scripts/stage_check.py E2M1 [E2M1 ...]"""
import os
import sys

sys.path.insert(0, os.path.join(os.path.dirname(os.path.abspath(__file__)), ".."))
import torch  # noqa: E402

from paper_2310_07854_b200 import binding as vb  # noqa: E402
from paper_2310_07854_b200 import search as S  # noqa: E402
from paper_2310_07854_b200.rollout import Rollout  # noqa: E402
from workloads import config5  # noqa: E402


def parse(s):
    e, m = s[1:].split("M")
    return (int(e), int(m))


fm = [parse(x) for x in sys.argv[1:]] or [(2, 1)] * 5
fm = (fm * 5)[:5]
wl = config5(problems_per_env=2, seeds=4)
r = Rollout(wl, formats=tuple(fm))
B, H, P = wl.B, wl.H, wl.poses
lay = vb.vapr_cost_grad_workspace_layout(r.ctx.h, B, H, 1)
W = {i: vb.vapr_packed_row_words(r.ctx.formats[i], 156) for i in range(5)}
ws = r.workspace


def slot(i):
    return ws[lay[i]:lay[i] + 4 * W[i] * P]


steps = [
    ("fk", lambda: vb.vapr_fk_spheres(r.ctx.h, r.q, B, H, slot(0))),
    ("world", lambda: vb.vapr_world_collision(r.ctx.h, slot(0), r.world_idx, B, H, 1, 1, 0.025, 1.0,
                                              r.cost_pose, slot(4))),
    ("self", lambda: vb.vapr_self_collision(r.ctx.h, slot(0), B, H, 0.01, 1.0, r.cost_pose, slot(2))),
    ("fused", lambda: vb.vapr_collision(r.ctx.h, slot(0), r.world_idx, B, H, wl.params, r.cost_pose,
                                        r.cost_traj, slot(4), slot(2))),
    ("run", lambda: r.run()),
]
print("formats", fm, "W", W)
for name, fn in steps:
    try:
        fn()
        torch.cuda.synchronize()
        print(name, "ok")
    except Exception as e:  # noqa: BLE001
        print(name, "FAILED", e)
        try:
            torch.cuda.synchronize()
            print("sync ok (error was a launch error, not sticky)")
        except Exception as e2:  # noqa: BLE001
            print("sticky:", e2)
        break
