"""Latency of vapr_cost_grad and of its stages on the small BASELINE configs
(config 1: 128 poses, config 2: 384 poses), CUDA events, many repetitions."""
import os
import sys

sys.path.insert(0, os.path.join(os.path.dirname(os.path.abspath(__file__)), ".."))
import torch  # noqa: E402

from paper_2310_07854_b200 import binding as vb  # noqa: E402
from paper_2310_07854_b200.rollout import Rollout  # noqa: E402
from workloads import config1, config2  # noqa: E402


def t(fn, reps=200):
    for _ in range(20):
        fn()
    torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record()
    for _ in range(reps):
        fn()
    e1.record()
    torch.cuda.synchronize()
    return 1e3 * e0.elapsed_time(e1) / reps


for name, wl in (("config1", config1()), ("config2", config2())):
    for sparse in (False, True):
        r = Rollout(wl, sparse=sparse)
        g = r.capture_graph()
        line = f"{name} sparse={int(sparse)} eager {t(r.run):7.1f} us  graph {t(g.replay):7.1f} us"
        if not sparse:
            lay = vb.vapr_cost_grad_workspace_layout(r.ctx.h, wl.B, wl.H, 1)
            fm = r.ctx.formats
            Wd = {i: vb.vapr_packed_row_words(fm[i], 156) for i in range(5)}
            P = wl.poses
            sl = lambda i: r.workspace[lay[i]:lay[i] + 4 * Wd[i] * P]
            line += (f"  | fk {t(lambda: vb.vapr_fk_spheres(r.ctx.h, r.q, wl.B, wl.H, sl(0))):6.1f}"
                     f" coll {t(lambda: vb.vapr_collision(r.ctx.h, sl(0), r.world_idx, wl.B, wl.H, r.params, r.cost_pose, r.cost_traj, sl(4), sl(2))):6.1f}"
                     f" agg {t(lambda: vb.vapr_aggregate(r.ctx.h, sl(4), 1, sl(2), P, sl(1))):6.1f}"
                     f" bk {t(lambda: vb.vapr_backward_kinematics(r.ctx.h, r.q, wl.B, wl.H, sl(1), r.grad_q)):6.1f}")
        print(line, flush=True)
