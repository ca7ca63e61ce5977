"""Run a few vapr_cost_grad steps of the bench workload (config 4 per GPU) for
ncu: `python scripts/prof_step.py [--formats 43bit] [--steps 3]`.
Launch order per step: fk, collision (world pass, self pass), traj_reduce, aggregate, bk."""
import argparse
import os
import sys

sys.path.insert(0, os.path.join(os.path.dirname(os.path.abspath(__file__)), ".."))

import torch  # noqa: E402

from paper_2310_07854_b200.rollout import Rollout  # noqa: E402
from workloads import config4  # noqa: E402

ap = argparse.ArgumentParser()
ap.add_argument("--formats", default="43bit")
ap.add_argument("--steps", type=int, default=3)
ap.add_argument("--problems-per-env", type=int, default=100)
a = ap.parse_args()
wl = config4(problems_per_env=a.problems_per_env, formats=a.formats)
r = Rollout(wl)
for _ in range(a.steps):
    r.run()
torch.cuda.synchronize()
print("ok", wl.poses, a.formats)
