"""bench.py's per-environment Table II leg alone: the eight environments'
sub-batches (each with its own Table II formats) back to back as one step."""
import os
import sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch
from paper_2310_07854_b200 import binding as vb
from paper_2310_07854_b200.rollout import Rollout
from workloads import config4
from workloads.configs import FORMAT_SETS
from workloads.scenes import ENVIRONMENTS

subs = []
for e, env in enumerate(ENVIRONMENTS):
    eids = [p for p in range(800) if p % 8 == e]
    we = config4(problems_per_env=100, seeds=100, H=32, formats=FORMAT_SETS[env], problem_ids=eids)
    subs.append((env, Rollout(we, sparse=True)))


def step():
    for _, r in subs:
        r.run()


def t(fn, k=10):
    for _ in range(3):
        fn()
    torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record()
    for _ in range(k):
        fn()
    e1.record()
    torch.cuda.synchronize()
    return e0.elapsed_time(e1) / k


line = f"{os.environ.get('VAPR_SO', 'release')}: step {t(step):.3f} ms |"
for env, r in subs:
    line += f" {env} {t(r.run):.3f}"
print(line, flush=True)
