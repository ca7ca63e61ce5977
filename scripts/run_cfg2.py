"""A few vapr_cost_grad calls on config 2 alone (ncu)."""
import os
import sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch
from paper_2310_07854_b200.rollout import Rollout
from workloads import config2

r = Rollout(config2(), sparse=True)
for _ in range(3):
    r.run()
torch.cuda.synchronize()
print("ok")
