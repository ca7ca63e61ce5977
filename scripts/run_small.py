"""A few vapr_cost_grad calls on config 1 / config 2 (ncu launch lists)."""
import os
import sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch
from paper_2310_07854_b200.rollout import Rollout
from workloads import config1, config2

for wl in (config1(), config2()):
    r = Rollout(wl, sparse=len(sys.argv) > 1 and sys.argv[1] == "sparse")
    for _ in range(3):
        r.run()
    torch.cuda.synchronize()
print("ok")
