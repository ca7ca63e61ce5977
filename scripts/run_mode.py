"""One vapr_cost_grad of the bench workload in a given mode (for ncu captures):
python scripts/run_mode.py <formats> <sparse|dense|fused> [reps]"""
import os
import sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch
from paper_2310_07854_b200.rollout import Rollout
from workloads import config4
from workloads.configs import FORMAT_SETS

fs, mode = sys.argv[1], sys.argv[2]
reps = int(sys.argv[3]) if len(sys.argv) > 3 else 1
wl = config4(formats=FORMAT_SETS[fs])
r = Rollout(wl, sparse=(mode == "sparse"), fused=(mode == "fused"))
for _ in range(reps):
    r.run()
torch.cuda.synchronize()
print("ok", fs, mode)
