import sys, os; sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch, json
from paper_2310_07854_b200.rollout import Rollout
from workloads import config4
from workloads.configs import FORMAT_SETS
res = {}
for fs in ("43bit", "fp32", "fp16"):
    wl = config4(formats=FORMAT_SETS[fs])
    for mode in ("sparse", "dense", "fused"):
        r = Rollout(wl, sparse=(mode == "sparse"), fused=(mode == "fused"))
        for _ in range(3): r.run()
        torch.cuda.synchronize()
        e0 = torch.cuda.Event(enable_timing=True); e1 = torch.cuda.Event(enable_timing=True)
        e0.record()
        for _ in range(10): r.run()
        e1.record(); torch.cuda.synchronize()
        res[f"{fs}_{mode}"] = e0.elapsed_time(e1) / 10
        del r; torch.cuda.empty_cache()
print(json.dumps(res))
