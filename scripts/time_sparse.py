import sys, os
sys.path.insert(0, os.getcwd())
import torch, numpy as np
from paper_2310_07854_b200.rollout import Rollout
from workloads import config4
wl = config4(problems_per_env=100, formats="43bit")
res = {}
for sparse in (False, True, False, True):
    r = Rollout(wl, sparse=sparse)
    for _ in range(3): r.run()
    torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record()
    for _ in range(10): r.run()
    e1.record(); torch.cuda.synchronize()
    ms = e0.elapsed_time(e1) / 10
    extra = ""
    if sparse:
        sg = r.sparse_gos()
        P = wl.B * wl.H
        extra = f"used words {sg['used']} sparse bytes {12*P + 4*sg['used']} dense bytes {P*4*32}"
    print(f"sparse={sparse} cost_grad {ms:.3f} ms {extra}", flush=True)
    del r; torch.cuda.empty_cache()
