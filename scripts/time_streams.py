import os, sys
sys.path.insert(0, os.getcwd())
import torch, numpy as np
from paper_2310_07854_b200.rollout import Rollout
from workloads import config4
wl = config4(formats="43bit")
r = Rollout(wl)
ref = None
for ns in (1, 2, 3, 4, 1):
    r.ctx.set_streams(ns)
    for _ in range(3): r.run()
    torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record()
    for _ in range(10): r.run()
    e1.record(); torch.cuda.synchronize()
    out = r.results()
    g = out["grad_q"].copy()
    same = ref is None or np.array_equal(g.view(np.uint32), ref.view(np.uint32))
    ref = g if ref is None else ref
    print(ns, round(e0.elapsed_time(e1) / 10, 3), "identical" if same else "DIFFERENT")
