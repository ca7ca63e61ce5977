"""End-to-end host-buffer call (vapr_cost_grad_host) on the bench workload vs
the number of trajectory chunks (0 = the library's automatic choice)."""
import os
import sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np
import torch
from paper_2310_07854_b200.rollout import Rollout
from workloads import config4

wl = config4(formats="43bit")
r = Rollout(wl, sparse=True)
qh = torch.from_numpy(np.ascontiguousarray(wl.q)).pin_memory()
gh = torch.empty(wl.poses * 7, dtype=torch.float32).pin_memory()
ch = torch.empty(wl.B, dtype=torch.float32).pin_memory()
for nc in (0, 2, 3, 4, 5, 6, 8):
    for _ in range(3):
        r.run_host(qh, gh, ch, n_chunks=nc)
    torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record()
    for _ in range(10):
        r.run_host(qh, gh, ch, n_chunks=nc)
    e1.record()
    torch.cuda.synchronize()
    print(f"chunks {nc}: {e0.elapsed_time(e1) / 10:.3f} ms", flush=True)
