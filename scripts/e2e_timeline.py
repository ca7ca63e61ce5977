"""Kernel / memcpy timeline of one vapr_cost_grad_host step (torch.profiler,
CUDA activities) on the bench workload: where the end-to-end time goes."""
import json
import os
import sys

sys.path.insert(0, os.path.join(os.path.dirname(os.path.abspath(__file__)), ".."))
import numpy as np  # noqa: E402
import torch  # noqa: E402
from torch.profiler import ProfilerActivity, profile  # noqa: E402

from paper_2310_07854_b200.rollout import Rollout  # noqa: E402
from workloads import config4  # noqa: E402

chunks = int(sys.argv[1]) if len(sys.argv) > 1 else 0
wl = config4(problems_per_env=100, formats="43bit")
r = Rollout(wl, sparse=True)
P = wl.poses
qh = torch.from_numpy(np.ascontiguousarray(wl.q)).pin_memory()
gh = torch.empty(P * 7, dtype=torch.float32).pin_memory()
ch = torch.empty(wl.B, dtype=torch.float32).pin_memory()
for _ in range(3):
    r.run_host(qh, gh, ch, n_chunks=chunks)
torch.cuda.synchronize()
with profile(activities=[ProfilerActivity.CUDA]) as prof:
    r.run_host(qh, gh, ch, n_chunks=chunks)
    torch.cuda.synchronize()
evs = []
for e in prof.events():
    if e.device_type.name != "CUDA":
        continue
    evs.append((e.time_range.start, e.time_range.end, e.name[:60]))
evs.sort()
t0 = evs[0][0]
for s, t, n in evs:
    print(f"{(s - t0) / 1000:8.3f} {(t - t0) / 1000:8.3f} {(t - s) / 1000:7.3f} ms  {n}")
print("span", (max(t for _, t, _ in evs) - t0) / 1000, "ms")
