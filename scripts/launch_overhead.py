"""Host-side enqueue cost of vapr_cost_grad (launch overhead check)."""
import os
import sys
import time

sys.path.insert(0, os.path.join(os.path.dirname(os.path.abspath(__file__)), ".."))
import torch  # noqa: E402

from paper_2310_07854_b200.rollout import Rollout  # noqa: E402
from workloads import config4  # noqa: E402

for ppe, seeds in ((1, 2), (10, 10), (25, 12), (50, 25), (100, 100)):
    wl = config4(problems_per_env=ppe, seeds=seeds, formats="43bit")
    r = Rollout(wl)
    for _ in range(3):
        r.run()
    torch.cuda.synchronize()
    n = 50 if ppe < 50 else 5
    t0 = time.perf_counter()
    for _ in range(n):
        r.run()
    t1 = time.perf_counter()
    torch.cuda.synchronize()
    t2 = time.perf_counter()
    print(f"poses {wl.poses}: host enqueue {1e3 * (t1 - t0) / n:.3f} ms/call, "
          f"wall incl. GPU {1e3 * (t2 - t0) / n:.3f} ms/call")
