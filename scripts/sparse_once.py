"""One dense and one sparse vapr_cost_grad on the bench workload (for ncu launch lists)."""
import os
import sys

sys.path.insert(0, os.path.join(os.path.dirname(os.path.abspath(__file__)), ".."))
import torch  # noqa: E402

from paper_2310_07854_b200.rollout import Rollout  # noqa: E402
from workloads import config4  # noqa: E402

wl = config4(problems_per_env=100, formats=sys.argv[1] if len(sys.argv) > 1 else "43bit")
for sparse in (False, True):
    r = Rollout(wl, sparse=sparse)
    r.run()
    r.run()
    torch.cuda.synchronize()
    del r
    torch.cuda.empty_cache()
