"""Small-batch latency of vapr_cost_grad vs poses per collision tile
(VAPR_TILE_POSES; unset = the launcher's choice)."""
import os
import sys

sys.path.insert(0, os.path.join(os.path.dirname(os.path.abspath(__file__)), ".."))
import torch  # noqa: E402

from paper_2310_07854_b200.rollout import Rollout  # noqa: E402
from workloads import config1, config2, config4  # noqa: E402


def t(fn, reps=200):
    for _ in range(20):
        fn()
    torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record()
    for _ in range(reps):
        fn()
    e1.record()
    torch.cuda.synchronize()
    return 1e3 * e0.elapsed_time(e1) / reps


wls = (("config1", config1()), ("config2", config2()),
       ("c4_small", config4(problems_per_env=1, seeds=10, H=32)))
for tp in ("auto", "15", "8", "4", "2", "1"):
    if tp == "auto":
        os.environ.pop("VAPR_TILE_POSES", None)
    else:
        os.environ["VAPR_TILE_POSES"] = tp
    line = f"tile_poses={tp:>4s}"
    for name, wl in wls:
        r = Rollout(wl, sparse=True)
        g = r.capture_graph()
        line += f"  {name} {t(g.replay):7.1f} us"
        del g, r
    print(line, flush=True)
