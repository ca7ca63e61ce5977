import os, sys
sys.path.insert(0, os.path.join(os.path.dirname(os.path.abspath(__file__)), ".."))
import numpy as np, torch
from paper_2310_07854_b200.rollout import Rollout
from paper_2310_07854_b200 import search as S
from workloads import config5
wl = config5(problems_per_env=2, seeds=4)
r = Rollout(wl, formats=(S.FP32,)*5)
def run(cfg):
    r.set_formats(cfg); r.run(); x = r.results()
    return {k: np.array(v).copy() for k, v in x.items()}
c1 = ((2, 1),) * 5
c2 = ((5, 10), (4, 3), (2, 2), (4, 3), (4, 3))
a = run(c1); b = run(c2); a2 = run(c1); b2 = run(c2); a3 = run(c1)
for n, (u, v) in {"c1": (a, a2), "c2": (b, b2), "c1b": (a2, a3)}.items():
    for k in u:
        d = np.array_equal(u[k].view(np.uint8), v[k].view(np.uint8))
        if not d:
            uu, vv = u[k].ravel(), v[k].ravel()
            bad = np.nonzero(uu.view(np.uint32) != vv.view(np.uint32))[0] if uu.dtype.itemsize == 4 else []
            print(n, k, "DIFF", len(bad), bad[:10], uu[bad[:5]], vv[bad[:5]])
        else:
            print(n, k, "same")
