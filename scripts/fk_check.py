"""FK alone for one out_spheres format (debugging aid)."""
import os
import sys

sys.path.insert(0, os.path.join(os.path.dirname(os.path.abspath(__file__)), ".."))
import torch  # noqa: E402

from paper_2310_07854_b200 import binding as vb  # noqa: E402
from paper_2310_07854_b200.rollout import Context  # noqa: E402
from workloads import config1  # noqa: E402

e, m = sys.argv[1][1:].split("M")
fm = ((int(e), int(m)),) + ((4, 3),) * 4
n = int(sys.argv[2]) if len(sys.argv) > 2 else 1
wl = config1()
ctx = Context(0, wl.robot, fm, wl.cuboids, wl.world_offsets)
P = n
q = torch.zeros(P * 7, device="cuda")
W = vb.vapr_packed_row_words(fm[0], 156)
os_ = torch.zeros(P * W * 4, dtype=torch.uint8, device="cuda")
try:
    vb.vapr_fk_spheres(ctx.h, q, P, 1, os_)
    torch.cuda.synchronize()
    print(sys.argv[1], P, "ok")
except Exception as ex:  # noqa: BLE001
    print(sys.argv[1], P, "FAILED", str(ex).splitlines()[0])
