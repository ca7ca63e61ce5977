"""Build libvapr with -DVAPR_PHASES into /tmp and print per-phase cycles of the
collision kernel (thread 0 of each CTA, summed over CTAs).
    python scripts/phases.py [stage]"""
import ctypes
import os
import subprocess
import sys

ROOT = os.path.join(os.path.dirname(os.path.abspath(__file__)), "..")
sys.path.insert(0, ROOT)
from paper_2310_07854_b200 import build as b  # noqa: E402

so = "/tmp/libvapr_phases.so"
subprocess.check_call([b.NVCC, *b.FLAGS, "-DVAPR_PHASES", "-o", so] +
                      [os.path.join(b.CSRC, f) for f in b.SOURCES])
import paper_2310_07854_b200.binding as vb  # noqa: E402
vb.SO_PATH = so
vb.lib = vb._load()
import torch  # noqa: E402
from paper_2310_07854_b200.rollout import Rollout  # noqa: E402
from workloads import config4  # noqa: E402

stage = sys.argv[1] if len(sys.argv) > 1 else "fused"
wl = config4(formats="43bit")
r = Rollout(wl)
B, H, P = wl.B, wl.H, wl.poses
lay = vb.vapr_cost_grad_workspace_layout(r.ctx.h, B, H, 1)
W = {i: vb.vapr_packed_row_words(r.ctx.formats[i], 156) for i in range(5)}
ws = r.workspace


def slot(i):
    return ws[lay[i]:lay[i] + 4 * W[i] * P]


vb.vapr_fk_spheres(r.ctx.h, r.q, B, H, slot(0))
fn = vb.lib.vapr_debug_phase_cycles
fn.argtypes = [ctypes.c_void_p, ctypes.c_int]
buf = (ctypes.c_ulonglong * 16)()
torch.cuda.synchronize()
fn(buf, 1)
if stage == "world_discrete":
    vb.vapr_world_collision(r.ctx.h, slot(0), r.world_idx, B, H, 0, 0, 0.025, 1.0, r.cost_pose, slot(4))
elif stage == "self":
    vb.vapr_self_collision(r.ctx.h, slot(0), B, H, 0.01, 1.0, r.cost_pose, slot(2))
else:
    vb.vapr_collision(r.ctx.h, slot(0), r.world_idx, B, H, wl.params, r.cost_pose, r.cost_traj, slot(4), slot(2))
torch.cuda.synchronize()
fn(buf, 1)
tot = sum(buf[1:10])
names = ["", "wait", "rows+decode+zero", "balls", "world masks + self L1", "wtask list + self L2",
         "tasks (world, self)", "per-pose cost + touched list", "self gather", "stores"]
for i in range(1, 10):
    print(f"phase {i} {names[i]:24s} {100 * buf[i] / max(tot, 1):5.1f}%  {buf[i] / 1e6:10.1f} Mcyc")
tiles = (P + 31) // 32
print(f"per tile: world tasks {buf[10]/tiles:.1f}  self group-pair tasks {buf[11]/tiles:.1f}  live link pairs {buf[12]/tiles:.1f}  touched spheres {buf[13]/tiles:.1f}  kmax {buf[14]/tiles:.2f}")
print(f"cycles per tile (thread 0 view, summed phases): {sum(buf[1:10])/tiles:.0f}")
