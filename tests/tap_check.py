"""Parity contract (i): run under VAPR_SO=libvapr_tap.so
(tests/test_gpu_tap.py does).  For every packed tensor vapr_cost_grad
produces, the oracle codec (oracle/codec.c) applied to the kernel's own FP32
pre-quantisation values (vapr_debug_tap) must equal the packed words bit for
bit.  Prints one JSON line per (workload, slot); exit status 1 on a mismatch."""
import json
import os
import sys

HERE = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, os.path.join(HERE, ".."))
import numpy as np  # noqa: E402
import torch  # noqa: E402

from paper_2310_07854_b200 import binding as vb  # noqa: E402
from paper_2310_07854_b200.rollout import Rollout  # noqa: E402
from oracle import codec  # noqa: E402
from workloads import config4, config_iko  # noqa: E402

assert hasattr(vb.lib, "vapr_debug_tap"), "not the tap build (set VAPR_SO)"
cases = [("43bit", config4(problems_per_env=1, seeds=8, H=32, formats="43bit")),
         ("pf5_pf8", config4(problems_per_env=1, seeds=8, H=32, formats="pf5_pf8")),
         ("bookshelf_tall", config4(problems_per_env=1, seeds=8, H=32, formats="bookshelf_tall")),
         ("table_pick", config4(problems_per_env=1, seeds=8, H=32, formats="table_pick")),
         ("fp16", config4(problems_per_env=1, seeds=8, H=32, formats="fp16")),
         ("iko_43bit", config_iko(problems_per_env=1, seeds=32, formats="43bit"))]
ok_all = True
for name, wl in cases:
    r = Rollout(wl)
    P, cols = wl.poses, 3 * len(wl.robot["sphere_link"])
    slots = [0, 1, 2, 4 if wl.params["swept"] else 3]
    taps = {sl: torch.full((P * cols,), float("nan"), dtype=torch.float32, device="cuda")
            for sl in slots}
    for sl, t in taps.items():
        vb._check(vb.lib.vapr_debug_tap(r.ctx.h, sl, t.data_ptr()), "vapr_debug_tap")
    r.run()
    torch.cuda.synchronize()
    for sl, t in taps.items():
        fmt = r.ctx.formats[sl]
        v = t.cpu().numpy().reshape(P, cols)
        ref = codec.quantize_packed(v, *fmt)
        got = r.packed(sl)
        same = bool(np.array_equal(got, ref))
        nz = int(np.count_nonzero(v))
        ok_all &= same and not np.isnan(v).any()
        print(json.dumps({"workload": name, "slot": sl, "format": "E%dM%d" % fmt,
                          "bit_exact": same, "nonzero_values": nz, "rows": P}), flush=True)
    del r
sys.exit(0 if ok_all else 1)
