"""Throughput of vapr_quantize / vapr_dequantize (BASELINE config 3 codec
sweep shape: 2^28 FP32 elements per format, position-shaped values).
    python scripts/codec_bench.py [--log2n 28] [--formats all|E5M10,E2M1]"""
import argparse
import json
import os
import sys

sys.path.insert(0, os.path.join(os.path.dirname(os.path.abspath(__file__)), ".."))
import torch  # noqa: E402

from paper_2310_07854_b200 import binding as vb  # noqa: E402
from paper_2310_07854_b200.search import enumerate_formats  # noqa: E402

ap = argparse.ArgumentParser()
ap.add_argument("--log2n", type=int, default=28)
ap.add_argument("--formats", default="all")
ap.add_argument("--cols", type=int, default=156)
a = ap.parse_args()
fmts = enumerate_formats() if a.formats == "all" else [vb.vapr_format_parse(f) for f in a.formats.split(",")]
n = 1 << a.log2n
cols = a.cols
rows = n // cols
x = (torch.rand(rows * cols, device="cuda") * 2.2 - 1.0)
y = torch.empty_like(x)
peak = json.load(open(os.path.join(os.path.dirname(__file__), "..", "MEASURED_PEAKS.json")))["hbm_gbs"] \
    if os.path.exists(os.path.join(os.path.dirname(__file__), "..", "MEASURED_PEAKS.json")) else 6650.0
out = []
for f in fmts:
    W = vb.vapr_packed_row_words(f, cols)
    packed = torch.empty(rows * W, dtype=torch.int32, device="cuda")
    for name, fn, nbytes in (
            ("quantize", lambda: vb.vapr_quantize(f, x, rows, cols, packed), 4 * rows * cols + 4 * rows * W),
            ("dequantize", lambda: vb.vapr_dequantize(f, packed, rows, cols, y), 4 * rows * cols + 4 * rows * W)):
        for _ in range(3):
            fn()
        torch.cuda.synchronize()
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record()
        reps = 10
        for _ in range(reps):
            fn()
        e1.record()
        torch.cuda.synchronize()
        ms = e0.elapsed_time(e1) / reps
        gbs = nbytes / (ms * 1e-3) / 1e9
        out.append({"format": "E%dM%d" % f, "op": name, "ms": round(ms, 4), "GB_s": round(gbs, 1),
                    "frac": round(gbs / peak, 3), "Gelem_s": round(rows * cols / (ms * 1e-3) / 1e9, 2)})
        print(json.dumps(out[-1]), flush=True)
