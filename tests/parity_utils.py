"""Comparison rules GPU <-> oracle.

Packed outputs: the GPU code of element i must lie in the code interval
[Q(v_i - delta_i), Q(v_i + delta_i)] of the oracle's double pre-quantisation
value v_i, with delta_i = TOL * (|v_i| + scale_i) and Q the oracle's
double-input quantiser (monotone).  When no rounding midpoint lies within
delta_i the interval is a single code (exact match); otherwise either
neighbouring code is accepted (one step of the stored format).  FP32 outputs:
|gpu - ref| <= TOL * (|ref| + scale) + ATOL, scale = sum of |terms|.
"""
import numpy as np

from oracle import codec

TOL = 1e-5
ATOL = 1e-7


def signed_order(codes, E, M):
    """Map sign-magnitude codes to integers that are monotone in value."""
    t = 1 + E + M
    c = codes.astype(np.int64)
    sign = (c >> (t - 1)) & 1
    mag = c & ((1 << (t - 1)) - 1)
    return np.where(sign == 1, -mag, mag)


def check_codes(gpu_words, v, scale, fmt, cols, skip=None, min_exact=None, what=""):
    """Element-wise interval check of packed GPU output against oracle values.

    gpu_words [P, W] uint32, v [P, cols] float64, scale broadcastable to v."""
    E, M = fmt
    got = codec.unpack(np.asarray(gpu_words, np.uint32), E, M, cols)
    v = np.asarray(v, np.float64).reshape(got.shape)
    delta = TOL * (np.abs(v) + np.broadcast_to(scale, v.shape))
    lo = codec.quantize_f64(v - delta, E, M)
    hi = codec.quantize_f64(v + delta, E, M)
    ref = codec.quantize_f64(v, E, M)
    g = signed_order(got, E, M)
    ok = (g >= signed_order(lo, E, M)) & (g <= signed_order(hi, E, M))
    # +0 / -0 are the same value: accept either sign of zero for a zero interval
    zero_ok = (codec.dequantize(got, E, M) == 0) & (codec.dequantize(lo, E, M) <= 0) & \
              (codec.dequantize(hi, E, M) >= 0)
    ok |= zero_ok
    if skip is not None:
        ok |= np.broadcast_to(skip, ok.shape)
    bad = np.nonzero(~ok)
    assert ok.all(), (f"{what}: {len(bad[0])} codes outside the interval; first at "
                      f"{[b[:5] for b in bad]}: gpu={got[bad][:5]} ref={ref[bad][:5]} "
                      f"v={v[bad][:5]}")
    exact = float(np.mean(got == ref))
    # an exact-match rate is meaningful only when the format's step is far
    # coarser than FP32 evaluation error (M <= 10); E8M23 codes are FP32 bits
    if min_exact is not None and M <= 10:
        assert exact >= min_exact, f"{what}: only {exact:.5f} of codes exact"
    return exact


def check_close(gpu, ref, scale, what="", tol=TOL, atol=ATOL):
    gpu = np.asarray(gpu, np.float64)
    ref = np.asarray(ref, np.float64).reshape(gpu.shape)
    lim = tol * (np.abs(ref) + np.broadcast_to(scale, ref.shape).reshape(gpu.shape)) + atol
    err = np.abs(gpu - ref)
    bad = np.nonzero(err > lim)
    assert not len(bad[0]), (f"{what}: {len(bad[0])} values out of tolerance; first "
                             f"gpu={gpu[bad][:5]} ref={ref[bad][:5]} lim={lim[bad][:5]}")
    return float(np.max(err / lim)) if err.size else 0.0


def sphere_to_elem(scale_ps, S=52):
    """[P, S] per-sphere scale -> [P, 3S] per-element scale."""
    return np.repeat(np.asarray(scale_ps), 3, axis=-1)
