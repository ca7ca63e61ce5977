"""Pins for the ExMy codec oracle (CPU only).

Every check compares the oracle against something other than itself: printed
values (tests/golden/codec_examples.txt), library routines that implement the
same rounding for some formats (numpy float16, torch bfloat16/float8,
ml_dtypes fp4/fp6/fp8), an independent enumeration oracle, and invariants.
"""
import numpy as np
import pytest
import torch

from conftest import golden
from oracle import codec
from oracle.formats import enumerate_formats
from workloads.configs import codec_sweep_inputs, edge_values

ALL_FORMATS = enumerate_formats() + [(6, 6), (5, 9), (6, 8)]   # + Table II FP13/FP15


def parse_fmt(s):
    s = s.upper()
    return int(s[1:s.index("M")]), int(s[s.index("M") + 1:])


def fq(x, f):
    return codec.fake_quant(np.asarray(x, np.float32), *f)


def midpoints(E, M):
    """All midpoints between adjacent non-negative magnitudes, and the FP32
    neighbours one ulp either side, as float32 (exact: each midpoint has at
    most M + 2 significant bits)."""
    mags = codec.representable_magnitudes(E, M)
    mids = ((mags[:-1] + mags[1:]) / 2).astype(np.float32)
    up = np.nextafter(mids, np.float32(np.inf))
    dn = np.nextafter(mids, np.float32(0))
    vals = np.concatenate([mids, up, dn, mags.astype(np.float32)])
    return np.concatenate([vals, -vals])


def test_golden_examples():
    for fmt, x, want in golden("codec_examples.txt"):
        f = parse_fmt(fmt)
        got = fq([float(x)], f)[0]
        assert got == np.float32(want), (fmt, x, got, want)


def test_e2m1_representable_set():
    # {0, 0.5, 1, 1.5, 2, 3, 4, 6}
    vals = codec.dequantize(np.arange(8, dtype=np.uint32), 2, 1)
    assert list(vals) == [0, 0.5, 1, 1.5, 2, 3, 4, 6]
    assert list(codec.representable_magnitudes(2, 1)) == [0, 0.5, 1, 1.5, 2, 3, 4, 6]


def test_max_finite_table():
    # SURVEY.md Appendix A max_finite column (E8 formats clamp to <= FLT_MAX)
    table = {(2, 1): 6, (2, 2): 7, (3, 1): 24, (2, 3): 7.5, (3, 2): 28, (4, 1): 384,
             (2, 5): 7.875, (3, 4): 31, (4, 3): 480, (5, 2): 114688, (2, 7): 7.96875,
             (3, 6): 31.75, (4, 5): 504, (5, 4): 126976, (5, 10): 131008, (5, 9): 130944}
    for (E, M), v in table.items():
        assert fq([1e30], (E, M))[0] == np.float32(v), (E, M)
        assert fq([-np.inf], (E, M))[0] == -np.float32(v)
    assert fq([np.float32(3.4e38)], (8, 7))[0] == np.float32(torch.finfo(torch.bfloat16).max)


def _ref_compare(x, f, ref):
    got = fq(x, f)
    np.testing.assert_array_equal(got.view(np.uint32), np.asarray(ref, np.float32).view(np.uint32))


def _inputs(n=200000, key=1):
    x = np.concatenate([codec_sweep_inputs(n, "bits", key), codec_sweep_inputs(n, "position", key),
                        codec_sweep_inputs(n, "gradient", key),
                        (codec_sweep_inputs(n, "position", key + 7) * 1e3).astype(np.float32),
                        (codec_sweep_inputs(n, "position", key + 9) * 1e-3).astype(np.float32)])
    return x[np.isfinite(x)]


def test_library_float16_is_e5m10():
    x = np.concatenate([_inputs(), midpoints(5, 10)])
    x = x[np.abs(x) < 65520]
    _ref_compare(x, (5, 10), x.astype(np.float16).astype(np.float32))


def test_library_bfloat16_is_e8m7():
    x = np.concatenate([_inputs(), midpoints(8, 7)[:200000]])
    bmax = float(torch.finfo(torch.bfloat16).max)
    x = x[np.abs(x.astype(np.float64)) < bmax]
    ref = torch.from_numpy(x).to(torch.bfloat16).to(torch.float32).numpy()
    _ref_compare(x, (8, 7), ref)


@pytest.mark.parametrize("fmt,dtype,limit", [
    ((4, 3), torch.float8_e4m3fn, 464.0),
    ((5, 2), torch.float8_e5m2, 61440.0),
])
def test_library_torch_float8(fmt, dtype, limit):
    x = np.concatenate([_inputs(), midpoints(*fmt)])
    x = x[np.abs(x) < limit]
    ref = torch.from_numpy(x).to(dtype).to(torch.float32).numpy()
    _ref_compare(x, fmt, ref)


@pytest.mark.parametrize("fmt,name,limit", [
    ((2, 1), "float4_e2m1fn", None),
    ((2, 3), "float6_e2m3fn", None),
    ((3, 2), "float6_e3m2fn", None),
    ((3, 4), "float8_e3m4", 15.75),
    ((4, 3), "float8_e4m3", 248.0),
])
def test_library_ml_dtypes(fmt, name, limit):
    ml = pytest.importorskip("ml_dtypes")
    x = np.concatenate([_inputs(), midpoints(*fmt)])
    if limit is not None:
        x = x[np.abs(x) < limit]
    x = x[~np.isnan(x)]
    ref = x.astype(getattr(ml, name)).astype(np.float32)
    _ref_compare(x, fmt, ref)


@pytest.mark.parametrize("fmt", [f for f in ALL_FORMATS if 1 + f[0] + f[1] <= 16])
def test_formula_matches_enumeration(fmt):
    x = np.concatenate([_inputs(50000, key=3), midpoints(*fmt), edge_values()])
    a = codec.quantize(x, *fmt)
    b = codec.quantize_enum(x, *fmt)
    np.testing.assert_array_equal(a, b)


@pytest.mark.parametrize("fmt", [f for f in ALL_FORMATS if 1 + f[0] + f[1] <= 16])
def test_code_round_trip_exhaustive(fmt):
    E, M = fmt
    t = 1 + E + M
    codes = np.arange(2 ** t, dtype=np.uint32)
    if E == 8:          # exponent field 255 is never produced (c7)
        expf = (codes >> M) & 0xFF
        codes = codes[expf != 255]
    vals = codec.dequantize(codes, E, M)
    assert np.all(np.isfinite(vals))
    np.testing.assert_array_equal(codec.quantize(vals, E, M), codes)


@pytest.mark.parametrize("fmt", ALL_FORMATS)
def test_invariants(fmt):
    x = _inputs(50000, key=5)
    q1 = fq(x, fmt)
    np.testing.assert_array_equal(fq(q1, fmt).view(np.uint32), q1.view(np.uint32))   # idempotent
    np.testing.assert_array_equal(fq(-x, fmt).view(np.uint32), (-q1).view(np.uint32))  # odd
    xs = np.sort(x)
    assert np.all(np.diff(fq(xs, fmt).astype(np.float64)) >= 0)                        # monotone
    # NaN -> +max_finite (c6); E8M23 passes NaN through
    nan = fq([np.nan], fmt)[0]
    if fmt == (8, 23):
        assert np.isnan(nan)
    else:
        assert nan == fq([np.float32(3e38)], fmt)[0] or nan == fq([np.inf], fmt)[0]
    # -0 keeps its sign (c8)
    assert np.signbit(fq([-0.0], fmt)[0])


def test_e8m23_identity_all_patterns_sampled():
    bits = codec_sweep_inputs(1 << 20, "bits", 11).view(np.uint32)
    bits = np.concatenate([bits, edge_values().view(np.uint32)])
    codes = codec.quantize(bits.view(np.float32), 8, 23)
    np.testing.assert_array_equal(codes, bits)


@pytest.mark.parametrize("fmt", ALL_FORMATS)
def test_quantize_f64_matches_f32_path(fmt):
    x = _inputs(20000, key=13)
    a = codec.quantize_f64(x.astype(np.float64), *fmt)
    if fmt == (8, 23):
        np.testing.assert_array_equal(a, x.view(np.uint32))
    else:
        np.testing.assert_array_equal(a, codec.quantize(x, *fmt))


def _between_fp32_doubles(E, M, key):
    """Doubles that are NOT FP32 values: each format midpoint (the RNE tie)
    nudged by +-2^-40 relative, and random doubles -- the inputs on which a
    double -> FP32 -> ExMy double rounding would differ from one rounding."""
    mags = codec.representable_magnitudes(E, M)
    mids = (mags[:-1] + mags[1:]) / 2
    rng = np.random.default_rng(key)
    rnd = rng.uniform(-1.0, 1.0, 20000) * 2.0 ** rng.integers(-30, 20, 20000)
    x = np.concatenate([mids * (1 + 2.0 ** -40), mids * (1 - 2.0 ** -40), rnd])
    x = x[np.isfinite(x)]
    x = x[x.astype(np.float32).astype(np.float64) != x]
    return np.concatenate([x, -x])


@pytest.mark.parametrize("fmt", [f for f in ALL_FORMATS if 1 + f[0] + f[1] <= 16])
def test_quantize_f64_single_rounding_vs_enumeration(fmt):
    """quantize_f64 pinned on non-FP32 doubles by the independent enumeration
    oracle (nearest magnitude, ties to the even code) -- a double rounding
    (double -> FP32 -> ExMy) fails at the nudged midpoints."""
    x = _between_fp32_doubles(*fmt, key=17)
    np.testing.assert_array_equal(codec.quantize_f64(x, *fmt), codec.quantize_enum_f64(x, *fmt))


def test_quantize_f64_vs_numpy_float16_and_float32():
    """numpy's float64 -> float16 and float64 -> float32 conversions round once
    (RNE) from the double: E5M10 below 65520 and E8M23 on finite values."""
    x = _between_fp32_doubles(5, 10, key=19)
    x = x[np.abs(x) < 65520.0]
    np.testing.assert_array_equal(codec.quantize_f64(x, 5, 10),
                                  x.astype(np.float16).view(np.uint16).astype(np.uint32))
    y = _between_fp32_doubles(8, 7, key=23)
    np.testing.assert_array_equal(codec.quantize_f64(y, 8, 23), y.astype(np.float32).view(np.uint32))


def test_quantize_f64_double_rounding_traps():
    """Hand-worked (reading c4, one rounding): 1 + 2^-4 + 2^-30 lies just above
    the E4M3 tie between 1 (code 0x38) and 1.125 (0x39), so it rounds up to
    0x39, whereas via FP32 it would first become the tie 1.0625 and then round
    to the even 1.0.  Likewise 1 + 2^-11 + 2^-40 -> E5M10 1 + 2^-10 (0x3C01),
    and 2.5 + 2^-30 -> E2M1 3.0 (0x5) instead of the tie's even 2.0 (0x4)."""
    assert codec.quantize_f64(np.array([1 + 2.0 ** -4 + 2.0 ** -30]), 4, 3)[0] == 0x39
    assert codec.quantize_f64(np.array([1 + 2.0 ** -4 - 2.0 ** -30]), 4, 3)[0] == 0x38
    assert codec.quantize_f64(np.array([1 + 2.0 ** -11 + 2.0 ** -40]), 5, 10)[0] == 0x3C01
    assert codec.quantize_f64(np.array([2.5 + 2.0 ** -30]), 2, 1)[0] == 0x5
    assert codec.quantize_f64(np.array([2.5]), 2, 1)[0] == 0x4


def test_pack_layout_hand_built():
    # E2M1: eight 4-bit codes per word, LSB first ("eight FP4")
    w = codec.pack(np.array([[1, 2, 3, 4, 5, 6, 7, 0]], np.uint32), 2, 1)
    assert w.shape == (1, 4) and w[0, 0] == 0x07654321 and not w[0, 1:].any()
    # E3M6 (t=10): three codes per word, top 2 bits zero ("three FP10")
    w = codec.pack(np.array([[0x3FF, 0x001, 0x2AA, 0x155]], np.uint32), 3, 6)
    assert w[0, 0] == (0x3FF | (0x001 << 10) | (0x2AA << 20)) and w[0, 1] == 0x155
    # E5M10: two per word
    w = codec.pack(np.array([[0xABCD, 0x1234, 0xFFFF]], np.uint32), 5, 10)
    assert w[0, 0] == 0x1234ABCD and w[0, 1] == 0xFFFF
    # E2M2 (t=5, pf=6): 156 columns -> 26 words -> padded to 28
    assert codec.row_words(2, 2, 156) == 28
    assert [codec.row_words(*f, 156) for f in [(2, 1), (3, 2), (4, 3), (3, 6), (5, 10), (8, 23)]] == \
        [20, 32, 40, 52, 80, 156]


def test_pack_unpack_round_trip():
    rng = np.random.default_rng(0)
    for (E, M) in ALL_FORMATS:
        t = 1 + E + M
        codes = rng.integers(0, 2 ** t, (7, 157), dtype=np.uint64).astype(np.uint32)
        np.testing.assert_array_equal(codec.unpack(codec.pack(codes, E, M), E, M, 157), codes)


def test_data_movement_model():
    # 1024 x FP4 -> 512 B; 300 x FP10 -> 400 B (4 n / pf)
    assert 1024 * 4 // codec.packing_factor(2, 1) == 512
    assert 300 * 4 // codec.packing_factor(3, 6) == 400
    assert [codec.packing_factor(*f) for f in [(8, 23), (5, 10), (3, 6), (4, 3), (3, 2), (3, 1), (2, 1)]] \
        == [1, 2, 3, 4, 5, 6, 8]
