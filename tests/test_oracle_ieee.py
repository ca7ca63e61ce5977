"""Pins of the IEEE-mode oracle (oracle/codec.py quantize_ieee; N4): IEEE
binary16 / bfloat16 reference values, and agreement with the all-finite
reading wherever neither special values nor saturation are involved."""
import numpy as np

from oracle import codec


def test_binary16_reference_values():
    # 2^-25 is half the subnormal quantum (tie -> even 0), 3 * 2^-25 is 1.5
    # quanta (tie -> even 2), 3 * 2^-26 is 0.75 quanta (-> 1)
    x = np.array([0.0, -0.0, 1.0, 65504.0, 65519.0, 65520.0, 1e6, -1e6, 2.0 ** -24,
                  2.0 ** -25, 3 * 2.0 ** -25, 3 * 2.0 ** -26, np.inf, -np.inf], np.float32)
    ref = [0x0000, 0x8000, 0x3C00, 0x7BFF, 0x7BFF, 0x7C00, 0x7C00, 0xFC00, 0x0001,
           0x0000, 0x0002, 0x0001, 0x7C00, 0xFC00]
    assert codec.quantize_ieee(x, 5, 10).tolist() == ref
    c = codec.quantize_ieee(np.array([np.nan], np.float32), 5, 10)[0]
    assert (c & 0x7C00) == 0x7C00 and (c & 0x3FF) != 0          # a NaN
    d = codec.dequantize_ieee(np.array([0x7C00, 0xFC00, 0x7E00, 0x7BFF]), 5, 10)
    assert d[0] == np.inf and d[1] == -np.inf and np.isnan(d[2]) and d[3] == 65504.0


def test_bfloat16_reference_values():
    # 1 + 2^-8 is half a bf16 ulp above 1 (tie -> even 0x3F80); 1 + 3 * 2^-8 is
    # 1.5 ulp (tie -> even 0x3F82)
    x = np.array([1.0, -2.5, 3.3895313892515355e38, 3.4e38, np.inf, 1.0 + 2 ** -8,
                  1.0 + 3 * 2 ** -8], np.float32)
    ref = [0x3F80, 0xC020, 0x7F7F, 0x7F80, 0x7F80, 0x3F80, 0x3F82]
    assert codec.quantize_ieee(x, 8, 7).tolist() == ref
    assert np.isnan(codec.dequantize_ieee(np.array([0x7FC0]), 8, 7)[0])


def test_ieee_equals_all_finite_reading_in_range():
    rng = np.random.default_rng(0)
    x = (rng.normal(size=200000) * 10.0 ** rng.uniform(-8, 4.5, 200000)).astype(np.float32)
    x = x[np.abs(x) < 65504.0]
    assert np.array_equal(codec.quantize_ieee(x, 5, 10), codec.quantize(x, 5, 10))
    y = (rng.normal(size=200000) * 10.0 ** rng.uniform(-30, 30, 200000)).astype(np.float32)
    assert np.array_equal(codec.quantize_ieee(y, 8, 7), codec.quantize(y, 8, 7))
