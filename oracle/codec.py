"""ExMy codec oracle: two independent references plus the packed layout.

TEST INFRASTRUCTURE ONLY -- see oracle/__init__.py.

* `quantize` / `dequantize`: the exact formula, in C double
  (oracle/codec.c; SURVEY.md §8(c) step 1 "Formula").
* `quantize_enum`: a second, independent reference by enumeration -- list all
  2^(t-1) magnitudes of the format from the definition of an ExMy value
  (bias 2^(E-1)-1, subnormals, no inf/NaN codes) and pick the
  nearest, ties to the code whose mantissa LSB is 0 (SURVEY.md §8(c) step 1
  "Enumeration").  Used for t <= 16.
* `pack` / `unpack`: floor(32/t) codes per little-endian 32-bit word,
  LSB-first, unused high bits zero, rows padded to a multiple of 4 words
  ("A 32-bit GPU register can store one FP32, two FP16, three
  FP10, four FP8, five FP6, six FP5, or eight FP4"; reading c10).
"""
import ctypes
import os
import subprocess

import numpy as np

_HERE = os.path.dirname(os.path.abspath(__file__))
_SO = os.path.join(_HERE, "liboracle_codec.so")
_lib = None


def build(force=False):
    """Compile oracle/codec.c with gcc (plain C, no CUDA)."""
    src = os.path.join(_HERE, "codec.c")
    if force or not os.path.exists(_SO) or os.path.getmtime(_SO) < os.path.getmtime(src):
        subprocess.check_call(["gcc", "-O2", "-fPIC", "-shared", "-std=c11",
                               "-fno-fast-math", "-ffp-contract=off",
                               "-o", _SO, src, "-lm", "-lpthread"])
    return _SO


def _load():
    global _lib
    if _lib is None:
        build()
        lib = ctypes.CDLL(_SO)
        P = ctypes.c_void_p
        lib.oracle_quantize.argtypes = [P, ctypes.c_size_t, ctypes.c_int, ctypes.c_int, P]
        lib.oracle_dequantize.argtypes = [P, ctypes.c_size_t, ctypes.c_int, ctypes.c_int, P]
        lib.oracle_quantize_mt.argtypes = [P, ctypes.c_size_t, ctypes.c_int, ctypes.c_int, P, ctypes.c_int]
        lib.oracle_quantize_bits_range.argtypes = [ctypes.c_uint32, ctypes.c_size_t, ctypes.c_int,
                                                   ctypes.c_int, P, ctypes.c_int]
        lib.oracle_quantize_f64.argtypes = [P, ctypes.c_size_t, ctypes.c_int, ctypes.c_int, P]
        lib.oracle_quantize_code.argtypes = [ctypes.c_float, ctypes.c_int, ctypes.c_int]
        lib.oracle_quantize_code.restype = ctypes.c_uint32
        _lib = lib
    return _lib


def total_bits(E, M):
    return 1 + E + M


def packing_factor(E, M):
    """Codes per 32-bit word: floor(32 / t)."""
    return 32 // total_bits(E, M)


def row_words(E, M, cols):
    """Words per packed row: ceil(cols / pf) rounded up to a multiple of 4
    (16-byte rows, reading c10)."""
    pf = packing_factor(E, M)
    w = -(-cols // pf)
    return -(-w // 4) * 4


def quantize(x, E, M, threads=1):
    """FP32 array -> uint32 codes (one code per element, unpacked)."""
    x = np.ascontiguousarray(x, dtype=np.float32)
    out = np.empty(x.shape, np.uint32)
    lib = _load()
    if threads > 1:
        lib.oracle_quantize_mt(x.ctypes.data, x.size, E, M, out.ctypes.data, threads)
    else:
        lib.oracle_quantize(x.ctypes.data, x.size, E, M, out.ctypes.data)
    return out


def quantize_f64(x, E, M):
    """float64 array -> codes with ONE rounding from the double value."""
    x = np.ascontiguousarray(x, dtype=np.float64)
    out = np.empty(x.shape, np.uint32)
    _load().oracle_quantize_f64(x.ctypes.data, x.size, E, M, out.ctypes.data)
    return out


def quantize_bits_range(base, n, E, M, threads=8):
    """codes[i] = quantize(float_from_bits(base + i)) for i < n."""
    out = np.empty(n, np.uint32)
    _load().oracle_quantize_bits_range(base, n, E, M, out.ctypes.data, threads)
    return out


def dequantize(codes, E, M):
    c = np.ascontiguousarray(codes, dtype=np.uint32)
    out = np.empty(c.shape, np.float32)
    _load().oracle_dequantize(c.ctypes.data, c.size, E, M, out.ctypes.data)
    return out


def fake_quant(x, E, M):
    """dequant(quant(x)): the paper's error-injection operator."""
    return dequantize(quantize(x, E, M), E, M)


# ---------------------------------------------------------------- enumeration
def representable_magnitudes(E, M):
    """All 2^(t-1) non-negative magnitudes, indexed by code, in float64.

    value(e, m) = m 2^(1-bias-M) for e = 0, (1 + m 2^-M) 2^(e-bias) else
    (PAPER.md:221 with readings c1-c3, c7)."""
    bias = 2 ** (E - 1) - 1
    e = np.repeat(np.arange(2 ** E, dtype=np.float64), 2 ** M)
    m = np.tile(np.arange(2 ** M, dtype=np.float64), 2 ** E)
    v = np.where(e == 0, m * 2.0 ** (1 - bias - M),
                 (1.0 + m / 2.0 ** M) * 2.0 ** (e - bias))
    if E == 8:          # exponent field 255 is never produced (c7)
        v = v[: 255 * 2 ** M]
    return v


def quantize_enum(x, E, M):
    """Nearest representable magnitude, ties to the even code (t <= 16)."""
    return _enum_nearest(np.asarray(x, np.float32), E, M)


def quantize_enum_f64(x, E, M):
    """The enumeration oracle on DOUBLE inputs (one rounding from the double
    value): the independent pin of `quantize_f64` for values between FP32
    numbers.  Near a tie the distances a - mags[lo] and mags[hi] - a are
    exact in double (adjacent magnitudes lie within a factor 2, Sterbenz)."""
    return _enum_nearest(np.asarray(x, np.float64), E, M)


def _enum_nearest(x, E, M):
    t = total_bits(E, M)
    assert t <= 16, "enumeration oracle is for t <= 16"
    mags = representable_magnitudes(E, M)
    a = np.abs(x.astype(np.float64))
    sign = np.signbit(x).astype(np.uint32) << np.uint32(t - 1)
    top = len(mags) - 1
    hi = np.searchsorted(mags, a, side="left")          # mags[hi] >= a
    hi = np.minimum(hi, top)
    lo = np.maximum(hi - 1, 0)
    dlo = a - mags[lo]
    dhi = mags[hi] - a
    pick_hi = (dhi < dlo) | ((dhi == dlo) & (hi % 2 == 0))
    idx = np.where(a >= mags[top], top, np.where(pick_hi, hi, lo))
    idx = np.where(a <= 0.0, 0, idx)
    code = idx.astype(np.uint32) | sign
    code = np.where(np.isnan(x), np.uint32(top), code)          # c6
    return code.astype(np.uint32)


# ---------------------------------------------------------------- packing
def pack(codes, E, M):
    """codes [rows, cols] uint32 -> words [rows, row_words] uint32."""
    codes = np.asarray(codes, np.uint32)
    if codes.ndim == 1:
        codes = codes[None, :]
    rows, cols = codes.shape
    t = total_bits(E, M)
    pf = packing_factor(E, M)
    W = row_words(E, M, cols)
    padded = np.zeros((rows, W * pf), np.uint64)
    padded[:, :cols] = codes
    padded = padded.reshape(rows, W, pf)
    shifts = (np.arange(pf, dtype=np.uint64) * np.uint64(t))
    words = np.zeros((rows, W), np.uint64)
    for j in range(pf):
        words |= padded[:, :, j] << shifts[j]
    return (words & np.uint64(0xFFFFFFFF)).astype(np.uint32)


def unpack(words, E, M, cols):
    """words [rows, row_words] -> codes [rows, cols]."""
    words = np.asarray(words, np.uint32)
    if words.ndim == 1:
        words = words[None, :]
    rows, W = words.shape
    t = total_bits(E, M)
    pf = packing_factor(E, M)
    mask = np.uint64((1 << t) - 1) if t < 32 else np.uint64(0xFFFFFFFF)
    w = words.astype(np.uint64)
    out = np.zeros((rows, W, pf), np.uint64)
    for j in range(pf):
        out[:, :, j] = (w >> np.uint64(j * t)) & mask
    return out.reshape(rows, W * pf)[:, :cols].astype(np.uint32)


def quantize_packed(x, E, M):
    """[rows, cols] FP32 -> packed words (oracle of vapr_quantize)."""
    x = np.asarray(x, np.float32)
    if x.ndim == 1:
        x = x[None, :]
    return pack(quantize(x, E, M), E, M)


def dequantize_packed(words, E, M, cols):
    """packed words -> [rows, cols] FP32 (oracle of vapr_dequantize)."""
    return dequantize(unpack(words, E, M, cols), E, M)


# ----------------------------------------------------------------- IEEE mode
# VAPR_FMT_IEEE (N4; "__floats2half2_rn"): E5M10 / E8M7 with the
# IEEE special values -- round to nearest even, overflow to +-inf, NaN kept.
# The definitions are the library conversions themselves: numpy float16 for
# E5M10 and torch bfloat16 (CPU) for E8M7.
FMT_IEEE = 0x100


def quantize_ieee(x, E, M):
    """float32 array -> IEEE binary16 / bfloat16 codes (uint32)."""
    x = np.asarray(x, np.float32)
    if (E, M) == (5, 10):
        return x.astype(np.float16).view(np.uint16).astype(np.uint32)
    if (E, M) == (8, 7):
        import torch
        t = torch.from_numpy(np.ascontiguousarray(x)).to(torch.bfloat16)
        return t.view(torch.int16).numpy().view(np.uint16).astype(np.uint32)
    raise ValueError("IEEE mode is defined for E5M10 and E8M7 only")


def dequantize_ieee(codes, E, M):
    c = np.asarray(codes, np.uint32).astype(np.uint16)
    if (E, M) == (5, 10):
        return c.view(np.float16).astype(np.float32)
    if (E, M) == (8, 7):
        return (c.astype(np.uint32) << 16).view(np.float32)
    raise ValueError("IEEE mode is defined for E5M10 and E8M7 only")
