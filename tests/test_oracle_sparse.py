"""Pins of oracle/sparse.py (reading c42): hand-worked
rows, the full-mask case against the dense packing of oracle/codec.py (an
independent implementation of the same LSB-first layout), invariants and
the round trip on random sparse code matrices of every packing factor."""
import numpy as np
import pytest

from oracle import codec
from oracle import sparse as sp

FORMATS = [(2, 1), (2, 2), (3, 2), (2, 3), (4, 3), (3, 4), (5, 10), (4, 9), (8, 7), (8, 23),
           (6, 9), (5, 4)]


def test_hand_example_e2m1():
    """E2M1: t = 4, pf = 8.  Three spheres: sphere 0 all zero, sphere 1
    (1, 0, 0xF), sphere 2 (0, 8, 0) -- code 8 is -0 (sign bit only) and
    counts as non-zero.  mask = 0b110; the six codes 1,0,F,0,8,0 packed
    LSB-first in 4-bit slots: 0x00080F01."""
    codes = np.array([[0, 0, 0, 1, 0, 0xF, 0, 8, 0]], np.uint32)
    m, rows = sp.sparsify(codes, 2, 1)
    assert int(m[0]) == 0b110
    assert rows[0].tolist() == [0x00080F01]
    assert sp.row_words(m[0], 2, 1) == 1


def test_hand_example_e4m3_two_words():
    """E4M3: t = 8, pf = 4.  Spheres 1 and 3 of four non-zero: six codes
    0x11, 0x22, 0x33, 0x44, 0x00, 0x66 -> words 0x44332211, 0x00006600."""
    codes = np.zeros((1, 12), np.uint32)
    codes[0, 3:6] = [0x11, 0x22, 0x33]
    codes[0, 9:12] = [0x44, 0x00, 0x66]
    m, rows = sp.sparsify(codes, 4, 3)
    assert int(m[0]) == 0b1010
    assert rows[0].tolist() == [0x44332211, 0x00006600]


def test_empty_rows():
    codes = np.zeros((3, 156), np.uint32)
    m, rows = sp.sparsify(codes, 3, 2)
    assert np.all(m == 0) and all(len(r) == 0 for r in rows)
    assert sp.sparse_bytes(m, 3, 2) == 36


@pytest.mark.parametrize("E,M", FORMATS)
def test_full_mask_equals_dense_packing(E, M):
    """Every sphere non-zero: the sparse row is the dense row (codec.pack)
    without the padding to four words."""
    rng = np.random.default_rng(E * 31 + M)
    t = 1 + E + M
    codes = rng.integers(1, 1 << min(t, 31), size=(4, 156), dtype=np.uint64).astype(np.uint32)
    m, rows = sp.sparsify(codes, E, M)
    dense = codec.pack(codes, E, M)
    n = -(-156 // sp.packing_factor(E, M))
    for p in range(4):
        assert int(m[p]) == (1 << 52) - 1
        assert np.array_equal(rows[p], dense[p, :n])


@pytest.mark.parametrize("E,M", FORMATS)
def test_roundtrip_and_invariants(E, M):
    rng = np.random.default_rng(100 + E * 31 + M)
    t = 1 + E + M
    P, S = 40, 52
    codes = rng.integers(0, 1 << min(t, 31), size=(P, 3 * S), dtype=np.uint64).astype(np.uint32)
    # ~5 % of the spheres non-zero, some rows empty, one row full
    keep = rng.random((P, S)) < 0.05
    keep[0] = False
    keep[1] = True
    codes = codes * np.repeat(keep, 3, axis=1)
    m, rows = sp.sparsify(codes, E, M)
    nz = np.any(codes.reshape(P, S, 3) != 0, axis=2)
    for p in range(P):
        assert bin(int(m[p])).count("1") == int(nz[p].sum())
        assert len(rows[p]) == -(-3 * int(nz[p].sum()) // sp.packing_factor(E, M))
    assert np.array_equal(sp.densify(m, rows, E, M, 3 * S), codes)
    assert sp.sparse_bytes(m, E, M) == 12 * P + 4 * sum(len(r) for r in rows)
