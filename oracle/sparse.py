"""oracle/sparse.py -- TEST INFRASTRUCTURE (see oracle/__init__.py).

Sparsity-aware storage of a packed sphere tensor.
PAPER.md:196: "grad_out_spheres, out_vec, closest_pt, and closest_pt_swept
have more than 99% of sparsity.  As a result, we adopt sparsity-aware
computation by skipping zero computations."  The paper gives no storage
format; the reading (c42) is a per-row sphere bitmap plus the
non-zero spheres' codes packed back to back:

  codes[p, 3s + c]  the dense row's codes (c = x, y, z of sphere s, S <= 64);
  mask[p]   = sum of 2^s over the spheres s whose three codes are not all 0
              (as t-bit integers: a -0 code counts as non-zero);
  row[p]    = codes[p, 3s : 3s + 3] for the set bits s of mask[p] in
              ascending order, concatenated (3 popc(mask[p]) codes);
  words[p]  = row[p] packed LSB-first, floor(32 / t) codes per 32-bit word
              (the dense rows' packing, PAPER.md:218 / reading c10), in
              ceil(3 popc / pf) words with the unused high slots 0 and no
              padding to 4 words.

The device layout adds off[p] (the row's first word in a shared pool); the
rows' order in the pool is the writer's choice, so parity compares words[p]
against pool[off[p] : off[p] + n_p] row by row.  Plain Python/numpy loops;
pinned by tests/test_oracle_sparse.py (hand examples, the full-mask case
against codec.pack, invariants).
"""
import numpy as np


def packing_factor(E, M):
    return 32 // (1 + E + M)


def sparsify(codes, E, M):
    """codes [P, cols] (cols = 3S) -> (mask uint64 [P], list of P uint32 word arrays)."""
    codes = np.asarray(codes, np.uint64)
    P, cols = codes.shape
    assert cols % 3 == 0 and cols // 3 <= 64
    S = cols // 3
    t = 1 + E + M
    pf = packing_factor(E, M)
    masks = np.zeros(P, np.uint64)
    rows = []
    for p in range(P):
        m = 0
        row = []
        for s in range(S):
            trip = [int(codes[p, 3 * s + c]) for c in range(3)]
            if any(v != 0 for v in trip):
                m |= 1 << s
                row.extend(trip)
        masks[p] = m
        n = (len(row) + pf - 1) // pf
        words = np.zeros(n, np.uint32)
        for i, v in enumerate(row):
            words[i // pf] |= np.uint32(v << ((i % pf) * t))
        rows.append(words)
    return masks, rows


def densify(masks, rows, E, M, cols):
    """Inverse of sparsify: (mask [P], rows) -> codes [P, cols] (uint32)."""
    t = 1 + E + M
    pf = packing_factor(E, M)
    cmask = (1 << t) - 1
    P = len(masks)
    out = np.zeros((P, cols), np.uint32)
    for p in range(P):
        m = int(masks[p])
        k = 0
        for s in range(cols // 3):
            if (m >> s) & 1:
                for c in range(3):
                    i = 3 * k + c
                    out[p, 3 * s + c] = (int(rows[p][i // pf]) >> ((i % pf) * t)) & cmask
                k += 1
    return out


def row_words(mask, E, M):
    """Words of a row with this mask: ceil(3 popc(mask) / pf)."""
    pf = packing_factor(E, M)
    return (3 * bin(int(mask)).count("1") + pf - 1) // pf


def sparse_bytes(masks, E, M):
    """Stored bytes of the sparse form: 8 (mask) + 4 (offset) per row plus the
    pool words in use."""
    return 12 * len(masks) + 4 * sum(row_words(m, E, M) for m in masks)
