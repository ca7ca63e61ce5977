"""The ExMy format space and the VaPr search-space arithmetic (oracle).

TEST INFRASTRUCTURE ONLY -- see oracle/__init__.py.

PAPER.md:218 ("FP4, FP5, FP6, FP8, FP10, FP16, and FP32")
("We consider 21 FP data types from FP4 to FP32, which gives the search space
21^5 = 4,084,101"), PAPER.md:249 (per-tensor minimum, "from 21 combinations to
3 combinations (i.e., E5M10, E8M7, and E8M23)"; "decreases by 7.35x, from
4,084,101 down to 555,660").  The rule that reproduces these counts
(SPEC.md:52-60): widths {4,5,6,8,10} take every E in [2,8] with M >= 1;
width 16 is exactly {E5M10, E8M7}; width 32 is exactly {E8M23}.
"""
WIDTHS = (4, 5, 6, 8, 10, 16, 32)


def enumerate_formats():
    out = []
    for t in WIDTHS:
        if t == 16:
            out += [(5, 10), (8, 7)]
        elif t == 32:
            out += [(8, 23)]
        else:
            for E in range(2, 9):
                M = t - 1 - E
                if M >= 1:
                    out.append((E, M))
    return out


def formats_at_or_above(min_bits):
    return [f for f in enumerate_formats() if 1 + f[0] + f[1] >= min_bits]


def space_size(min_bits_per_slot):
    n = 1
    for b in min_bits_per_slot:
        n *= len(formats_at_or_above(b))
    return n


def total_bits(fmts):
    return sum(1 + E + M for (E, M) in fmts)
