"""Pins for the format-space arithmetic."""
from oracle.formats import enumerate_formats, formats_at_or_above, space_size, total_bits
from workloads.configs import FORMAT_SETS
from workloads.scenes import ENVIRONMENTS


def test_21_formats():
    f = enumerate_formats()
    assert len(f) == 21
    widths = [1 + E + M for E, M in f]
    assert [widths.count(w) for w in (4, 5, 6, 8, 10, 16, 32)] == [1, 2, 3, 5, 7, 2, 1]


def test_counts_at_or_above():
    # SPEC.md:121
    want = {4: 21, 5: 20, 6: 18, 8: 15, 10: 10, 13: 3, 16: 3, 17: 1, 32: 1}
    assert {b: len(formats_at_or_above(b)) for b in want} == want
    assert formats_at_or_above(13) == [(5, 10), (8, 7), (8, 23)]


def test_search_space_sizes():
    assert space_size([4] * 5) == 4084101
    # table_pick: E6M6 (13), 4, FP5 out_vec, 4, 4 (Table II per-tensor rows)
    assert space_size([13, 4, 5, 4, 4]) == 555660
    assert space_size([16, 4, 4, 4, 5]) == 555660                  # table_under_pick
    assert round(4084101 / 555660, 2) == 7.35
    assert space_size([16, 4, 4, 4, 4]) == 583443                  # "by 7x"
    assert round(4084101 / 583443, 1) == 7.0


def test_table2_total_bits():
    # PAPER.md:305-312 rows; max 43 ("160 bits down to 43 bits or less")
    bits = {e: total_bits(FORMAT_SETS[e]) for e in ENVIRONMENTS}
    assert [bits[e] for e in ENVIRONMENTS] == [41, 34, 38, 38, 36, 38, 37, 43]
    assert total_bits(FORMAT_SETS["fp32"]) == 160
    # per-slot maxima quoted in the appendix: 16, 8, 6, 8, 8
    for slot, m in enumerate((16, 8, 6, 8, 8)):
        assert max(1 + FORMAT_SETS[e][slot][0] + FORMAT_SETS[e][slot][1] for e in ENVIRONMENTS) == m
