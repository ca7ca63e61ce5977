"""CPU checks of the C-ABI boundary: the library loads, exports every symbol
include/vapr.h declares, and its host-only helpers behave (no device work)."""
import ctypes
import os
import re

import pytest

from conftest import ROOT

HEADER = os.path.join(ROOT, "include", "vapr.h")


def declared_symbols():
    src = open(HEADER).read()
    src = re.sub(r"/\*.*?\*/", "", src, flags=re.S)
    # the test-only export of the tap build (libvapr_tap.so) is not in libvapr.so
    src = re.sub(r"#ifdef VAPR_DEBUG_TAP.*?#endif", "", src, flags=re.S)
    return sorted(set(re.findall(r"\b(vapr_[a-z_0-9]+)\s*\(", src)))


def test_library_exports_every_declared_symbol():
    from paper_2310_07854_b200 import binding as vb
    syms = declared_symbols()
    assert len(syms) >= 20
    for s in syms:
        assert hasattr(vb.lib, s), s
    assert sorted(vb.EXPORTS) == syms


def test_debug_tap_only_in_the_tap_build():
    """release builds omit vapr_debug_tap; the tap build
    (libvapr_tap.so) exports it and every release symbol."""
    from paper_2310_07854_b200 import binding as vb
    from paper_2310_07854_b200.build import TAP_SO
    assert not hasattr(vb.lib, "vapr_debug_tap")
    tap = ctypes.CDLL(TAP_SO)
    assert hasattr(tap, "vapr_debug_tap")
    for s in declared_symbols():
        assert hasattr(tap, s), s


def test_format_helpers():
    from paper_2310_07854_b200 import binding as vb
    assert vb.vapr_format_parse("E2M1") == (2, 1)
    assert vb.vapr_format_parse("e5m10") == (5, 10)
    for bad in ("E1M2", "E9M1", "E2M0", "E8M24", "X2M1", "E2M1x", ""):
        with pytest.raises(vb.VaprError):
            vb.vapr_format_parse(bad)
    assert vb.vapr_format_check((8, 23)) and not vb.vapr_format_check((5, 27))
    assert [vb.vapr_packed_row_words(f, 156) for f in [(2, 1), (2, 2), (3, 2), (4, 3), (3, 6), (5, 10), (8, 23)]] \
        == [20, 28, 32, 40, 52, 80, 156]
    assert vb.vapr_packed_row_words((2, 1), 1) == 4 and vb.vapr_packed_row_words((9, 1), 10) == 0


def test_no_gpu_create_fails_loudly():
    import torch
    from paper_2310_07854_b200 import binding as vb
    if torch.cuda.is_available():
        pytest.skip("GPU present")
    with pytest.raises(vb.VaprError):
        vb.vapr_create(0)


def test_library_is_sm100a():
    so = os.path.join(ROOT, "paper_2310_07854_b200", "libvapr.so")
    import subprocess
    out = subprocess.run(["/usr/local/cuda/bin/cuobjdump", "--list-elf", so],
                         capture_output=True, text=True).stdout
    assert "sm_100a" in out
