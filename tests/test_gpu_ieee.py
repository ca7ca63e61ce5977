"""IEEE special-value mode (VAPR_FMT_IEEE): vapr_quantize
and vapr_dequantize against the library conversions (oracle/codec.py
quantize_ieee: numpy float16, torch bfloat16), and vapr_cost_grad with
IEEE E5M10 / E8M7 slots bit-identical to the all-finite formats on robot data
(they differ only at overflow and NaN)."""
import numpy as np
import pytest
import torch

from oracle import codec
from workloads.configs import codec_sweep_inputs, edge_values

pytestmark = pytest.mark.gpu
IEEE = codec.FMT_IEEE


@pytest.fixture(scope="module")
def vb():
    if not torch.cuda.is_available():
        pytest.skip("needs a GPU")
    from paper_2310_07854_b200 import binding
    return binding


def same_or_nan(a, b, nan_of):
    return (a == b) | (nan_of(a) & nan_of(b))


@pytest.mark.parametrize("E,M", [(5, 10), (8, 7)])
@pytest.mark.parametrize("cols", [157, 4])
def test_quantize_ieee(vb, E, M, cols):
    x = np.concatenate([edge_values(), codec_sweep_inputs(1 << 16, "bits", 3),
                        codec_sweep_inputs(1 << 16, "position", 4),
                        np.array([65504, 65519, 65520, 65536, 1e9, -1e9, 3.4e38, np.inf, -np.inf,
                                  np.nan], np.float32)]).astype(np.float32)
    rows = len(x) // cols
    x = x[: rows * cols].reshape(rows, cols)
    fmt = (E, M | IEEE)
    W = vb.vapr_packed_row_words(fmt, cols)
    out = torch.empty(rows * W, dtype=torch.int32, device="cuda")
    vb.vapr_quantize(fmt, torch.from_numpy(x).cuda(), rows, cols, out)
    words = out.cpu().numpy().view(np.uint32).reshape(rows, W)
    got = codec.unpack(words, E, M, cols)
    ref = codec.quantize_ieee(x, E, M)
    if E == 5:
        nan_of = lambda c: ((c & 0x7C00) == 0x7C00) & ((c & 0x3FF) != 0)
    else:
        nan_of = lambda c: ((c & 0x7F80) == 0x7F80) & ((c & 0x7F) != 0)
    assert np.all(same_or_nan(got.astype(np.uint32), ref, nan_of))


@pytest.mark.parametrize("E,M", [(5, 10), (8, 7)])
def test_dequantize_ieee_all_codes(vb, E, M):
    codes = np.arange(1 << 16, dtype=np.uint32)
    cols = 128
    rows = len(codes) // cols
    codes = codes.reshape(rows, cols)
    fmt = (E, M | IEEE)
    words = codec.pack(codes, E, M)
    y = torch.empty(rows * cols, dtype=torch.float32, device="cuda")
    vb.vapr_dequantize(fmt, torch.from_numpy(words.view(np.int32)).cuda(), rows, cols, y)
    got = y.cpu().numpy().reshape(rows, cols)
    ref = codec.dequantize_ieee(codes, E, M)
    assert np.all((got.view(np.uint32) == ref.view(np.uint32)) | (np.isnan(got) & np.isnan(ref)))


def test_cost_grad_ieee_equals_all_finite_on_robot_data(vb):
    from paper_2310_07854_b200.rollout import Rollout
    from workloads import config4
    wl = config4(problems_per_env=1, seeds=3, H=32, formats="fp16")
    a = Rollout(wl)
    a.run()
    ra = a.results()
    b = Rollout(wl, formats=((5, 10 | IEEE),) * 5)
    b.run()
    rb = b.results()
    for k in ("cost_traj", "grad_q"):
        assert np.array_equal(ra[k].view(np.uint32), rb[k].view(np.uint32)), k
    for slot in range(5):
        pa, pb = a.packed(slot), b.packed(slot)
        if pa is not None:
            assert np.array_equal(pa, pb), slot


def test_ieee_flag_validation(vb):
    with pytest.raises(vb.VaprError):
        vb._check(vb.lib.vapr_format_check(vb.vapr_format(4, 3 | IEEE)), "E4M3 has no IEEE mode")
    vb._check(vb.lib.vapr_format_check(vb.vapr_format(5, 10 | IEEE)), "E5M10 IEEE")
    vb._check(vb.lib.vapr_format_check(vb.vapr_format(8, 7 | IEEE)), "E8M7 IEEE")


def test_bk_ieee_gradient_overflow(vb):
    """The gradient slot (VAPR_GRAD_OUT_SPHERES) in IEEE E5M10 with a world
    weight large enough to overflow it: rows holding an exponent-31 (inf)
    code give a non-finite joint gradient for that pose (BK decodes them as
    inf, c41), every other pose matches the all-finite E5M10 run bit for bit
    (below the overflow threshold the two encodings agree)."""
    import dataclasses
    from paper_2310_07854_b200.rollout import Rollout
    from workloads import config4
    wl = config4(problems_per_env=1, seeds=8, H=32, formats="fp32")
    p = dict(wl.params)
    p.update(w_world=3e6)
    wl = dataclasses.replace(wl, params=p)
    fp32 = (8, 23)
    base = [fp32] * 5
    a_fmt, b_fmt = list(base), list(base)
    a_fmt[1] = (5, 10)
    b_fmt[1] = (5, 10 | IEEE)
    a = Rollout(wl, formats=tuple(a_fmt))
    a.run()
    ra = a.results()
    b = Rollout(wl, formats=tuple(b_fmt))
    b.run()
    rb = b.results()
    words = b.packed(1)
    cols = 3 * len(wl.robot["sphere_link"])
    codes = codec.unpack(words, 5, 10, cols)
    special = np.any((codes & 0x7C00) == 0x7C00, axis=1)
    assert special.any() and (~special).any()
    ga = ra["grad_q"].reshape(-1, 7)
    gb = rb["grad_q"].reshape(-1, 7)
    assert np.array_equal(ga[~special].view(np.uint32), gb[~special].view(np.uint32))
    assert np.all(np.any(~np.isfinite(gb[special]), axis=1))
    assert np.all(np.isfinite(ga))
