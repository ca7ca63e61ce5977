"""GPU <-> oracle parity through the C ABI (needs a B200)."""
import numpy as np
import pytest
import torch

from oracle import codec
from oracle import rollout as orc
from oracle.formats import enumerate_formats
from parity_utils import check_codes, check_close, cost_kw, e2e_kw, self_kw, sphere_to_elem, step_bound, world_kw
from workloads import config1, config2, config4, make_workload
from workloads.configs import FORMAT_SETS, codec_sweep_inputs, edge_values

pytestmark = pytest.mark.gpu

CANONICAL = enumerate_formats() + [(6, 6), (5, 9), (6, 8)]   # P:221 + Table II
# every format vapr_format_check accepts: E in [2,8], M in [1,23], t <= 32
# (PAPER.md:221 defines ExMy for any split) -- 161 formats
ALL_VALID = [(E, M) for E in range(2, 9) for M in range(1, 24) if 1 + E + M <= 32]
ALL_FORMATS = CANONICAL
# canonical formats at four ragged column counts, the rest of the 161 at one
CODEC_CASES = ([(f, c) for f in CANONICAL for c in (157, 156, 1, 4097)] +
               [(f, 157) for f in ALL_VALID if f not in CANONICAL])


@pytest.fixture(scope="module")
def vb():
    if not torch.cuda.is_available():
        pytest.skip("no GPU")
    from paper_2310_07854_b200 import binding
    return binding


def dev(a):
    return torch.from_numpy(np.ascontiguousarray(a)).cuda()


def dataclasses_replace(wl, **kw):
    import dataclasses
    return dataclasses.replace(wl, **kw)


def sampled_magnitudes(E, M, n=1 << 16, key=11):
    """Up to n representable magnitudes of the format, in code order, from the
    oracle's decoder: every one for t <= 17, else a seeded sample of codes
    plus the ends of every binade (so every exponent field is probed)."""
    t = 1 + E + M
    ncodes = 255 << M if E == 8 else 1 << (E + M)     # exponent 255 never produced (c7)
    if ncodes <= n:
        codes = np.arange(ncodes, dtype=np.uint64)
    else:
        rng = np.random.default_rng(key + 97 * E + M)
        nexp = ncodes >> M
        ends = np.concatenate([(np.arange(nexp, dtype=np.uint64) << np.uint64(M)),
                               (np.arange(nexp, dtype=np.uint64) << np.uint64(M)) + np.uint64((1 << M) - 1),
                               (np.arange(nexp, dtype=np.uint64) << np.uint64(M)) + np.uint64(1)])
        codes = np.unique(np.concatenate([rng.integers(0, ncodes, n, dtype=np.uint64), ends]))
        codes = codes[codes < ncodes]
    pairs = np.stack([codes, np.minimum(codes + 1, ncodes - 1)]).astype(np.uint32)
    v = codec.dequantize(pairs, E, M).astype(np.float64)
    return v[0], v[1]


def codec_inputs(fmt, n=1 << 16):
    """Random FP32 patterns, tensor-shaped values, and for the format: sampled
    representable values, the midpoints between neighbours (the RNE ties) and
    the FP32 values on either side of each midpoint, and FP32 edge cases."""
    lo, hi = sampled_magnitudes(*fmt)
    mids = ((lo + hi) / 2).astype(np.float32)      # exact for M <= 22; M = 23 rounds
    x = np.concatenate([codec_sweep_inputs(n, "bits", 1), codec_sweep_inputs(n, "position", 2),
                        codec_sweep_inputs(n, "gradient", 3), mids,
                        np.nextafter(mids, np.float32(np.inf)), np.nextafter(mids, np.float32(0)),
                        lo.astype(np.float32), edge_values()])
    return np.concatenate([x, -x])


# --------------------------------------------------------------------- a1
def test_codec_cases_cover_every_valid_format():
    assert len(ALL_VALID) == 161
    assert {f for f, _ in CODEC_CASES} == set(ALL_VALID)


@pytest.mark.parametrize("fmt,cols", CODEC_CASES, ids=lambda v: str(v))
def test_quantize_bit_exact(vb, fmt, cols):
    x = codec_inputs(fmt)
    rows = len(x) // cols
    x = x[: rows * cols].reshape(rows, cols)
    W = vb.vapr_packed_row_words(fmt, cols)
    out = torch.empty(rows * W, dtype=torch.int32, device="cuda")
    vb.vapr_quantize(fmt, dev(x), rows, cols, out)
    got = out.cpu().numpy().view(np.uint32).reshape(rows, W)
    np.testing.assert_array_equal(got, codec.quantize_packed(x, *fmt))


@pytest.mark.parametrize("fmt", ALL_VALID)
def test_dequantize_bit_exact(vb, fmt):
    E, M = fmt
    t = 1 + E + M
    if t <= 16:
        codes = np.arange(2 ** t, dtype=np.uint32)
    else:
        codes = codec_sweep_inputs(1 << 18, "bits", 7).view(np.uint32) & np.uint32((1 << t) - 1 if t < 32 else 0xFFFFFFFF)
    if E == 8 and M < 23:
        codes = codes[((codes >> M) & 0xFF) != 255]
    cols = 131
    rows = len(codes) // cols
    codes = codes[: rows * cols].reshape(rows, cols)
    words = codec.pack(codes, E, M)
    y = torch.empty(rows * cols, dtype=torch.float32, device="cuda")
    vb.vapr_dequantize(fmt, dev(words.view(np.int32)), rows, cols, y)
    got = y.cpu().numpy().reshape(rows, cols)
    ref = codec.dequantize(codes, E, M)
    same = (got.view(np.uint32) == ref.view(np.uint32)) | (np.isnan(got) & np.isnan(ref))
    assert same.all()


@pytest.mark.parametrize("fmt", [(E, 23) for E in range(2, 8)])
def test_quantize_m23_odd_mantissas(vb, fmt):
    """E<8, M=23 keeps all 23 FP32 mantissa bits: the code of a normal-range
    value is its FP32 pattern re-biased, odd mantissas included (round 1
    added the tie bit of an exact value and bumped every odd one)."""
    E, M = fmt
    bias = 2 ** (E - 1) - 1
    x = np.float32(2.0 ** (1 - bias)) * (1 + np.arange(1, 4001, dtype=np.float32) * np.float32(2 ** -23))
    out = torch.empty(vb.vapr_packed_row_words(fmt, len(x)), dtype=torch.int32, device="cuda")
    vb.vapr_quantize(fmt, dev(x[None, :]), 1, len(x), out)
    got = codec.unpack(out.cpu().numpy().view(np.uint32)[None, :], E, M, len(x))[0]
    want = (1 << 23) + np.arange(1, 4001, dtype=np.uint32)      # exponent field 1, mantissa k
    np.testing.assert_array_equal(got, want)


def test_codec_empty_and_errors(vb):
    x = torch.zeros(16, device="cuda")
    out = torch.zeros(16, dtype=torch.int32, device="cuda")
    vb.vapr_quantize((2, 1), x, 0, 16, out)          # empty: no-op
    with pytest.raises(vb.VaprError):
        vb.vapr_quantize((9, 1), x, 1, 16, out)
    with pytest.raises(vb.VaprError):
        vb.vapr_quantize((2, 1), x[1:], 1, 8, out)    # misaligned


@pytest.mark.slow
@pytest.mark.parametrize("fmt", ALL_VALID)
def test_quantize_exhaustive_all_fp32(vb, fmt):
    """All 2^32 FP32 bit patterns (SURVEY.md §4 codec tier).  Long: runs only
    with VAPR_EXHAUSTIVE=1 (a dedicated GPU call), not in the default suite."""
    import os
    if os.environ.get("VAPR_EXHAUSTIVE") != "1":
        pytest.skip("set VAPR_EXHAUSTIVE=1")
    E, M = fmt
    t = 1 + E + M
    pf = 32 // t
    chunk = 1 << 26
    cols = chunk
    W = vb.vapr_packed_row_words(fmt, cols)
    out = torch.empty(W, dtype=torch.int32, device="cuda")
    base_bits = torch.arange(chunk, dtype=torch.int64, device="cuda")
    threads = os.cpu_count() or 8
    shifts = torch.arange(pf, device="cuda", dtype=torch.int64) * t
    mask = (1 << t) - 1 if t < 32 else 0xFFFFFFFF
    for base in range(0, 1 << 32, chunk):
        x = ((base_bits + base) & 0xFFFFFFFF).to(torch.int64)
        xi = torch.where(x >= 2 ** 31, x - 2 ** 32, x).to(torch.int32)
        vb.vapr_quantize(fmt, xi.view(torch.float32), 1, cols, out)
        w = out.to(torch.int64) & 0xFFFFFFFF
        codes = ((w[:, None] >> shifts[None, :]) & mask).reshape(-1)[:chunk]
        ref = torch.from_numpy(codec.quantize_bits_range(base, chunk, E, M, threads).view(np.int32)).cuda()
        ref = ref.to(torch.int64) & 0xFFFFFFFF
        assert torch.equal(codes, ref), (fmt, hex(base))


# --------------------------------------------------------------------- helpers
class Ctx:
    def __init__(self, vb, wl, formats=None):
        self.vb = vb
        self.wl = wl
        self.h = vb.vapr_create(0)
        vb.vapr_set_robot(self.h, wl.robot)
        vb.vapr_set_worlds(self.h, wl.cuboids, wl.world_offsets)
        self.formats = tuple(formats or wl.formats)
        vb.vapr_set_formats(self.h, self.formats)

    def __del__(self):
        self.vb.vapr_destroy(self.h)

    def W(self, slot):
        return self.vb.vapr_packed_row_words(self.formats[slot], 156)


def ragged_workload(B=3, H=5, formats="43bit", salt=9):
    from workloads.scenes import ENVIRONMENTS
    envs = [ENVIRONMENTS[i % 8] for i in range(B)]
    return make_workload("ragged", envs, list(range(B)), 1, H, FORMAT_SETS[formats], salt=salt)


def _rot(rng):
    """Uniform random rotation (row-major 3x3) from a unit quaternion."""
    w, x, y, z = rng.normal(size=4) / 1.0
    n = np.sqrt(w * w + x * x + y * y + z * z)
    w, x, y, z = w / n, x / n, y / n, z / n
    return np.array([[1 - 2 * (y * y + z * z), 2 * (x * y - z * w), 2 * (x * z + y * w)],
                     [2 * (x * y + z * w), 1 - 2 * (x * x + z * z), 2 * (y * z - x * w)],
                     [2 * (x * z - y * w), 2 * (y * z + x * w), 1 - 2 * (x * x + y * y)]])


def edge_worlds_workload(formats="43bit", H=16, seeds=4):
    """Edge cases of the world tables: an empty world, a world at the
    16-cuboid maximum (rotated boxes all around the arm), and a world whose
    one large box engulfs the lower arm (sphere centres inside: the SDF's
    inside branch and the linear part of the hinge)."""
    rng = np.random.Generator(np.random.Philox(key=0xED6E))
    rows = []
    for k in range(16):
        r = np.zeros(16, np.float32)
        r[0:9] = _rot(rng).reshape(-1)
        ang = 2 * np.pi * k / 16
        rad = rng.uniform(0.25, 0.7)
        r[9:12] = (rad * np.cos(ang), rad * np.sin(ang), rng.uniform(0.05, 0.9))
        r[12:15] = rng.uniform(0.03, 0.15, 3)
        rows.append(r)
    big = np.zeros(16, np.float32)
    big[0:9] = np.eye(3).reshape(-1)
    big[9:12] = (0.0, 0.0, 0.35)
    big[12:15] = (0.25, 0.25, 0.35)
    rows.append(big)
    cub = np.stack(rows).astype(np.float32)
    off = np.array([0, 0, 16, 17], np.int32)
    return make_workload("edge_worlds", ["empty", "max16", "engulf"], [0, 1, 2], seeds, H,
                         FORMAT_SETS[formats], cuboids=cub, offsets=off, salt=21)


WORKLOADS = {
    "config1": lambda: config1(),
    "config1_fp32": lambda: config1(reduced=False),
    "config2": lambda: config2(),
    "ragged_43": lambda: ragged_workload(),
    "mixed_envs": lambda: config4(problems_per_env=1, seeds=3, H=32),
    "bookshelf_tall": lambda: config4(problems_per_env=1, seeds=2, H=32, formats="bookshelf_tall"),
    "fp16": lambda: config4(problems_per_env=1, seeds=2, H=32, formats="fp16"),
    "fp32": lambda: config4(problems_per_env=1, seeds=2, H=32, formats="fp32"),
    "pf5_pf8": lambda: config4(problems_per_env=1, seeds=2, H=32, formats="pf5_pf8"),
    "pf3": lambda: config4(problems_per_env=1, seeds=2, H=32, formats="pf3"),
    "bf16": lambda: config4(problems_per_env=1, seeds=2, H=32, formats="bf16"),
    "edge_worlds": lambda: edge_worlds_workload(),
    "edge_worlds_fp32": lambda: edge_worlds_workload(formats="fp32"),
    "h2_min_swept": lambda: ragged_workload(B=4, H=2, salt=23),
}


# --------------------------------------------------------------------- a2
@pytest.mark.parametrize("name", list(WORKLOADS))
def test_fk_spheres(vb, name):
    wl = WORKLOADS[name]()
    c = Ctx(vb, wl)
    P = wl.poses
    fos = c.formats[0]
    out = torch.empty(P * c.W(0), dtype=torch.int32, device="cuda")
    vb.vapr_fk_spheres(c.h, dev(wl.q), wl.B, wl.H, out)
    words, v = orc.fk_stage(wl.q.reshape(-1, 7), wl.robot, fos)
    got = out.cpu().numpy().view(np.uint32).reshape(P, -1)
    exact, _ = check_codes(got, v, 1.0, 0.0, fos, 156, what="out_spheres",
                           min_exact=0.999 if fos != (8, 23) else None)
    assert exact > 0.99 or fos == (8, 23)


@pytest.mark.parametrize("formats", ["43bit", "fp32", "pf3", "pf5_pf8"])
def test_fk_chunk_tails(vb, formats):
    """FK's per-warp chunk drains (fk.cu): 287 poses = two full 128-pose CTAs
    and a tail CTA whose one warp has 31 live lanes, with row widths that
    leave a partial last chunk (FP32: 156 words = 4 x 32 + 28).  Every row
    word, padding included, against the oracle; the buffer past the last
    pose stays untouched."""
    wl = ragged_workload(B=7, H=41, formats=formats, salt=31)
    c = Ctx(vb, wl)
    P, W = wl.poses, c.W(0)
    assert P == 287
    fos = c.formats[0]
    out = torch.full((P * W + 64,), 0x5A5A5A5A, dtype=torch.int32, device="cuda")
    vb.vapr_fk_spheres(c.h, dev(wl.q), wl.B, wl.H, out)
    words, v = orc.fk_stage(wl.q.reshape(-1, 7), wl.robot, fos)
    got = out[:P * W].cpu().numpy().view(np.uint32).reshape(P, -1)
    check_codes(got, v, 1.0, 0.0, fos, 156, what="out_spheres",
                min_exact=0.999 if fos != (8, 23) else None)
    # padding: the unused code slots of the last used word and every word after it are +0
    t = 1 + fos[0] + fos[1]
    pf = 32 // t
    used = -(-156 // pf)
    tail_bits = (156 - (used - 1) * pf) * t
    if tail_bits < 32:
        assert (got[:, used - 1] >> np.uint32(tail_bits) == 0).all()
    assert (got[:, used:] == 0).all()
    assert (out[P * W:].cpu().numpy() == 0x5A5A5A5A).all()


# --------------------------------------------------------------------- a3/a4
@pytest.mark.parametrize("name", list(WORKLOADS))
@pytest.mark.parametrize("swept", [1, 0])
def test_collision_stage(vb, name, swept):
    wl = WORKLOADS[name]()
    c = Ctx(vb, wl)
    P, B, H = wl.poses, wl.B, wl.H
    p = dict(wl.params, swept=swept)
    f = c.formats
    os_words, _ = orc.fk_stage(wl.q.reshape(-1, 7), wl.robot, f[0])
    slot = 4 if swept else 3
    cp = torch.empty(P * c.W(slot), dtype=torch.int32, device="cuda")
    ov = torch.empty(P * c.W(2), dtype=torch.int32, device="cuda")
    cost = torch.empty(P, dtype=torch.float32, device="cuda")
    ctraj = torch.empty(B, dtype=torch.float32, device="cuda")
    vb.vapr_collision(c.h, dev(os_words.view(np.int32)), dev(wl.world_idx), B, H, p, cost, ctraj, cp, ov)
    ws = orc.world_stage(os_words, f[0], wl.world_idx, wl.cuboids, wl.world_offsets, wl.robot,
                         B, H, p["eta_world"], p["w_world"], swept, p["sweep_steps"], f[slot])
    ss = orc.self_stage(os_words, f[0], wl.robot, p["eta_self"], p["w_self"], f[2])
    ref_cost = ws["cost"].reshape(-1) + ss["cost"]
    ck = cost_kw(ws, ss)
    check_close(cost.cpu().numpy(), ref_cost, what="cost_pose", **ck)
    check_close(ctraj.cpu().numpy(), ref_cost.reshape(B, H).sum(1), ck["terms"].reshape(B, H).sum(1),
                "cost_traj", kappa=ck["kappa"].reshape(B, H).sum(1))
    check_codes(cp.cpu().numpy().view(np.uint32).reshape(P, -1), ws["v"], fmt=f[slot], cols=156,
                what="closest_pt", min_exact=0.999, max_steps=step_bound(f[slot]), **world_kw(ws))
    check_codes(ov.cpu().numpy().view(np.uint32).reshape(P, -1), ss["v"], fmt=f[2], cols=156,
                what="out_vec", min_exact=0.999, max_steps=step_bound(f[2]), **self_kw(ss))


def test_world_and_self_separately(vb):
    wl = config2()
    c = Ctx(vb, wl)
    P, B, H = wl.poses, wl.B, wl.H
    f = c.formats
    p = wl.params
    os_words, _ = orc.fk_stage(wl.q.reshape(-1, 7), wl.robot, f[0])
    osd = dev(os_words.view(np.int32))
    cp = torch.empty(P * c.W(4), dtype=torch.int32, device="cuda")
    cost = torch.empty(P, dtype=torch.float32, device="cuda")
    vb.vapr_world_collision(c.h, osd, dev(wl.world_idx), B, H, 1, 1, p["eta_world"], p["w_world"], cost, cp)
    ws = orc.world_stage(os_words, f[0], wl.world_idx, wl.cuboids, wl.world_offsets, wl.robot,
                         B, H, p["eta_world"], p["w_world"], 1, 1, f[4])
    check_close(cost.cpu().numpy(), ws["cost"].reshape(-1), ws["cost_terms"].reshape(-1), "world cost",
                kappa=ws["cost_kappa"].reshape(-1))
    check_codes(cp.cpu().numpy().view(np.uint32).reshape(P, -1), ws["v"], fmt=f[4], cols=156,
                what="closest_pt_swept", max_steps=step_bound(f[4]), **world_kw(ws))
    ov = torch.empty(P * c.W(2), dtype=torch.int32, device="cuda")
    vb.vapr_self_collision(c.h, osd, B, H, p["eta_self"], p["w_self"], cost, ov)
    ss = orc.self_stage(os_words, f[0], wl.robot, p["eta_self"], p["w_self"], f[2])
    check_close(cost.cpu().numpy(), ss["cost"], ss["cost_terms"], "self cost", kappa=ss["cost_kappa"])
    check_codes(ov.cpu().numpy().view(np.uint32).reshape(P, -1), ss["v"], fmt=f[2], cols=156,
                what="out_vec", max_steps=step_bound(f[2]), **self_kw(ss))


# --------------------------------------------------------------------- a5
@pytest.mark.parametrize("fs", ["43bit", "bookshelf_tall", "cage", "fp32", "table_pick"])
def test_aggregate(vb, fs):
    wl = config4(problems_per_env=1, seeds=2, H=32, formats=fs)
    c = Ctx(vb, wl)
    P = wl.poses
    f = c.formats
    res = orc.rollout_workload(wl)
    gos = torch.empty(P * c.W(1), dtype=torch.int32, device="cuda")
    vb.vapr_aggregate(c.h, dev(res.cp_words.view(np.int32)), 1, dev(res.ov_words.view(np.int32)), P, gos)
    ag = res.stages["aggregate"]
    # FP32 sum then one rounding: the only allowed differences are at midpoints
    # within 2^-24 (|a| + |b|) of v
    check_codes(gos.cpu().numpy().view(np.uint32).reshape(P, -1), ag["v"], ag["terms"], 0.0, f[1], 156,
                what="grad_out_spheres", min_exact=0.999, max_steps=step_bound(f[1]))


# --------------------------------------------------------------------- a6
@pytest.mark.parametrize("name", ["config2", "ragged_43", "mixed_envs", "fp32"])
def test_backward_kinematics(vb, name):
    wl = WORKLOADS[name]()
    c = Ctx(vb, wl)
    P = wl.poses
    res = orc.rollout_workload(wl)
    gq = torch.empty(P * 7, dtype=torch.float32, device="cuda")
    vb.vapr_backward_kinematics(c.h, dev(wl.q), wl.B, wl.H, dev(res.gos_words.view(np.int32)), gq)
    bk = res.stages["bk"]
    check_close(gq.cpu().numpy().reshape(P, 7), bk["grad_q"], bk["scale"], "grad_q")


# --------------------------------------------------------------------- a7
@pytest.mark.parametrize("name", list(WORKLOADS))
def test_cost_grad_stagewise(vb, name):
    """Run the composed path; check each stage against the oracle fed with the
    GPU's own upstream packed tensor (read back from the workspace)."""
    from paper_2310_07854_b200.rollout import Rollout
    wl = WORKLOADS[name]()
    r = Rollout(wl)
    r.run()
    out = r.results()
    f = r.ctx.formats
    p = wl.params
    B, H, P = wl.B, wl.H, wl.poses
    slot = 4 if p["swept"] else 3
    os_w, cp_w, ov_w, gos_w = r.packed(0), r.packed(slot), r.packed(2), r.packed(1)
    _, v = orc.fk_stage(wl.q.reshape(-1, 7), wl.robot, f[0])
    check_codes(os_w, v, 1.0, 0.0, f[0], 156, what="out_spheres")
    ws = orc.world_stage(os_w, f[0], wl.world_idx, wl.cuboids, wl.world_offsets, wl.robot, B, H,
                         p["eta_world"], p["w_world"], p["swept"], p["sweep_steps"], f[slot])
    ss = orc.self_stage(os_w, f[0], wl.robot, p["eta_self"], p["w_self"], f[2])
    check_codes(cp_w, ws["v"], fmt=f[slot], cols=156, what="closest_pt_swept",
                max_steps=step_bound(f[slot]), **world_kw(ws))
    check_codes(ov_w, ss["v"], fmt=f[2], cols=156, what="out_vec", max_steps=step_bound(f[2]), **self_kw(ss))
    ref_cost = (ws["cost"].reshape(-1) + ss["cost"]).reshape(B, H)
    ck = cost_kw(ws, ss)
    check_close(out["cost_pose"], ref_cost, ck["terms"].reshape(B, H), "cost_pose",
                kappa=ck["kappa"].reshape(B, H))
    check_close(out["cost_traj"], ref_cost.sum(1), ck["terms"].reshape(B, H).sum(1), "cost_traj",
                kappa=ck["kappa"].reshape(B, H).sum(1))
    ag = orc.aggregate_stage(cp_w, f[slot], ov_w, f[2], f[1], 156)
    check_codes(gos_w, ag["v"], ag["terms"], 0.0, f[1], 156, what="grad_out_spheres",
                max_steps=step_bound(f[1]))
    bk = orc.bk_stage(wl.q.reshape(-1, 7), gos_w, f[1], wl.robot)
    check_close(out["grad_q"].reshape(P, 7), bk["grad_q"], bk["scale"], "grad_q")


def test_cost_grad_fp32_end_to_end(vb):
    """All-E8M23: the composed GPU result agrees with the oracle rollout
    directly (no stage re-feeding), within the norm-relative tolerance."""
    from paper_2310_07854_b200.rollout import Rollout
    wl = config4(problems_per_env=1, seeds=2, H=32, formats="fp32")
    r = Rollout(wl)
    r.run()
    out = r.results()
    res = orc.rollout_workload(wl)
    kw = e2e_kw(res, wl)
    r1 = check_close(out["cost_traj"], res.cost_traj, what="cost_traj", **kw["cost_traj"])
    r2 = check_close(out["grad_q"].reshape(-1, 7), res.grad_q.reshape(-1, 7), what="grad_q", **kw["grad_q"])
    print(f"fp32 end-to-end: max err/limit cost_traj {r1:.3g}, grad_q {r2:.3g}")


@pytest.mark.parametrize("n_chunks,pinned", [(1, True), (5, True), (0, True), (7, False)])
def test_cost_grad_host_matches_device_path(vb, n_chunks, pinned):
    """vapr_cost_grad_host (pipelined host copies, trajectory chunks) gives
    bit-identical grad_q / cost_traj / cost_pose to vapr_cost_grad, for
    ragged chunkings and pageable host memory; the workspace tensors too."""
    from paper_2310_07854_b200.rollout import Rollout
    wl = config4(problems_per_env=1, seeds=3, H=32)          # B = 24: ragged chunks
    r = Rollout(wl)
    r.run()
    ref = r.results()
    ref_ws = r.workspace.clone()
    r.grad_q.zero_()
    r.cost_traj.zero_()
    r.cost_pose.zero_()
    r.q.zero_()                                  # the host path must upload q itself
    q_host = torch.from_numpy(np.ascontiguousarray(wl.q, np.float32))
    gq_host = torch.full((wl.B * wl.H * 7,), float("nan"), dtype=torch.float32)
    ct_host = torch.full((wl.B,), float("nan"), dtype=torch.float32)
    if pinned:
        q_host, gq_host, ct_host = q_host.pin_memory(), gq_host.pin_memory(), ct_host.pin_memory()
    r.run_host(q_host, gq_host, ct_host, n_chunks=n_chunks)
    torch.cuda.current_stream().synchronize()
    assert np.array_equal(gq_host.numpy().view(np.uint32),
                          ref["grad_q"].reshape(-1).view(np.uint32))
    assert np.array_equal(ct_host.numpy().view(np.uint32), ref["cost_traj"].view(np.uint32))
    assert np.array_equal(r.cost_pose.cpu().numpy().view(np.uint32),
                          ref["cost_pose"].reshape(-1).view(np.uint32))
    assert torch.equal(r.workspace, ref_ws)


def test_cost_grad_host_errors(vb):
    from paper_2310_07854_b200.rollout import Rollout
    wl = config2()
    r = Rollout(wl)
    q_host = torch.from_numpy(np.ascontiguousarray(wl.q, np.float32))
    gq = torch.zeros(wl.B * wl.H * 7)
    with pytest.raises(vb.VaprError):          # negative chunk count
        r.run_host(q_host, gq, None, n_chunks=-1)
    with pytest.raises(ValueError):            # device tensor where a host buffer is expected
        r.run_host(r.q, gq, None)


def test_cost_grad_errors(vb):
    from paper_2310_07854_b200.rollout import Rollout
    wl = config2()
    r = Rollout(wl)
    with pytest.raises(vb.VaprError):          # swept with H = 1
        vb.vapr_cost_grad(r.ctx.h, r.q, r.world_idx, wl.B * wl.H, 1, wl.params, r.workspace,
                          r.cost_pose, r.cost_traj, r.grad_q)
    small = torch.zeros(16, dtype=torch.uint8, device="cuda")
    with pytest.raises(vb.VaprError):          # workspace too small
        vb.vapr_cost_grad(r.ctx.h, r.q, r.world_idx, wl.B, wl.H, wl.params, small,
                          r.cost_pose, r.cost_traj, r.grad_q)
    h = vb.vapr_create(0)
    with pytest.raises(vb.VaprError):          # not initialised
        vb.vapr_cost_grad(h, r.q, r.world_idx, wl.B, wl.H, wl.params, r.workspace,
                          r.cost_pose, r.cost_traj, r.grad_q)
    vb.vapr_destroy(h)


def test_discrete_h1_and_best_per_problem(vb):
    from paper_2310_07854_b200.rollout import Rollout
    wl = ragged_workload(B=5, H=1)
    wl.params["swept"] = 0
    r = Rollout(wl)
    r.run()
    out = r.results()
    # 43-bit formats: compare stage-wise (the GPU's own packed intermediates)
    f = r.ctx.formats
    p = wl.params
    os_w = r.packed(0)
    ws = orc.world_stage(os_w, f[0], wl.world_idx, wl.cuboids, wl.world_offsets, wl.robot, wl.B, 1,
                         p["eta_world"], p["w_world"], 0, p["sweep_steps"], f[3])
    ss = orc.self_stage(os_w, f[0], wl.robot, p["eta_self"], p["w_self"], f[2])
    ck = cost_kw(ws, ss)
    check_close(out["cost_traj"], ws["cost"].reshape(-1) + ss["cost"], what="cost_traj h=1", **ck)
    check_codes(r.packed(3), ws["v"], fmt=f[3], cols=156, what="closest_pt h=1",
                max_steps=step_bound(f[3]), **world_kw(ws))
    bc = torch.empty(1, dtype=torch.float32, device="cuda")
    bs = torch.empty(1, dtype=torch.int32, device="cuda")
    vb.vapr_best_per_problem(r.cost_traj, 1, 5, bc, bs)
    ct = r.cost_traj.cpu().numpy()
    assert bs.item() == int(np.argmin(ct)) and bc.item() == ct.min()


@pytest.mark.parametrize("storage", ["sparse", "dense"])
def test_full_size_sampled(vb, storage):
    """config4 at full size (2.56M poses) in the bench's launch -- sparse
    storage is the bench default -- checked on a sample of trajectories the
    oracle recomputes one by one: every packed tensor (out_spheres,
    closest_pt_swept, out_vec, grad_out_spheres) and the FP32 outputs."""
    from oracle import sparse as osp
    from paper_2310_07854_b200.rollout import Rollout
    wl = config4()
    r = Rollout(wl, sparse=(storage == "sparse"))
    r.run()
    out = r.results()
    rng = np.random.default_rng(0)
    picks = np.sort(rng.choice(wl.B, 12, replace=False))
    picks[-1] = wl.B - 1                   # the last trajectory (tail tile) too
    f = r.ctx.formats
    p = wl.params
    cols = 156
    for b in picks:
        w = wl.world_idx[b]
        cub = wl.cuboids[wl.world_offsets[w]:wl.world_offsets[w + 1]]
        offs = np.array([0, len(cub)], np.int32)
        q = wl.q[b:b + 1].reshape(-1, 7)
        rows = slice(b * wl.H, (b + 1) * wl.H)
        os_w = r.packed(0, rows)
        _, v = orc.fk_stage(q, wl.robot, f[0])
        check_codes(os_w, v, 1.0, 0.0, f[0], cols, what=f"out_spheres traj {b}")
        ws = orc.world_stage(os_w, f[0], np.zeros(1, np.int32), cub, offs, wl.robot, 1, wl.H,
                             p["eta_world"], p["w_world"], 1, p["sweep_steps"], f[4])
        ss = orc.self_stage(os_w, f[0], wl.robot, p["eta_self"], p["w_self"], f[2])
        if storage == "sparse":
            cp_w, ov_w = r.packed_dense(4, rows), r.packed_dense(2, rows)
            sg = r.sparse_gos(rows)
            gos_w = codec.pack(osp.densify(sg["mask"], sg["row_words"], *f[1], cols), *f[1])
        else:
            cp_w, ov_w, gos_w = r.packed(4, rows), r.packed(2, rows), r.packed(1, rows)
        check_codes(cp_w, ws["v"], fmt=f[4], cols=cols, what=f"closest_pt_swept traj {b}",
                    max_steps=step_bound(f[4]), **world_kw(ws))
        check_codes(ov_w, ss["v"], fmt=f[2], cols=cols, what=f"out_vec traj {b}",
                    max_steps=step_bound(f[2]), **self_kw(ss))
        ag = orc.aggregate_stage(cp_w, f[4], ov_w, f[2], f[1], cols)
        check_codes(gos_w, ag["v"], ag["terms"], 0.0, f[1], cols, what=f"grad_out_spheres traj {b}",
                    max_steps=step_bound(f[1]))
        bk = orc.bk_stage(q, gos_w, f[1], wl.robot)
        check_close(out["grad_q"][b], bk["grad_q"], bk["scale"], f"grad_q traj {b}")
        ck = cost_kw(ws, ss)
        check_close(out["cost_pose"][b], ws["cost"].reshape(-1) + ss["cost"], what=f"cost_pose traj {b}", **ck)
        check_close(np.atleast_1d(out["cost_traj"][b]), np.atleast_1d(ws["cost"].sum() + ss["cost"].sum()),
                    ck["terms"].sum(), f"cost_traj {b}", kappa=ck["kappa"].sum())


@pytest.mark.parametrize("name", ["config2", "mixed_envs", "bookshelf_tall", "fp32", "ragged_43"])
def test_cull_is_exact(vb, name):
    """Broadphase culling skips only exactly-zero terms: outputs and every
    packed intermediate are bit-identical with VAPR_OPT_CULL on and off."""
    from paper_2310_07854_b200.rollout import Rollout
    wl = WORKLOADS[name]()
    outs = []
    for cull in (1, 0):
        r = Rollout(wl)
        r.ctx.set_cull(cull)
        r.run()
        res = r.results()
        outs.append((res, [r.packed(i) for i in range(5)]))
    (a, pa), (b, pb) = outs
    for k in a:
        np.testing.assert_array_equal(a[k].view(np.uint32), b[k].view(np.uint32), err_msg=k)
    for x, y in zip(pa, pb):
        if x is not None:
            np.testing.assert_array_equal(x, y)


# ------------------------------------------------- a4, 16-bit tile rows (H16)
@pytest.mark.parametrize("shift", [0.0, 7.0e4, -1.2e5])
def test_self_pass_16bit_rows(vb, shift, monkeypatch):
    """The self pass keeps E5M10 out_spheres as 16-bit tile rows (collision.cu
    RowView): the hardware f16 conversion is exact for every E5M10 code but
    the exponent-31 ones, which the all-finite reading (DESIGN.md c3-c7)
    makes finite |x| >= 65536 and a tile holding one reads through the
    generic decoder.  shift != 0 moves every fifth trajectory by that many
    metres in x (exponent-31 codes; coarse quantisation puts spheres on top
    of each other, so those poses self-collide): against the oracle, and bit
    for bit against the FP32-row pass (VAPR_NO_H16)."""
    wl = config2()                       # E5M10 out_spheres (43-bit set)
    c = Ctx(vb, wl)
    P, B, H = wl.poses, wl.B, wl.H
    f = c.formats
    assert tuple(f[0]) == (5, 10)
    p = wl.params
    _, v = orc.fk_stage(wl.q.reshape(-1, 7), wl.robot, f[0])
    v = v.copy()
    moved = (np.arange(P) // H) % 5 == 2
    v[moved, 0::3] += shift
    os_words = orc.quantize_rows(v, f[0])
    osd = dev(os_words.view(np.int32))
    ss = orc.self_stage(os_words, f[0], wl.robot, p["eta_self"], p["w_self"], f[2])
    monkeypatch.setenv("VAPR_H16_MIN_POSES", "0")     # (the 16-bit rows on this small batch too)
    outs = []
    for no16 in (False, True):
        if no16:
            monkeypatch.setenv("VAPR_NO_H16", "1")
        cost = torch.empty(P, dtype=torch.float32, device="cuda")
        ov = torch.empty(P * c.W(2), dtype=torch.int32, device="cuda")
        vb.vapr_self_collision(c.h, osd, B, H, p["eta_self"], p["w_self"], cost, ov)
        outs.append((cost.cpu().numpy(), ov.cpu().numpy().view(np.uint32).reshape(P, -1)))
    monkeypatch.delenv("VAPR_NO_H16", raising=False)
    (cost16, ov16), (cost32, ov32) = outs
    assert np.array_equal(cost16.view(np.uint32), cost32.view(np.uint32))
    assert np.array_equal(ov16, ov32)
    check_close(cost16, ss["cost"].reshape(-1), ss["cost_terms"].reshape(-1), "self cost",
                kappa=ss["cost_kappa"].reshape(-1))
    check_codes(ov16, ss["v"], fmt=f[2], cols=156, what="out_vec", min_exact=0.999,
                max_steps=step_bound(f[2]), **self_kw(ss))
    if shift:
        assert (np.abs(v[moved]) >= 65536).any() and ss["cost"].reshape(-1)[moved].max() > 0


@pytest.mark.parametrize("H", [1, 7, 4096, 4097])
def test_traj_reduce_shapes(vb, H):
    """cost_traj = the in-order FP32 sum of each trajectory's cost_pose (a CTA
    stages whole trajectories for H <= 4096, a thread per trajectory above):
    bit for bit against numpy's sequential float32 sum of the GPU's own
    cost_pose, at the tile boundaries (H = 4096 / 4097) and for ragged B."""
    from workloads.scenes import ENVIRONMENTS
    B = 3 if H > 1000 else 37
    wl = make_workload("traj", [ENVIRONMENTS[i % 8] for i in range(B)], list(range(B)), 1, H,
                       FORMAT_SETS["43bit"], salt=5)
    c = Ctx(vb, wl)
    P = wl.poses
    os_words, _ = orc.fk_stage(wl.q.reshape(-1, 7), wl.robot, c.formats[0])
    cp = torch.empty(P * c.W(4), dtype=torch.int32, device="cuda")
    ov = torch.empty(P * c.W(2), dtype=torch.int32, device="cuda")
    cost = torch.empty(P, dtype=torch.float32, device="cuda")
    ctraj = torch.empty(B, dtype=torch.float32, device="cuda")
    p = dict(wl.params, swept=1 if H >= 2 else 0)      # (a swept cost needs H >= 2)
    vb.vapr_collision(c.h, dev(os_words.view(np.int32)), dev(wl.world_idx), B, H, p, cost, ctraj, cp, ov)
    cp_ = cost.cpu().numpy().reshape(B, H)
    ref = np.zeros(B, np.float32)
    for h in range(H):
        ref = (ref + cp_[:, h]).astype(np.float32)
    assert np.array_equal(ctraj.cpu().numpy().view(np.uint32), ref.view(np.uint32))


@pytest.mark.parametrize("shift", [0.0, 7.0e4])
@pytest.mark.parametrize("swept", [1, 0])
def test_world_pass_16bit_rows(vb, shift, swept, monkeypatch):
    """The world pass keeps E5M10 out_spheres as 16-bit tile rows too (halo
    rows included for the swept samples): against the oracle, and bit for bit
    against the FP32-row pass (VAPR_NO_H16); shift moves every fifth
    trajectory (and its cuboids' world) by that many metres in x, so its
    tiles hold exponent-31 codes and read through the generic decoder."""
    wl = config2()
    c = Ctx(vb, wl)
    P, B, H = wl.poses, wl.B, wl.H
    f = c.formats
    assert tuple(f[0]) == (5, 10)
    p = wl.params
    _, v = orc.fk_stage(wl.q.reshape(-1, 7), wl.robot, f[0])
    v = v.copy()
    moved = (np.arange(P) // H) % 5 == 2
    v[moved, 0::3] += shift
    os_words = orc.quantize_rows(v, f[0])
    osd = dev(os_words.view(np.int32))
    slot = 4 if swept else 3
    ws = orc.world_stage(os_words, f[0], wl.world_idx, wl.cuboids, wl.world_offsets, wl.robot,
                         B, H, p["eta_world"], p["w_world"], swept, p["sweep_steps"], f[slot])
    monkeypatch.setenv("VAPR_H16_MIN_POSES", "0")     # (the 16-bit rows on this small batch too)
    outs = []
    for no16 in (False, True):
        if no16:
            monkeypatch.setenv("VAPR_NO_H16", "1")
        cost = torch.empty(P, dtype=torch.float32, device="cuda")
        cp = torch.empty(P * c.W(slot), dtype=torch.int32, device="cuda")
        vb.vapr_world_collision(c.h, osd, dev(wl.world_idx), B, H, swept, p["sweep_steps"],
                                p["eta_world"], p["w_world"], cost, cp)
        outs.append((cost.cpu().numpy(), cp.cpu().numpy().view(np.uint32).reshape(P, -1)))
    monkeypatch.delenv("VAPR_NO_H16", raising=False)
    (cost16, cp16), (cost32, cp32) = outs
    assert np.array_equal(cost16.view(np.uint32), cost32.view(np.uint32))
    assert np.array_equal(cp16, cp32)
    check_close(cost16, ws["cost"].reshape(-1), ws["cost_terms"].reshape(-1), "world cost",
                kappa=ws["cost_kappa"].reshape(-1))
    check_codes(cp16, ws["v"], fmt=f[slot], cols=156, what="closest_pt", min_exact=0.999,
                max_steps=step_bound(f[slot]), **world_kw(ws))


@pytest.mark.parametrize("fs", ["43bit", "fp16"])
@pytest.mark.parametrize("sparse", [True, False])
def test_cost_grad_16bit_rows_identical(vb, fs, sparse, monkeypatch):
    """vapr_cost_grad with both collision passes on 16-bit tile rows (forced
    onto this small batch) against the FP32-row passes, bit for bit: cost_pose,
    cost_traj, grad_q and (sparse storage) every collision output's sparse
    rows -- the narrow (43-bit: three codes per word) and wide (FP16: a word
    per code) sparse instantiations and the dense one."""
    from paper_2310_07854_b200.rollout import Rollout
    from workloads.configs import FORMAT_SETS
    wl = dataclasses_replace(config2(), formats=tuple(FORMAT_SETS[fs]))
    res = []
    for no16 in (False, True):
        monkeypatch.setenv("VAPR_H16_MIN_POSES", "0")
        if no16:
            monkeypatch.setenv("VAPR_NO_H16", "1")
        r = Rollout(wl, device=0, sparse=sparse)
        r.run()
        out = r.results()
        extra = []
        if sparse:
            for slot in (vb.VAPR_CLOSEST_PT_SWEPT, vb.VAPR_OUT_VEC):
                sp = r.sparse_slot(slot)
                extra.append((sp["mask"], [w.tolist() for w in sp["row_words"]]))
        res.append((out, extra))
        monkeypatch.delenv("VAPR_NO_H16", raising=False)
    (a, ea), (b, eb) = res
    for k in ("cost_pose", "cost_traj", "grad_q"):
        assert np.array_equal(np.asarray(a[k]).view(np.uint32), np.asarray(b[k]).view(np.uint32)), k
    for (ma, wa), (mb, wb) in zip(ea, eb):
        assert np.array_equal(ma, mb) and wa == wb
