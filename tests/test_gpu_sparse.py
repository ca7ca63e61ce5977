"""N3 on the GPU (reading c42): the sparse sphere-tensor
form through the C ABI.

* vapr_sparsify against oracle/sparse.py row by row (bitmap bit-exact, each
  row's pool words bit-exact, rows disjoint inside [0, used), used = the
  oracle's word total), every packing factor, ragged and empty inputs;
* vapr_densify of an oracle-built sparse form against codec.pack of the
  oracle's densify (independent of vapr_sparsify);
* vapr_cost_grad with VAPR_OPT_SPARSE: cost and grad_q bit-identical to the
  dense mode, grad_out_spheres' sparse rows equal to the oracle's sparsify
  of the dense mode's codes, and grad_q against the oracle rollout; also
  under trajectory chunks on streams, the host path and the IKO workload.
"""
import dataclasses

import numpy as np
import pytest
import torch

from oracle import codec
from oracle import rollout as orc
from oracle import sparse as osp
from parity_utils import check_close, check_codes, ik_kw
from workloads import config4, config_iko

pytestmark = pytest.mark.gpu

FORMATS = [(2, 1), (2, 2), (3, 2), (2, 3), (4, 3), (3, 4), (5, 10), (4, 9), (8, 7), (8, 23),
           (6, 9), (5, 4)]


@pytest.fixture(scope="module")
def vb():
    if not torch.cuda.is_available():
        pytest.skip("needs a GPU")
    from paper_2310_07854_b200 import binding
    return binding


def dev(a):
    return torch.from_numpy(np.ascontiguousarray(a)).cuda()


def random_sparse_codes(fmt, P, S=52, density=0.06, seed=0):
    E, M = fmt
    t = 1 + E + M
    rng = np.random.default_rng(seed)
    codes = rng.integers(0, 1 << min(t, 31), size=(P, 3 * S), dtype=np.uint64).astype(np.uint32)
    keep = rng.random((P, S)) < density
    if P > 2:
        keep[0] = False           # an empty row
        keep[1] = True            # a full row
    codes = codes * np.repeat(keep, 3, axis=1)
    if P > 3:                     # a sphere whose only non-zero code is -0 (sign bit)
        codes[2, :] = 0
        codes[2, min(4, 3 * S - 1)] = 1 << (t - 1) if t < 32 else 0x80000000
    return codes


def sparsify_gpu(vb, fmt, words, P, cols):
    mask = torch.zeros(P, dtype=torch.int64, device="cuda")
    off = torch.zeros(P, dtype=torch.int32, device="cuda")
    pool = torch.full((max(1, vb.vapr_sparse_pool_words(fmt, cols, P)),), -1, dtype=torch.int32,
                      device="cuda")
    used = torch.full((1,), 12345, dtype=torch.int32, device="cuda")
    vb.vapr_sparsify(fmt, dev(words.view(np.int32)), P, cols, mask, off, pool, used)
    torch.cuda.synchronize()
    return (mask.cpu().numpy().view(np.uint64), off.cpu().numpy().view(np.uint32),
            pool.cpu().numpy().view(np.uint32), int(used.cpu().numpy().view(np.uint32)[0]))


def check_sparse_rows(mask, off, pool, used, ref_mask, ref_rows):
    """pool: the whole capacity.  Bitmaps bit-exact, each row's words bit-exact,
    rows disjoint inside the capacity, used = the words in use."""
    assert np.array_equal(mask, ref_mask)
    assert used == sum(len(r) for r in ref_rows)
    cover = np.zeros(len(pool), np.int32)
    for p, r in enumerate(ref_rows):
        n = len(r)
        if n == 0:
            assert int(off[p]) == 0
            continue
        o = int(off[p])
        assert o + n <= len(pool)
        assert np.array_equal(pool[o:o + n], r), p
        cover[o:o + n] += 1
    assert cover.max(initial=0) <= 1   # disjoint


@pytest.mark.parametrize("fmt", FORMATS)
@pytest.mark.parametrize("P", [1, 37, 1000])
def test_sparsify_matches_oracle(vb, fmt, P):
    cols = 156
    codes = random_sparse_codes(fmt, P, seed=P + 7 * fmt[0] + fmt[1])
    words = codec.pack(codes, *fmt)
    mask, off, pool, used = sparsify_gpu(vb, fmt, words, P, cols)
    ref_mask, ref_rows = osp.sparsify(codes, *fmt)
    check_sparse_rows(mask, off, pool, used, ref_mask, ref_rows)


@pytest.mark.parametrize("fmt", [(2, 1), (3, 2), (8, 23)])
def test_sparsify_small_sphere_counts(vb, fmt):
    """S = 1 and S = 64 (the bitmap's full width)."""
    for S in (1, 64):
        codes = random_sparse_codes(fmt, 50, S=S, density=0.3, seed=S)
        words = codec.pack(codes, *fmt)
        mask, off, pool, used = sparsify_gpu(vb, fmt, words, 50, 3 * S)
        ref_mask, ref_rows = osp.sparsify(codes, *fmt)
        check_sparse_rows(mask, off, pool, used, ref_mask, ref_rows)


@pytest.mark.parametrize("fmt", FORMATS)
def test_densify_of_oracle_sparse_form(vb, fmt):
    P, cols = 300, 156
    codes = random_sparse_codes(fmt, P, seed=3 + fmt[0])
    ref_mask, ref_rows = osp.sparsify(codes, *fmt)
    # the oracle's rows laid out back to front (any disjoint placement is valid)
    offs = np.zeros(P, np.uint32)
    pool = []
    at = 0
    for p in reversed(range(P)):
        offs[p] = at if len(ref_rows[p]) else 0
        pool.extend(ref_rows[p].tolist())
        at += len(ref_rows[p])
    pool = np.array(pool + [0], np.uint32)
    W = vb.vapr_packed_row_words(fmt, cols)
    out = torch.full((P * W,), -1, dtype=torch.int32, device="cuda")
    vb.vapr_densify(fmt, dev(ref_mask.view(np.int64)), dev(offs.view(np.int32)),
                    dev(pool.view(np.int32)), P, cols, out)
    got = out.cpu().numpy().view(np.uint32).reshape(P, W)
    np.testing.assert_array_equal(got, codec.pack(osp.densify(ref_mask, ref_rows, *fmt, cols), *fmt))


@pytest.mark.parametrize("fmt", [(3, 2), (5, 10), (8, 23)])
def test_sparsify_densify_roundtrip(vb, fmt):
    P, cols = 2000, 156
    codes = random_sparse_codes(fmt, P, density=0.1, seed=11)
    words = codec.pack(codes, *fmt)
    mask = torch.zeros(P, dtype=torch.int64, device="cuda")
    off = torch.zeros(P, dtype=torch.int32, device="cuda")
    pool = torch.zeros(vb.vapr_sparse_pool_words(fmt, cols, P), dtype=torch.int32, device="cuda")
    used = torch.zeros(1, dtype=torch.int32, device="cuda")
    vb.vapr_sparsify(fmt, dev(words.view(np.int32)), P, cols, mask, off, pool, used)
    out = torch.zeros(words.size, dtype=torch.int32, device="cuda")
    vb.vapr_densify(fmt, mask, off, pool, P, cols, out)
    np.testing.assert_array_equal(out.cpu().numpy().view(np.uint32).reshape(words.shape), words)


def test_sparse_errors(vb):
    fmt = (3, 2)
    P, cols = 10, 156
    t = lambda n, d=torch.int32: torch.zeros(n, dtype=d, device="cuda")
    words = t(P * vb.vapr_packed_row_words(fmt, cols))
    with pytest.raises(vb.VaprError):       # pool below the worst case
        vb.vapr_sparsify(fmt, words, P, cols, t(P, torch.int64), t(P),
                         t(vb.vapr_sparse_pool_words(fmt, cols, P) - 1), t(1))
    with pytest.raises(vb.VaprError):       # cols not a multiple of 3
        vb.vapr_sparsify(fmt, words, P, 155, t(P, torch.int64), t(P), t(10000), t(1))
    with pytest.raises(vb.VaprError):       # more than 64 spheres
        vb.vapr_densify(fmt, t(P, torch.int64), t(P), t(10), P, 195, words)
    assert vb.vapr_sparse_pool_words(fmt, cols, P) == P * (-(-cols // 5))
    h = vb.vapr_create(0)
    try:
        with pytest.raises(vb.VaprError):   # layout query with the option off
            vb.vapr_cost_grad_sparse_layout(h, 2, 2)
        with pytest.raises(vb.VaprError):
            vb._check(vb.lib.vapr_set_option(h, vb.VAPR_OPT_SPARSE, 2), "bad value")
    finally:
        vb.vapr_destroy(h)


# ------------------------------------------------------ vapr_cost_grad
def run_pair(wl, streams=1):
    from paper_2310_07854_b200.rollout import Rollout
    a = Rollout(wl)
    b = Rollout(wl, sparse=True)
    a.ctx.set_streams(streams)
    b.ctx.set_streams(streams)
    a.run()
    b.run()
    return a, b


def check_pair(wl, a, b):
    ra, rb = a.results(), b.results()
    for k in ("cost_pose", "cost_traj", "grad_q"):
        assert np.array_equal(ra[k].view(np.uint32), rb[k].view(np.uint32)), k
    fg = a.ctx.formats[1]
    cols = 3 * len(wl.robot["sphere_link"])
    dense_codes = codec.unpack(a.packed(1), *fg, cols)
    ref_mask, ref_rows = osp.sparsify(dense_codes, *fg)
    sg = b.sparse_gos()
    check_sparse_rows(sg["mask"], sg["off"], sg["pool"], sg["used"], ref_mask, ref_rows)
    assert b.packed(1) is None         # no dense slot in sparse mode
    # the collision outputs in the sparse form: exactly the oracle's sparse
    # form of the dense mode's rows (mask and packed codes), and densified
    # they are those rows
    slot = 4 if wl.params["swept"] else 3
    for sl in (slot, 2):
        fs = a.ctx.formats[sl]
        assert b.packed(sl) is None, sl          # no dense slot in sparse mode
        m_ref, rows_ref = osp.sparsify(codec.unpack(a.packed(sl), *fs, cols), *fs)
        got = b.sparse_slot(sl)
        assert np.array_equal(got["mask"], m_ref), sl
        for k, (x, y) in enumerate(zip(got["row_words"], rows_ref)):
            assert np.array_equal(x, y), (sl, k)
        assert np.array_equal(b.packed_dense(sl), a.packed(sl)), sl
    # oracle parity of the sparse mode itself: its rows, densified by the
    # oracle, against the oracle's aggregation of the GPU's own collision
    # outputs (the dense stagewise rule), and BK of those codes
    p = wl.params
    f = b.ctx.formats
    g_codes = osp.densify(sg["mask"], [sg["pool"][int(o):int(o) + osp.row_words(m, *fg)]
                                       for m, o in zip(sg["mask"], sg["off"])], *fg, cols)
    g_words = codec.pack(g_codes, *fg)
    ag = orc.aggregate_stage(b.packed_dense(slot), f[slot], b.packed_dense(2), f[2], fg, cols)
    check_codes(g_words, ag["v"], ag["terms"], 0.0, fg, cols, what="sparse grad_out_spheres")
    bk = orc.bk_stage(wl.q.reshape(-1, 7), g_words, fg, wl.robot)
    ik = orc.ik_terms(wl.q, wl.world_idx, wl.robot, p, getattr(wl, "goals", None), wl.H)
    ref = bk["grad_q"] + (ik[1] if ik is not None else 0.0)
    terms, kappa = bk["scale"], 0.0
    if ik is not None:
        G = np.asarray(wl.goals, np.float64)[np.repeat(wl.world_idx, wl.H)]
        ikw = ik_kw(wl.q, wl.robot, G, p["w_pose_pos"], p["w_pose_rot"], p["w_bound"])["grad"]
        terms, kappa = terms + ikw["terms"], ikw["kappa"]
    check_close(rb["grad_q"].reshape(-1, 7), ref, terms, "grad_q", kappa=kappa)
    return rb


@pytest.mark.parametrize("formats", ["43bit", "fp32", "pf5_pf8", "bookshelf_tall"])
def test_cost_grad_sparse_equals_dense(vb, formats):
    wl = config4(problems_per_env=1, seeds=6, H=32, formats=formats)
    a, b = run_pair(wl)
    check_pair(wl, a, b)


def test_cost_grad_sparse_stale_rows(vb):
    """Sparse mode never zero-fills the collision rows: a second batch after a
    first one (different trajectories, stale fields everywhere) must give
    exactly the dense mode's results on the second batch."""
    from paper_2310_07854_b200.rollout import Rollout
    wl1 = config4(problems_per_env=1, seeds=8, H=32, formats="43bit")
    rng = np.random.default_rng(77)
    wl2 = dataclasses.replace(wl1, q=(wl1.q + rng.normal(0, 0.3, wl1.q.shape)).astype(np.float32))
    assert not np.array_equal(wl1.q, wl2.q)
    b = Rollout(wl1, sparse=True)
    b.run()
    b.run()
    b.q.copy_(torch.from_numpy(np.ascontiguousarray(wl2.q)))
    b.run()
    a = Rollout(wl2)
    a.run()
    b.wl = wl2
    check_pair(wl2, a, b)


def test_cost_grad_sparse_streams_and_host(vb):
    wl = config4(problems_per_env=1, seeds=10, H=32, formats="43bit")
    a, b = run_pair(wl, streams=3)
    check_pair(wl, a, b)
    # host path, chunked
    qh = torch.from_numpy(np.ascontiguousarray(wl.q)).pin_memory()
    gh = torch.zeros(wl.B * wl.H * 7, dtype=torch.float32).pin_memory()
    ch = torch.zeros(wl.B, dtype=torch.float32).pin_memory()
    b.run_host(qh, gh, ch, n_chunks=5)
    torch.cuda.synchronize()
    ra = a.results()
    assert np.array_equal(gh.numpy().view(np.uint32), ra["grad_q"].reshape(-1).view(np.uint32))
    assert np.array_equal(ch.numpy().view(np.uint32), ra["cost_traj"].view(np.uint32))


def test_cost_grad_sparse_iko(vb):
    """IKO: every pose is active in BK (hand force / torque), the bound
    gradient is per joint; the sparse mode changes nothing."""
    wl = config_iko(problems_per_env=1, seeds=24, formats="43bit")
    a, b = run_pair(wl)
    check_pair(wl, a, b)


def test_sparse_bytes_below_dense(vb):
    """The sparse form's stored bytes (12 per row + the pool words in use)
    on the bench-shaped workload, against the dense slot."""
    wl = config4(problems_per_env=2, seeds=20, H=32, formats="43bit")
    from paper_2310_07854_b200.rollout import Rollout
    b = Rollout(wl, sparse=True)
    b.run()
    sg = b.sparse_gos()
    P = wl.B * wl.H
    dense = P * 4 * vb.vapr_packed_row_words(b.ctx.formats[1], 156)
    sparse = 12 * P + 4 * sg["used"]
    assert sparse == osp.sparse_bytes(sg["mask"], *b.ctx.formats[1])
    assert sparse < dense / 3


def test_cost_grad_sparse_ieee_formats(vb):
    """Sparse storage with IEEE E5M10 slots (c41; BK's SP + SPR
    instantiation): bit-identical to the dense mode with the same formats."""
    from oracle.codec import FMT_IEEE
    wl = config4(problems_per_env=1, seeds=6, H=32, formats="fp16")
    wl = dataclasses.replace(wl, formats=((5, 10 | FMT_IEEE),) * 5)
    a, b = run_pair(wl)
    ra, rb = a.results(), b.results()
    for k in ("cost_pose", "cost_traj", "grad_q"):
        assert np.array_equal(ra[k].view(np.uint32), rb[k].view(np.uint32)), k


@pytest.mark.parametrize("case", ["ragged", "edge_worlds", "discrete_h1", "no_contact"])
def test_cost_grad_sparse_edge_cases(vb, case):
    """Sparse storage on the parity suite's edge workloads: ragged B x H (rows
    not a multiple of the 16-row tiles), obstacle-dense edge worlds, the
    discrete H = 1 workload (closest_pt, slot 3), and a batch with no contact
    at all (every bitmap empty, no pool words)."""
    from test_gpu_parity import edge_worlds_workload, ragged_workload
    if case == "ragged":
        wl = ragged_workload()
    elif case == "edge_worlds":
        wl = edge_worlds_workload()
    elif case == "discrete_h1":
        wl = config_iko(problems_per_env=1, seeds=40, formats="43bit")
        p = dict(wl.params)
        p.update(w_pose_pos=0.0, w_pose_rot=0.0, w_bound=0.0)
        wl = dataclasses.replace(wl, params=p)
    else:
        wl = config4(problems_per_env=1, seeds=4, H=8, formats="43bit")
        cub = wl.cuboids.copy()
        cub[:, 9:12] += 100.0                 # every obstacle far away
        p = dict(wl.params)
        p.update(w_self=0.0)
        wl = dataclasses.replace(wl, cuboids=cub, params=p)
    a, b = run_pair(wl)
    check_pair(wl, a, b)
    if case == "no_contact":
        sg = b.sparse_gos()
        assert sg["used"] == 0 and not sg["mask"].any()
