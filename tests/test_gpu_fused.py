"""N4 on the GPU: the fused on-chip
rollout -- FK, world + self collision, aggregation and BK in one kernel, every
slot's tensor quantise->dequantised in registers and never stored.

* bit-identity with the materialised path (whose every stage
  test_gpu_parity.py checks against the oracle) over format sets, swept and
  discrete, culling on and off, ragged / empty-world / engulfing edge cases
  and at the bench's full size;
* the all-E8M23 fused result against the oracle rollout directly (no stage
  re-feeding), with the end-to-end tolerances of parity_utils.e2e_kw;
* the workspace it needs (the cost scratch only) and its refusals (IKO
  weights, VAPR_OPT_SPARSE).
"""
import dataclasses

import numpy as np
import pytest
import torch

from oracle import rollout as orc
from parity_utils import check_close, e2e_kw
from workloads import config2, config4, config_iko, make_workload
from workloads.configs import FORMAT_SETS

pytestmark = pytest.mark.gpu


@pytest.fixture(scope="module")
def vb():
    if not torch.cuda.is_available():
        pytest.skip("needs a GPU")
    from paper_2310_07854_b200 import binding
    return binding


def _ragged(B=3, H=5, salt=9, formats="43bit"):
    from workloads.scenes import ENVIRONMENTS
    envs = [ENVIRONMENTS[i % 8] for i in range(B)]
    return make_workload("ragged", envs, list(range(B)), 1, H, FORMAT_SETS[formats], salt=salt)


def _edge_worlds():
    from test_gpu_parity import edge_worlds_workload
    return edge_worlds_workload()


def _discrete(wl):
    p = dict(wl.params)
    p["swept"] = 0
    return dataclasses.replace(wl, params=p)


WORKLOADS = {
    "config2": config2,
    "mixed_envs": lambda: config4(problems_per_env=1, seeds=3, H=32),
    "discrete": lambda: _discrete(config4(problems_per_env=1, seeds=3, H=32)),
    "fp32": lambda: config4(problems_per_env=1, seeds=2, H=32, formats="fp32"),
    "fp16": lambda: config4(problems_per_env=1, seeds=2, H=32, formats="fp16"),
    "bf16": lambda: config4(problems_per_env=1, seeds=2, H=32, formats="bf16"),
    "pf3": lambda: config4(problems_per_env=1, seeds=2, H=32, formats="pf3"),
    "pf5_pf8": lambda: config4(problems_per_env=1, seeds=2, H=32, formats="pf5_pf8"),
    "bookshelf_tall": lambda: config4(problems_per_env=1, seeds=2, H=32, formats="bookshelf_tall"),
    "ragged_43": _ragged,
    "h2_min_swept": lambda: _ragged(B=4, H=2, salt=23),
    "edge_worlds": _edge_worlds,
}


def _pair(wl, cull=True):
    from paper_2310_07854_b200.rollout import Rollout
    mat = Rollout(wl)
    fus = Rollout(wl, fused=True)
    for r in (mat, fus):
        r.ctx.set_cull(cull)
        r.run()
    return mat.results(), fus.results(), mat, fus


def _assert_identical(a, b, what):
    for k in ("cost_pose", "cost_traj", "grad_q"):
        x, y = np.asarray(a[k]), np.asarray(b[k])
        bad = np.nonzero(x.view(np.uint32) != y.view(np.uint32))
        assert not len(bad[0]), (f"{what} {k}: {len(bad[0])} of {x.size} differ; first at "
                                 f"{[i[:3] for i in bad]}: materialised {x[bad][:3]} fused {y[bad][:3]}")


@pytest.mark.parametrize("name", list(WORKLOADS))
def test_fused_bit_identical_to_materialised(vb, name):
    wl = WORKLOADS[name]()
    mat, fus, _, _ = _pair(wl)
    _assert_identical(mat, fus, name)
    if name in ("config2", "mixed_envs", "fp32", "fp16"):
        assert np.any(mat["grad_q"] != 0)


@pytest.mark.parametrize("name", ["mixed_envs", "fp32"])
def test_fused_brute_force(vb, name):
    """Culling off (VAPR_OPT_CULL = 0) takes every test through the
    narrowphase: the same result."""
    wl = WORKLOADS[name]()
    mat, fus, _, _ = _pair(wl, cull=False)
    _assert_identical(mat, fus, name + " (no cull)")


def test_fused_fp32_end_to_end_vs_oracle(vb):
    """All-E8M23: the fused kernel against the oracle rollout directly."""
    from paper_2310_07854_b200.rollout import Rollout
    wl = config4(problems_per_env=1, seeds=2, H=32, formats="fp32")
    r = Rollout(wl, fused=True)
    r.run()
    out = r.results()
    res = orc.rollout_workload(wl)
    kw = e2e_kw(res, wl)
    check_close(out["cost_traj"], res.cost_traj, what="fused cost_traj", **kw["cost_traj"])
    check_close(out["cost_pose"], res.cost_pose, what="fused cost_pose", **kw["cost_pose"])
    check_close(out["grad_q"].reshape(-1, 7), res.grad_q.reshape(-1, 7), what="fused grad_q",
                **kw["grad_q"])


def test_fused_full_size(vb):
    """The bench workload (config4 full size, 2.56M poses), fused against
    materialised, bit for bit on the device."""
    from paper_2310_07854_b200.rollout import Rollout
    wl = config4()
    mat = Rollout(wl)
    fus = Rollout(wl, fused=True, ctx=None)
    mat.run()
    fus.run()
    torch.cuda.synchronize()
    for k in ("cost_pose", "cost_traj", "grad_q"):
        a, b = getattr(mat, k), getattr(fus, k)
        assert torch.equal(a.view(torch.int32), b.view(torch.int32)), k
    assert fus.workspace.numel() < mat.workspace.numel() // 20


def test_fused_streams_and_host_path(vb):
    """Trajectory chunks on several streams and the host-buffer path."""
    from paper_2310_07854_b200.rollout import Rollout
    wl = config4(problems_per_env=2, seeds=5, H=32)
    mat, fus, _, _ = _pair(wl)
    r = Rollout(wl, fused=True)
    r.ctx.set_streams(3)
    r.run()
    _assert_identical(mat, r.results(), "streams")
    r2 = Rollout(wl, fused=True)
    qh = torch.from_numpy(np.ascontiguousarray(wl.q)).pin_memory()
    gh = torch.zeros(wl.B * wl.H * 7, dtype=torch.float32).pin_memory()
    ch = torch.zeros(wl.B, dtype=torch.float32).pin_memory()
    r2.run_host(qh, gh, ch, n_chunks=3)
    torch.cuda.synchronize()
    assert np.array_equal(gh.numpy().view(np.uint32), mat["grad_q"].reshape(-1).view(np.uint32))
    assert np.array_equal(ch.numpy().view(np.uint32), mat["cost_traj"].view(np.uint32))


def test_fused_refusals(vb):
    from paper_2310_07854_b200.rollout import Rollout
    wl = config_iko(problems_per_env=1, seeds=2)
    r = Rollout(wl, fused=True)
    with pytest.raises(RuntimeError, match="UNSUPPORTED|unsupported"):
        r.run()
    wl2 = config4(problems_per_env=1, seeds=1, H=8)
    r2 = Rollout(wl2, fused=True)
    r2.ctx.set_sparse(True)
    with pytest.raises(RuntimeError, match="UNSUPPORTED|unsupported"):
        r2.run()


IEEE = 0x100
SWEEP_FORMATS = [(5, 10), (8, 7), (4, 3), (5, 2), (2, 1), (2, 3), (3, 2), (3, 4), (4, 9),
                 (6, 9), (2, 2), (7, 12), (3, 23), (8, 23), (5, 10 | IEEE), (8, 7 | IEEE)]


def _same(a, b):
    a, b = np.asarray(a), np.asarray(b)
    return np.all((a.view(np.uint32) == b.view(np.uint32)) | (np.isnan(a) & np.isnan(b)))


@pytest.mark.parametrize("fmt", SWEEP_FORMATS, ids=str)
def test_fused_format_sweep(vb, fmt):
    """Every hardware-conversion kind, the generic path, E < 8 with M = 23
    and both IEEE modes in all five slots: the in-register fake quantiser
    gives decode(encode(x)) value for value (through the materialised path's
    stored codes)."""
    from paper_2310_07854_b200.rollout import Rollout
    wl = config4(problems_per_env=1, seeds=2, H=32)
    mat = Rollout(wl, formats=(fmt,) * 5)
    fus = Rollout(wl, formats=(fmt,) * 5, fused=True)
    mat.run()
    fus.run()
    a, b = mat.results(), fus.results()
    for k in ("cost_pose", "cost_traj", "grad_q"):
        assert _same(a[k], b[k]), (fmt, k)


@pytest.mark.parametrize("gfmt", [(5, 10), (5, 10 | IEEE), (8, 7 | IEEE), (4, 3), (2, 1)], ids=str)
def test_fused_saturation_and_overflow(vb, gfmt):
    """A world weight that overflows the gradient formats: saturation
    (all-finite) and inf (IEEE) in grad_out_spheres reach BK the same way."""
    from paper_2310_07854_b200.rollout import Rollout
    wl = config4(problems_per_env=1, seeds=4, H=32, formats="fp32")
    p = dict(wl.params)
    p.update(w_world=3e6, w_self=3e6)
    wl = dataclasses.replace(wl, params=p)
    fm = [(8, 23)] * 5
    fm[1] = gfmt
    fm[4] = (5, 10) if gfmt[0] == 5 else gfmt
    mat = Rollout(wl, formats=tuple(fm))
    fus = Rollout(wl, formats=tuple(fm), fused=True)
    mat.run()
    fus.run()
    a, b = mat.results(), fus.results()
    for k in ("cost_pose", "cost_traj", "grad_q"):
        assert _same(a[k], b[k]), (gfmt, k)
    if gfmt == (5, 10 | IEEE):          # E8M7's range holds these gradients
        assert not np.all(np.isfinite(b["grad_q"]))
