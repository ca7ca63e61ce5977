"""N2 on the GPU: the IKO workload's pose and bound costs
inside vapr_cost_grad (FK computes the cost, BK carries the hand-frame force
and torque and the bound gradient) against oracle/ikcost.py; the complete
IKO cost (pose + bound + discrete world + self) in FP32 end to end; IK solved
by TrajOpt (H = 1, D = 7)."""
import dataclasses

import numpy as np
import pytest
import torch

from oracle import ikcost as K
from oracle import rollout as orc
from parity_utils import check_close, e2e_kw, ik_kw
from workloads import config_iko

pytestmark = pytest.mark.gpu


@pytest.fixture(scope="module")
def vb():
    if not torch.cuda.is_available():
        pytest.skip("needs a GPU")
    from paper_2310_07854_b200 import binding
    return binding


def ik_only(wl, **w):
    p = dict(wl.params)
    p.update(w_world=0.0, w_self=0.0)
    p.update(w)
    return dataclasses.replace(wl, params=p)


@pytest.mark.parametrize("w", [dict(w_pose_pos=1.0, w_pose_rot=0.0, w_bound=0.0),
                               dict(w_pose_pos=0.0, w_pose_rot=0.7, w_bound=0.0),
                               dict(w_pose_pos=0.0, w_pose_rot=0.0, w_bound=2.0),
                               dict(w_pose_pos=1.0, w_pose_rot=0.5, w_bound=1.0)])
def test_ik_terms_match_oracle(vb, w):
    """Collision weights 0: cost_pose and grad_q are the IKO terms alone."""
    from paper_2310_07854_b200.rollout import Rollout
    wl = ik_only(config_iko(problems_per_env=1, seeds=24, formats="43bit"), **w)
    # push some seeds outside the joint limits so the bound term is exercised
    rng = np.random.default_rng(5)
    q = wl.q.copy()
    q[::3, 0, :] += rng.uniform(-0.4, 0.4, size=q[::3, 0, :].shape).astype(np.float32)
    wl = dataclasses.replace(wl, q=q)
    r = Rollout(wl)
    r.run()
    out = r.results()
    q64 = wl.q.reshape(-1, 7).astype(np.float64)
    gi = wl.world_idx
    G = wl.goals.astype(np.float64)[gi]
    cost = np.zeros(len(q64))
    grad = np.zeros_like(q64)
    if w["w_pose_pos"] or w["w_pose_rot"]:
        c, g = K.pose_cost(q64, wl.robot, G[:, :9].reshape(-1, 3, 3), G[:, 9:], w["w_pose_pos"],
                           w["w_pose_rot"])
        cost += c
        grad += g
    if w["w_bound"]:
        c, g = K.bound_cost(q64, wl.robot["q_lo"], wl.robot["q_hi"], w["w_bound"])
        cost += c
        grad += g
    kw = ik_kw(q64, wl.robot, G, w["w_pose_pos"], w["w_pose_rot"], w["w_bound"])
    check_close(out["cost_pose"].reshape(-1), cost, what="ik cost", **kw["cost"])
    check_close(out["grad_q"].reshape(-1, 7), grad, what="ik grad", **kw["grad"])


def test_iko_full_cost_fp32_end_to_end(vb):
    """All terms (pose + bound + discrete world + self), all formats E8M23:
    the composed GPU result agrees with the oracle rollout directly."""
    from paper_2310_07854_b200.rollout import Rollout
    wl = config_iko(problems_per_env=1, seeds=16, formats="fp32")
    r = Rollout(wl)
    r.run()
    out = r.results()
    res = orc.rollout_workload(wl)
    kw = e2e_kw(res, wl)
    p = wl.params
    G = np.asarray(wl.goals, np.float64)[np.repeat(wl.world_idx, wl.H)]
    ik = ik_kw(wl.q, wl.robot, G, p["w_pose_pos"], p["w_pose_rot"], p["w_bound"])
    ct_terms = kw["cost_traj"]["terms"] + ik["cost"]["terms"].reshape(wl.B, wl.H).sum(1)
    ct_kappa = kw["cost_traj"]["kappa"] + ik["cost"]["kappa"].reshape(wl.B, wl.H).sum(1)
    check_close(out["cost_traj"], res.cost_traj, ct_terms, "cost_traj", kappa=ct_kappa)
    check_close(out["grad_q"].reshape(-1, 7), res.grad_q.reshape(-1, 7), kw["grad_q"]["terms"] + ik["grad"]["terms"],
                "grad_q", kappa=kw["grad_q"]["kappa"] + ik["grad"]["kappa"])


def test_iko_requires_goals(vb):
    from paper_2310_07854_b200.rollout import Rollout
    wl = config_iko(problems_per_env=1, seeds=2)
    wl = dataclasses.replace(wl, goals=None)
    r = Rollout(wl)
    with pytest.raises(vb.VaprError):
        r.run()


@pytest.mark.parametrize("formats", ["43bit", "fp32"])
def test_ik_solved_by_trajopt(vb, formats):
    """IK with the N1 optimiser on the IKO workload (H = 1): every seed's cost
    is non-increasing, the batch's pose error drops, and a fresh
    vapr_cost_grad at the solution reproduces cost and gradient bit for bit."""
    from paper_2310_07854_b200.optimize import TrajOpt
    from paper_2310_07854_b200.rollout import Rollout
    wl = config_iko(problems_per_env=1, seeds=32, formats=formats)
    opt = TrajOpt(wl)
    opt.reset()
    start = opt.cost.cpu().numpy().copy()
    prev = start.copy()
    for _ in range(30):
        opt.step()
        now = opt.cost.cpu().numpy().copy()
        assert np.all(now <= prev)
        prev = now
    assert np.median(prev) < 0.5 * np.median(start)
    x = opt.x.cpu().numpy().reshape(wl.B, 1, 7)
    fresh = Rollout(wl)
    fresh.q.copy_(torch.from_numpy(x))
    fresh.run()
    out = fresh.results()
    assert np.array_equal(out["cost_traj"].view(np.uint32), prev.view(np.uint32))
    assert np.array_equal(out["grad_q"].reshape(-1).view(np.uint32),
                          opt.g.cpu().numpy().view(np.uint32))


def test_set_goals_errors(vb):
    h = vb.vapr_create(0)
    try:
        with pytest.raises(vb.VaprError):                   # n > 0 with a null pointer
            vb._check(vb.lib.vapr_set_goals(h, None, 3), "null goals")
        vb._check(vb.lib.vapr_set_goals(h, None, 0), "empty goals")   # n = 0: allowed
        with pytest.raises(vb.VaprError):
            vb._check(vb.lib.vapr_set_goals(h, None, -1), "negative")
    finally:
        vb.vapr_destroy(h)


@pytest.mark.parametrize("fmt", ["43bit", "fp32"])
def test_fk_ee_pose_matches_oracle(vb, fmt):
    """vapr_fk_spheres' optional ee_pose (reading c43)
    against oracle/ikcost.ee_pose: positions within FP32 evaluation error,
    the quaternion unit with w >= 0 and its rotation equal to the oracle's
    (compared as matrices: q and -q are the same rotation when w ~ 0); the
    packed out_spheres are unchanged by asking for it."""
    from paper_2310_07854_b200.rollout import Rollout
    wl = config_iko(problems_per_env=2, seeds=64, formats=fmt)
    r = Rollout(wl)
    P = wl.poses
    W = vb.vapr_packed_row_words(r.ctx.formats[0], 156)
    os_a = torch.zeros(P * W, dtype=torch.int32, device="cuda")
    os_b = torch.zeros(P * W, dtype=torch.int32, device="cuda")
    ee = torch.full((P * 7,), float("nan"), dtype=torch.float32, device="cuda")
    vb.vapr_fk_spheres(r.ctx.h, r.q, wl.B, wl.H, os_a)
    vb.vapr_fk_spheres(r.ctx.h, r.q, wl.B, wl.H, os_b, ee_pose=ee)
    torch.cuda.synchronize()
    assert torch.equal(os_a, os_b)
    got = ee.cpu().numpy().reshape(P, 7).astype(np.float64)
    ref = K.ee_pose(wl.q.reshape(-1, 7), wl.robot)
    np.testing.assert_allclose(got[:, :3], ref[:, :3], atol=2e-5)
    np.testing.assert_allclose(np.linalg.norm(got[:, 3:], axis=1), 1.0, atol=2e-6)
    assert np.all(got[:, 3] >= 0)
    np.testing.assert_allclose(K.matrix_from_quat(got[:, 3:]), K.matrix_from_quat(ref[:, 3:]),
                               atol=2e-5)
