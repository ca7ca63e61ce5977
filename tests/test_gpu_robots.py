"""Other robot tables through the whole path (vapr_set_robot builds the
collision kernel's table image, the link / half-link groups and their balls
from whatever robot it is given): a thinned sphere set with a link that has
no sphere, all candidate pairs (no ready-pose pruning: 3x the pairs), and a
64-sphere robot (VAPR_MAX_SPHERES).  Each is checked stage by stage against
the oracle (as test_gpu_parity.test_cost_grad_stagewise) and for bit-identity
between dense, sparse and fused storage."""
import dataclasses

import numpy as np
import pytest
import torch

from oracle import rollout as orc
from parity_utils import check_close, check_codes, cost_kw, self_kw, step_bound, world_kw
from workloads import config4
from workloads.robot import candidate_pairs

pytestmark = pytest.mark.gpu


@pytest.fixture(scope="module")
def vb():
    if not torch.cuda.is_available():
        pytest.skip("needs a GPU")
    from paper_2310_07854_b200 import binding
    return binding


def _with_robot(wl, keep=None, extra=None, all_pairs=False):
    r = dict(wl.robot)
    link = np.asarray(r["sphere_link"], np.int32)
    xyzr = np.asarray(r["sphere_xyzr"], np.float32)
    if keep is not None:
        link, xyzr = link[keep], xyzr[keep]
    if extra is not None:                       # more spheres on the hand / last links
        el, ex = extra
        link = np.concatenate([link, el]).astype(np.int32)
        xyzr = np.concatenate([xyzr, ex]).astype(np.float32)
        o = np.argsort(link, kind="stable")
        link, xyzr = link[o], xyzr[o]
    r["sphere_link"] = link
    r["sphere_xyzr"] = xyzr
    if all_pairs or keep is not None or extra is not None:
        pairs = candidate_pairs(link)
        if not all_pairs:                       # a deterministic thinning below the cap
            pairs = pairs[::3]
        r["pairs"] = pairs
    return dataclasses.replace(wl, robot=r)


def _variants():
    base = config4(problems_per_env=1, seeds=2, H=16)
    n = len(base.robot["sphere_link"])
    link = np.asarray(base.robot["sphere_link"])
    # every other sphere, and none on link 2
    keep = np.array([i for i in range(n) if i % 2 == 0 and link[i] != 2])
    rng = np.random.default_rng(5)
    el = np.array([8] * 6 + [7] * 6, np.int32)
    ex = np.concatenate([rng.uniform(-0.05, 0.05, (12, 3)), rng.uniform(0.02, 0.05, (12, 1))], 1)
    return {
        "thinned_no_link2": _with_robot(base, keep=keep),
        "all_candidate_pairs": _with_robot(base, all_pairs=True),
        "max_spheres_64": _with_robot(base, extra=(el, ex)),
    }


VARIANTS = _variants()


@pytest.mark.parametrize("name", list(VARIANTS))
def test_robot_variant_stagewise(vb, name):
    from paper_2310_07854_b200.rollout import Rollout
    wl = VARIANTS[name]
    S = len(wl.robot["sphere_link"])
    cols = 3 * S
    assert S <= 64 and len(wl.robot["pairs"]) <= 1024
    r = Rollout(wl)
    r.run()
    out = r.results()
    f = r.ctx.formats
    p = wl.params
    B, H, P = wl.B, wl.H, wl.poses
    slot = 4 if p["swept"] else 3
    os_w, cp_w, ov_w, gos_w = r.packed(0), r.packed(slot), r.packed(2), r.packed(1)
    _, v = orc.fk_stage(wl.q.reshape(-1, 7), wl.robot, f[0])
    check_codes(os_w, v, 1.0, 0.0, f[0], cols, what=f"{name} out_spheres")
    ws = orc.world_stage(os_w, f[0], wl.world_idx, wl.cuboids, wl.world_offsets, wl.robot, B, H,
                         p["eta_world"], p["w_world"], p["swept"], p["sweep_steps"], f[slot])
    ss = orc.self_stage(os_w, f[0], wl.robot, p["eta_self"], p["w_self"], f[2])
    check_codes(cp_w, ws["v"], fmt=f[slot], cols=cols, what=f"{name} closest_pt_swept",
                max_steps=step_bound(f[slot]), **world_kw(ws))
    check_codes(ov_w, ss["v"], fmt=f[2], cols=cols, what=f"{name} out_vec",
                max_steps=step_bound(f[2]), **self_kw(ss))
    ref_cost = (ws["cost"].reshape(-1) + ss["cost"]).reshape(B, H)
    ck = cost_kw(ws, ss)
    check_close(out["cost_pose"], ref_cost, ck["terms"].reshape(B, H), f"{name} cost_pose",
                kappa=ck["kappa"].reshape(B, H))
    ag = orc.aggregate_stage(cp_w, f[slot], ov_w, f[2], f[1], cols)
    check_codes(gos_w, ag["v"], ag["terms"], 0.0, f[1], cols, what=f"{name} grad_out_spheres",
                max_steps=step_bound(f[1]))
    bk = orc.bk_stage(wl.q.reshape(-1, 7), gos_w, f[1], wl.robot)
    check_close(out["grad_q"].reshape(P, 7), bk["grad_q"], bk["scale"], f"{name} grad_q")
    assert np.any(ss["v"] != 0) or name == "thinned_no_link2"


@pytest.mark.parametrize("name", list(VARIANTS))
def test_robot_variant_storage_modes_identical(vb, name):
    from paper_2310_07854_b200.rollout import Rollout
    wl = VARIANTS[name]
    res = []
    for kw in ({}, {"sparse": True}, {"fused": True}):
        r = Rollout(wl, **kw)
        r.run()
        res.append(r.results())
    for other in res[1:]:
        for k in ("cost_pose", "cost_traj", "grad_q"):
            assert np.array_equal(res[0][k].view(np.uint32), other[k].view(np.uint32)), (name, k)
