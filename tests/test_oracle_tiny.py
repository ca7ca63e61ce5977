"""Brute force on tiny inputs ("Brute force on tiny inputs.
B=1-2, H=1-3, K=1"): the oracle rollout (oracle/rollout.py: vectorised
collision, aggregation and analytic backward kinematics) against a plain
loop over spheres, cuboids, pairs and swept samples written from the
definitions (readings c11-c18), and against central finite
differences of that brute-force total cost for grad_q.  Only the forward
kinematics (pinned separately in test_oracle_kinematics.py) is shared."""
import math

import numpy as np
import pytest

from oracle import rollout as orc
from oracle.kinematics import sphere_centers
from workloads import config1

FP32 = ((8, 23),) * 5


def hinge(phi, eta):
    if phi <= 0.0:
        return 0.0
    if phi <= eta:
        return phi * phi / (2.0 * eta)
    return phi - eta / 2.0


def box_sdf(c, cub):
    R = np.asarray(cub[0:9], np.float64).reshape(3, 3)
    t = np.asarray(cub[9:12], np.float64)
    h = np.asarray(cub[12:15], np.float64)
    p = R.T @ (np.asarray(c, np.float64) - t)
    u = [abs(p[k]) - h[k] for k in range(3)]
    outside = math.sqrt(sum(max(x, 0.0) ** 2 for x in u))
    return outside + min(max(u), 0.0)


def brute_cost_pose(q, robot, cuboids, params):
    """cost_pose [H] of one trajectory q [H, 7], loops only."""
    H = q.shape[0]
    c = sphere_centers(q.astype(np.float64), robot)          # [H, S, 3]
    r = robot["sphere_xyzr"][:, 3].astype(np.float64)
    S = len(r)
    ew, ww = params["eta_world"], params["w_world"]
    es, ws = params["eta_self"], params["w_self"]
    n = params["sweep_steps"] if params["swept"] else 0

    def world(x):
        tot = 0.0
        for s in range(S):
            for cub in cuboids:
                tot += ww * hinge(r[s] + ew - box_sdf(x[s], cub), ew)
        return tot

    out = np.zeros(H)
    for h in range(H):
        out[h] += world(c[h])
        for i, j in robot["pairs"]:
            d = math.sqrt(sum((c[h, i, k] - c[h, j, k]) ** 2 for k in range(3)))
            out[h] += ws * hinge(r[i] + r[j] + es - d, es)
        if h + 1 < H:
            for jj in range(1, n + 1):
                tau = jj / (n + 1.0)
                out[h] += world((1.0 - tau) * c[h] + tau * c[h + 1])
    return out


def tiny_case(seed, swept, H=3):
    """A window of H consecutive steps of config 1 (K = 1 cuboid) whose every
    pose has a non-zero cost (world and / or self), the seed-th such window."""
    wl = config1(reduced=False)
    params = dict(wl.params)
    params["swept"] = swept
    found = []
    for b in range(wl.B):
        for h0 in range(0, wl.H - H + 1, 2):
            cp = brute_cost_pose(wl.q[b, h0:h0 + H], wl.robot, wl.cuboids, params)
            if cp.min() > 0:
                found.append((b, h0))
        if len(found) > seed:
            break
    assert len(found) > seed, "no active window in config 1"
    b, h0 = found[seed]
    return wl, params, wl.q[b:b + 1, h0:h0 + H].copy()


@pytest.mark.parametrize("swept", [1, 0])
@pytest.mark.parametrize("seed", [0, 1])
def test_rollout_matches_brute_force(seed, swept):
    wl, params, q = tiny_case(seed, swept)
    res = orc.rollout(q, np.zeros(1, np.int32), wl.cuboids, wl.world_offsets, wl.robot, params,
                      FP32)
    ref = brute_cost_pose(q[0], wl.robot, wl.cuboids, params)
    assert ref.min() > 0
    # E8M23 storage rounds sphere centres to float32 (~6e-8 relative)
    np.testing.assert_allclose(res.cost_pose[0], ref, rtol=2e-5, atol=1e-9)
    np.testing.assert_allclose(res.cost_traj[0], ref.sum(), rtol=2e-5, atol=1e-9)
    # grad_q against central finite differences of the brute-force trajectory cost
    eps = 1e-6
    H = q.shape[1]
    fd = np.zeros((H, 7))
    for h in range(H):
        for j in range(7):
            qp = q[0].astype(np.float64).copy()
            qm = q[0].astype(np.float64).copy()
            qp[h, j] += eps
            qm[h, j] -= eps
            fd[h, j] = (brute_cost_pose(qp, wl.robot, wl.cuboids, params).sum()
                        - brute_cost_pose(qm, wl.robot, wl.cuboids, params).sum()) / (2 * eps)
    g = res.grad_q[0]
    scale = np.abs(fd).max()
    np.testing.assert_allclose(g, fd, atol=2e-4 * scale + 1e-6)
