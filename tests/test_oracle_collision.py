"""Pins for the world / self collision oracle: closed-form SDF cases, hinge
continuity, invariances, swept special cases and finite differences."""
import math

import numpy as np

from conftest import golden
from oracle.collision import hinge, box_sdf, world_point_cost, world_cost, self_cost


def cub_row(R, t, h, dtype=np.float64):
    row = np.zeros(16, dtype)
    row[0:9] = np.asarray(R, np.float64).reshape(-1)
    row[9:12] = t
    row[12:15] = h
    return row


BOX = cub_row(np.eye(3), (0, 0, 0), (0.1, 0.2, 0.3))[None]


def test_sdf_golden_cases():
    for row in golden("sdf_box_cases.txt"):
        cx, cy, cz, sdf, cost, gx, gy, gz = map(float, row)
        c = np.array([[[cx, cy, cz]]])
        s = box_sdf(c, np.eye(3), np.zeros(3), np.array([0.1, 0.2, 0.3]))[0]
        assert abs(s[0, 0] - sdf) < 1e-12
        r = world_point_cost(c, np.array([0.05]), BOX, 0.02, 1.0)
        f, g = r["cost"], r["grad"]
        assert abs(f[0, 0] - cost) < 1e-12, (row, f)
        np.testing.assert_allclose(g[0, 0], [gx, gy, gz], atol=1e-12)


def test_hinge_c1_and_values():
    eta = 0.02
    h, dh = hinge(np.array([-1.0, 0.0, 0.01, eta, 0.05]), eta)
    np.testing.assert_allclose(h, [0, 0, 0.0025, 0.01, 0.04])
    np.testing.assert_allclose(dh, [0, 0, 0.5, 1.0, 1.0])
    e = 1e-9
    for x in (0.0, eta):
        a, da = hinge(np.array([x - e, x + e]), eta)
        assert abs(a[1] - a[0]) < 1e-8 and abs(da[1] - da[0]) < 1e-6


def test_translation_and_rotation_invariance():
    rng = np.random.default_rng(0)
    c = rng.uniform(-0.3, 0.3, (1, 50, 3))
    r = rng.uniform(0.04, 0.08, 50)
    yaw = 0.6
    R = np.array([[math.cos(yaw), -math.sin(yaw), 0], [math.sin(yaw), math.cos(yaw), 0], [0, 0, 1]])
    t = np.array([0.3, -0.2, 0.5])
    w0 = world_point_cost(c, r, BOX, 0.025, 1.0)
    f0, g0 = w0["cost"], w0["grad"]
    moved = cub_row(R, t, (0.1, 0.2, 0.3), np.float32)[None].astype(np.float64)
    Rm = moved[0, 0:9].reshape(3, 3)   # the float32-rounded rotation the world stores
    tm = moved[0, 9:12]
    c2 = c @ Rm.T + tm
    w1 = world_point_cost(c2, r, moved, 0.025, 1.0)
    f1, g1 = w1["cost"], w1["grad"]
    np.testing.assert_allclose(f1, f0, atol=1e-6)
    np.testing.assert_allclose(g1, g0 @ Rm.T, atol=1e-5)


def _fd_grad(fun, c, h=1e-7):
    g = np.zeros_like(c)
    for idx in np.ndindex(*c.shape):
        cp = c.copy()
        cm = c.copy()
        cp[idx] += h
        cm[idx] -= h
        g[idx] = (fun(cp) - fun(cm)) / (2 * h)
    return g


def test_world_discrete_finite_differences():
    rng = np.random.default_rng(1)
    c = rng.uniform(-0.25, 0.25, (1, 1, 12, 3))
    r = rng.uniform(0.04, 0.08, 12)
    cub = np.stack([BOX[0], cub_row(np.eye(3), (0.2, 0.1, 0.0), (0.05, 0.05, 0.05))])
    wc = world_cost(c, r, cub, 0.025, 1.3)
    cost, grad, tie = wc["cost"], wc["grad"], wc["tie"]
    assert not tie.any()
    fd = _fd_grad(lambda x: world_cost(x, r, cub, 0.025, 1.3)["cost"].sum(), c)
    np.testing.assert_allclose(grad, fd, atol=2e-6)


def test_world_swept_finite_differences_and_n0():
    rng = np.random.default_rng(2)
    H, S = 4, 6
    c = rng.uniform(-0.3, 0.3, (2, H, S, 3))
    r = rng.uniform(0.04, 0.08, S)
    for n in (1, 2):
        wc = world_cost(c, r, BOX, 0.025, 1.0, swept=True, n=n)
        cost, grad = wc["cost"], wc["grad"]
        fd = _fd_grad(lambda x: world_cost(x, r, BOX, 0.025, 1.0, swept=True, n=n)["cost"].sum(), c)
        np.testing.assert_allclose(grad, fd, atol=2e-6)
    d = world_cost(c, r, BOX, 0.025, 1.0)
    s0 = world_cost(c, r, BOX, 0.025, 1.0, swept=True, n=0)
    for a, b in zip(d, s0):
        np.testing.assert_array_equal(a, b)                 # n = 0 equals discrete


def test_swept_through_slab_hits_only_at_sample():
    # Thin slab at x = 0; a sphere moves from x=-0.5 to x=+0.5 in one step.
    slab = cub_row(np.eye(3), (0, 0, 0), (0.01, 1.0, 1.0))[None]
    c = np.array([[[[-0.5, 0, 0]], [[0.5, 0, 0]]]])
    r = np.array([0.05])
    cost_d = world_cost(c, r, slab, 0.025, 1.0)["cost"]
    assert not cost_d.any()                                  # endpoints free
    ws_ = world_cost(c, r, slab, 0.025, 1.0, swept=True, n=1)
    cost_s, grad_s = ws_["cost"], ws_["grad"]
    # midpoint at the slab centre: sdf = -0.01, phi = 0.05+0.025+0.01 = 0.085 > eta
    assert abs(cost_s[0, 0] - (0.085 - 0.0125)) < 1e-12 and cost_s[0, 1] == 0
    # gradient split (1 - tau, tau) = (0.5, 0.5) between the endpoints; the
    # midpoint lies on the x-face tie plane p=0 -> sign(0) = +1 -> -e_x
    np.testing.assert_allclose(grad_s[0, 0, 0], [-0.5, 0, 0])
    np.testing.assert_allclose(grad_s[0, 1, 0], [-0.5, 0, 0])


def test_self_golden_pairs_and_action_reaction():
    for d, cost, gnorm in (map(float, r) for r in golden("self_pair_cases.txt")):
        c = np.array([[[0.0, 0, 0], [d, 0, 0]]])
        sc = self_cost(c, np.array([0.05, 0.05]), np.array([[0, 1]], np.uint16), 0.01, 1.0)
        f, g = sc["cost"], sc["grad"]
        assert abs(f[0] - cost) < 1e-12
        assert abs(np.linalg.norm(g[0, 0]) - gnorm) < 1e-12
        np.testing.assert_allclose(g[0, 0], -g[0, 1])
        if gnorm > 0:
            assert g[0, 0, 0] > 0          # pushes sphere 0 towards -x: dcost/dx0 > 0
    rng = np.random.default_rng(3)
    c = rng.uniform(-0.1, 0.1, (3, 10, 3))
    pairs = np.array([(i, j) for i in range(10) for j in range(i + 2, 10)], np.uint16)
    sc = self_cost(c, np.full(10, 0.05), pairs, 0.01, 1.0)
    f, g = sc["cost"], sc["grad"]
    np.testing.assert_allclose(g.sum(axis=1), 0, atol=1e-12)   # sum out_vec = 0
    fd = _fd_grad(lambda x: self_cost(x, np.full(10, 0.05), pairs, 0.01, 1.0)["cost"].sum(), c)
    np.testing.assert_allclose(g, fd, atol=2e-6)
    # coincident centres -> direction (1, 0, 0)
    sc = self_cost(np.zeros((1, 2, 3)), np.array([0.05, 0.05]), np.array([[0, 1]], np.uint16), 0.01, 1.0)
    f, g = sc["cost"], sc["grad"]
    np.testing.assert_allclose(g[0, 0], [-1, 0, 0])


def test_sdf_tie_runner_up_face():
    """Reading c16: inside a cube at its centre all three faces tie; the
    gradient takes the lowest index (+x, sign(0) = +1) and the alternative
    the runner-up face (+y); away from ties the alternative is the gradient."""
    cube = np.array([0.1, 0.1, 0.1])
    sdf, g, tie, g_alt, _ = box_sdf(np.zeros((1, 3)), np.eye(3), np.zeros(3), cube)
    assert tie[0] and sdf[0] == -0.1
    np.testing.assert_array_equal(g[0], [1.0, 0.0, 0.0])
    np.testing.assert_array_equal(g_alt[0], [0.0, 1.0, 0.0])
    c = np.array([[0.05, 0.0, -0.02]])          # x face nearest, no tie
    sdf, g, tie, g_alt, _ = box_sdf(c, np.eye(3), np.zeros(3), cube)
    assert not tie[0]
    np.testing.assert_array_equal(g_alt, g)
