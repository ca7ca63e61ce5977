"""Pins of oracle/ikcost.py (readings c34-c36): closed
forms of the pose and bound costs and central finite differences of every
analytic gradient."""
import numpy as np
import pytest

from oracle import ikcost as K
from workloads import panda_robot

ROBOT = panda_robot()


def rot(axis, th):
    a = np.asarray(axis, np.float64)
    a = a / np.linalg.norm(a)
    Kx = np.array([[0, -a[2], a[1]], [a[2], 0, -a[0]], [-a[1], a[0], 0]])
    return np.eye(3) + np.sin(th) * Kx + (1 - np.cos(th)) * Kx @ Kx


def rand_q(rng, n):
    return rng.uniform(ROBOT["q_lo"], ROBOT["q_hi"], size=(n, 7))


def test_pose_cost_zero_at_goal():
    q = rand_q(np.random.default_rng(0), 5)
    R, p = K.hand_pose(q, ROBOT)
    c, g = K.pose_cost(q, ROBOT, R, p, 1.0, 0.7)
    np.testing.assert_allclose(c, 0.0, atol=1e-28)
    np.testing.assert_allclose(g, 0.0, atol=1e-14)


def test_pose_cost_closed_forms():
    """Translation offset: cost = w |d|^2; rotation offset by angle th about
    any axis: |R - R Rot|_F^2 = |I - Rot|_F^2 = 4 (1 - cos th)."""
    q = rand_q(np.random.default_rng(1), 4)
    R, p = K.hand_pose(q, ROBOT)
    d = np.array([0.1, -0.2, 0.05])
    c, _ = K.pose_cost(q, ROBOT, R, p + d, 2.0, 0.0)
    np.testing.assert_allclose(c, 2.0 * d @ d, rtol=1e-12)
    for th in (0.3, 1.1, 2.9):
        gR = R @ rot([1.0, 2.0, -0.5], th)[None]
        c, _ = K.pose_cost(q, ROBOT, gR, p, 0.0, 1.5)
        np.testing.assert_allclose(c, 1.5 * 4.0 * (1.0 - np.cos(th)), rtol=1e-10)


def test_bound_cost_closed_forms():
    lo, hi = ROBOT["q_lo"], ROBOT["q_hi"]
    mid = 0.5 * (lo + hi)
    c, g = K.bound_cost(mid[None], lo, hi, 3.0)
    assert c[0] == 0.0 and np.all(g == 0.0)
    q = mid.copy()
    q[2] = hi[2] + 0.1
    q[5] = lo[5] - 0.2
    c, g = K.bound_cost(q[None], lo, hi, 3.0)
    np.testing.assert_allclose(c[0], 3.0 * (0.01 + 0.04), rtol=1e-12)
    np.testing.assert_allclose(g[0, 2], 3.0 * 2 * 0.1, rtol=1e-9)
    np.testing.assert_allclose(g[0, 5], -3.0 * 2 * 0.2, rtol=1e-9)
    assert np.count_nonzero(g) == 2


@pytest.mark.parametrize("seed", range(4))
def test_pose_gradient_finite_differences(seed):
    rng = np.random.default_rng(10 + seed)
    q = rand_q(rng, 3)
    gR = np.stack([rot(rng.normal(size=3), rng.uniform(0, 3)) for _ in range(3)])
    gp = rng.uniform([0.2, -0.5, 0.1], [0.8, 0.5, 0.9], size=(3, 3))
    _, g = K.pose_cost(q, ROBOT, gR, gp, 1.3, 0.4)
    h = 1e-6
    for j in range(7):
        e = np.zeros(7)
        e[j] = h
        cp, _ = K.pose_cost(q + e, ROBOT, gR, gp, 1.3, 0.4)
        cm, _ = K.pose_cost(q - e, ROBOT, gR, gp, 1.3, 0.4)
        np.testing.assert_allclose(g[:, j], (cp - cm) / (2 * h), rtol=1e-6, atol=1e-8)


def test_bound_gradient_finite_differences():
    rng = np.random.default_rng(3)
    lo, hi = ROBOT["q_lo"], ROBOT["q_hi"]
    q = rng.uniform(lo - 0.5, hi + 0.5, size=(6, 7))
    _, g = K.bound_cost(q, lo, hi, 0.8)
    h = 1e-6
    for j in range(7):
        e = np.zeros(7)
        e[j] = h
        cp, _ = K.bound_cost(q + e, lo, hi, 0.8)
        cm, _ = K.bound_cost(q - e, lo, hi, 0.8)
        np.testing.assert_allclose(g[:, j], (cp - cm) / (2 * h), rtol=1e-5, atol=1e-8)


def test_ee_pose_at_zero_closed_form():
    """q = 0: the flange sits at (0.088, 0, 0.926) with z pointing down
    (SURVEY.md §8(c) FK pins), i.e. R_flange = diag(1, -1, -1); the hand is
    the flange turned by hand_rz about its z: R = diag(1,-1,-1) RotZ(hand_rz),
    whose quaternion is (0, cos(hand_rz/2), -sin(hand_rz/2), 0) up to sign."""
    e = K.ee_pose(np.zeros((1, 7)), ROBOT)[0]
    np.testing.assert_allclose(e[:3], [0.088, 0.0, 0.926], atol=1e-3)
    th = ROBOT["hand_rz"]
    ref = np.array([0.0, np.cos(th / 2), -np.sin(th / 2), 0.0])
    assert np.allclose(e[3:], ref, atol=1e-9) or np.allclose(e[3:], -ref, atol=1e-9)


def test_quaternion_round_trip_and_branches():
    """Every Shepperd branch (positive trace, and each diagonal entry the
    largest): matrix -> quaternion -> matrix is the identity map, the
    quaternion is unit with w >= 0."""
    rng = np.random.default_rng(4)
    Rs = [rot([0, 0, 1], 0.3), rot([1, 0, 0], 3.0), rot([0, 1, 0], 3.0), rot([0, 0, 1], 3.0),
          rot([1, 1, 0], np.pi), np.eye(3)]
    Rs += [rot(rng.normal(size=3), rng.uniform(0, np.pi)) for _ in range(50)]
    R = np.stack(Rs)
    qt = K.quat_from_matrix(R)
    np.testing.assert_allclose(np.linalg.norm(qt, axis=1), 1.0, atol=1e-12)
    assert np.all(qt[:, 0] >= 0)
    np.testing.assert_allclose(K.matrix_from_quat(qt), R, atol=1e-12)


def test_ee_pose_matches_hand_frame():
    q = rand_q(np.random.default_rng(9), 20)
    R, p = K.hand_pose(q, ROBOT)
    e = K.ee_pose(q, ROBOT)
    np.testing.assert_allclose(e[:, :3], p, atol=0)
    np.testing.assert_allclose(K.matrix_from_quat(e[:, 3:]), R, atol=1e-12)
