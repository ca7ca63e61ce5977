"""Pins for the Panda FK / BK oracle (closed forms, equivariance, finite
differences)."""
import math

import numpy as np

from oracle import kinematics as K
from workloads import panda_robot, READY_POSE

ROBOT = panda_robot()


def test_flange_at_zero_pose():
    # SURVEY.md §8(c) "FK (ext closed forms)": q = 0 -> flange (0.088, 0, 0.926), z down
    F = K.flange_pose(np.zeros((1, 7)), ROBOT)[0]
    np.testing.assert_allclose(F[:3, 3], [0.088, 0.0, 0.926], atol=1e-12)
    np.testing.assert_allclose(F[:3, 2], [0.0, 0.0, -1.0], atol=1e-12)


def test_flange_at_ready_pose():
    F = K.flange_pose(np.array([READY_POSE]), ROBOT)[0]
    np.testing.assert_allclose(F[:3, 3], [0.307, 0.0, 0.590], atol=1e-3)
    # independent closed form in the arm's vertical plane: shoulder at z=0.333,
    # upper arm 0.316 at -45 deg pitch, elbow offsets 0.0825, forearm 0.384 ...
    # the ready pose is planar (q1 = q3 = q5 = 0) so y must vanish exactly
    assert abs(F[1, 3]) < 1e-12


def test_joint1_equivariance():
    rng = np.random.default_rng(1)
    q = rng.uniform(ROBOT["q_lo"], ROBOT["q_hi"], (5, 7))
    phi = 0.7
    q2 = q.copy()
    q2[:, 0] += phi
    c1 = K.sphere_centers(q, ROBOT)
    c2 = K.sphere_centers(q2, ROBOT)
    Rz = np.array([[math.cos(phi), -math.sin(phi), 0], [math.sin(phi), math.cos(phi), 0], [0, 0, 1]])
    base = ROBOT["sphere_link"] == 0
    np.testing.assert_allclose(c2[:, ~base], c1[:, ~base] @ Rz.T, atol=1e-12)
    np.testing.assert_allclose(c2[:, base], c1[:, base], atol=0)


def test_sphere_on_hand_matches_flange_offset():
    # hand = flange . RotZ(-pi/4): a sphere at hand-local (0,0,z) lies on the flange z axis
    q = np.array([READY_POSE])
    F = K.flange_pose(q, ROBOT)[0]
    H = K.link_frames(q, ROBOT)[0, 8]
    np.testing.assert_allclose(H[:3, 3], F[:3, 3], atol=1e-12)
    np.testing.assert_allclose(H[:3, 2], F[:3, 2], atol=1e-12)
    np.testing.assert_allclose(H[:3, 0], (F[:3, 0] - F[:3, 1]) / math.sqrt(2), atol=1e-12)


def test_bk_matches_finite_differences():
    # L(q) = sum_s g_s . c_s(q); dL/dq by central differences (SURVEY.md §8(c) BK pin)
    rng = np.random.default_rng(2)
    q = rng.uniform(ROBOT["q_lo"], ROBOT["q_hi"], (4, 7))
    g = rng.normal(size=(4, 52, 3))
    an = K.backward(q, g, ROBOT)
    h = 1e-6
    fd = np.zeros_like(an)
    for j in range(7):
        dq = np.zeros(7)
        dq[j] = h
        Lp = np.einsum("psi,psi->p", g, K.sphere_centers(q + dq, ROBOT))
        Lm = np.einsum("psi,psi->p", g, K.sphere_centers(q - dq, ROBOT))
        fd[:, j] = (Lp - Lm) / (2 * h)
    np.testing.assert_allclose(an, fd, rtol=1e-7, atol=1e-8)


def test_bk_explicit_jacobian_and_zero():
    rng = np.random.default_rng(3)
    q = rng.uniform(ROBOT["q_lo"], ROBOT["q_hi"], (1, 7))
    # explicit 3x7 Jacobian of one sphere by finite differences, one-hot g
    s = 40
    g = np.zeros((1, 52, 3))
    g[0, s] = [0.3, -1.2, 0.5]
    h = 1e-6
    J = np.zeros((3, 7))
    for j in range(7):
        dq = np.zeros(7)
        dq[j] = h
        J[:, j] = (K.sphere_centers(q + dq, ROBOT)[0, s] - K.sphere_centers(q - dq, ROBOT)[0, s]) / (2 * h)
    np.testing.assert_allclose(K.backward(q, g, ROBOT)[0], J.T @ g[0, s], rtol=1e-7, atol=1e-9)
    assert not K.backward(q, np.zeros((1, 52, 3)), ROBOT).any()
    # a sphere on link 3 does not move with joints 4..7
    g2 = np.zeros((1, 52, 3))
    s3 = int(np.nonzero(ROBOT["sphere_link"] == 3)[0][0])
    g2[0, s3] = [1.0, 2.0, 3.0]
    assert not K.backward(q, g2, ROBOT)[0, 3:].any()
