"""oracle/ikcost.py -- TEST INFRASTRUCTURE (see oracle/__init__.py).

The IKO workload's extra cost terms: PAPER.md:162 step
(3), "Compute cost functions which include pose, collision, self-collision,
and bound position".  The paper names the terms but not their formulas; the
readings:

  c34  the end-effector frame is the hand frame (link 8: flange . RotZ(hand_rz));
  c35  pose cost  C = w_pos |p - p_g|^2 + w_rot |R - R_g|_F^2  (goal (R_g, p_g)
       per problem); its gradient w.r.t. joint j (revolute about z_j through
       o_j) is  z_j . ((p - o_j) x F + tau)  with the force F = 2 w_pos (p - p_g)
       applied at p and the torque tau = -2 w_rot sum_k r_k x g_k (r_k, g_k the
       columns of R, R_g): dR = [w]x R for a rotation w, and
       <R - R_g, [w]x R> = w . sum_k r_k x (r_k - g_k);
  c36  bound cost  C = w_b sum_j (max(0, q_j - q_hi_j)^2 + max(0, q_lo_j - q_j)^2),
       gradient 2 w_b (max(0, q_j - q_hi_j) - max(0, q_lo_j - q_j)).

Plain float64 definitions; each is pinned by closed forms and central finite
differences in tests/test_oracle_ikcost.py.
"""
import numpy as np

from .kinematics import link_frames


def hand_pose(q, robot):
    """q [P, 7] -> (R [P, 3, 3], p [P, 3]) of the hand frame (c34)."""
    F = link_frames(q, robot)
    return F[:, 8, :3, :3], F[:, 8, :3, 3]


def pose_cost(q, robot, goal_R, goal_p, w_pos, w_rot):
    """c35: cost [P] and grad [P, 7]; goal_R [P, 3, 3], goal_p [P, 3]."""
    q = np.asarray(q, np.float64).reshape(-1, 7)
    F = link_frames(q, robot)
    R, p = F[:, 8, :3, :3], F[:, 8, :3, 3]
    gR = np.asarray(goal_R, np.float64).reshape(-1, 3, 3)
    gp = np.asarray(goal_p, np.float64).reshape(-1, 3)
    dp = p - gp
    cost = w_pos * np.sum(dp * dp, axis=1) + w_rot * np.sum((R - gR) ** 2, axis=(1, 2))
    force = 2.0 * w_pos * dp                                   # [P, 3] at p
    tau = -2.0 * w_rot * np.sum(np.cross(R.transpose(0, 2, 1), gR.transpose(0, 2, 1)), axis=1)
    grad = np.zeros((q.shape[0], 7))
    for j in range(1, 8):
        z = F[:, j, :3, 2]
        o = F[:, j, :3, 3]
        grad[:, j - 1] = np.einsum("pi,pi->p", z, np.cross(p - o, force) + tau)
    return cost, grad


def bound_cost(q, q_lo, q_hi, w_b):
    """c36: cost [P] and grad [P, 7]."""
    q = np.asarray(q, np.float64).reshape(-1, 7)
    hi = np.maximum(q - np.asarray(q_hi, np.float64)[None], 0.0)
    lo = np.maximum(np.asarray(q_lo, np.float64)[None] - q, 0.0)
    return w_b * np.sum(hi * hi + lo * lo, axis=1), 2.0 * w_b * (hi - lo)
