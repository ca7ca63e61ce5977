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
  c43  ee_pose: the hand frame as position + unit quaternion (w, x, y, z), the
       one with w >= 0 (`ee_pose`);
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


def quat_from_matrix(R):
    """R [P, 3, 3] -> unit quaternions [P, 4] = (w, x, y, z), w >= 0 (reading
    c43: the canonical one of the two).  Shepperd's method: the largest of
    1 + tr, 1 + 2 R_ii - tr gives the well-conditioned component."""
    R = np.asarray(R, np.float64).reshape(-1, 3, 3)
    out = np.zeros((R.shape[0], 4))
    for n, m in enumerate(R):
        tr = m[0, 0] + m[1, 1] + m[2, 2]
        if tr > 0:
            s = 2.0 * np.sqrt(1.0 + tr)
            w, x, y, z = 0.25 * s, (m[2, 1] - m[1, 2]) / s, (m[0, 2] - m[2, 0]) / s, (m[1, 0] - m[0, 1]) / s
        elif m[0, 0] > m[1, 1] and m[0, 0] > m[2, 2]:
            s = 2.0 * np.sqrt(1.0 + m[0, 0] - m[1, 1] - m[2, 2])
            w, x, y, z = (m[2, 1] - m[1, 2]) / s, 0.25 * s, (m[0, 1] + m[1, 0]) / s, (m[0, 2] + m[2, 0]) / s
        elif m[1, 1] > m[2, 2]:
            s = 2.0 * np.sqrt(1.0 + m[1, 1] - m[0, 0] - m[2, 2])
            w, x, y, z = (m[0, 2] - m[2, 0]) / s, (m[0, 1] + m[1, 0]) / s, 0.25 * s, (m[1, 2] + m[2, 1]) / s
        else:
            s = 2.0 * np.sqrt(1.0 + m[2, 2] - m[0, 0] - m[1, 1])
            w, x, y, z = (m[1, 0] - m[0, 1]) / s, (m[0, 2] + m[2, 0]) / s, (m[1, 2] + m[2, 1]) / s, 0.25 * s
        v = np.array([w, x, y, z])
        out[n] = -v if w < 0 else v
    return out


def matrix_from_quat(qt):
    """(w, x, y, z) [P, 4] -> R [P, 3, 3] (the textbook unit-quaternion form)."""
    w, x, y, z = (np.asarray(qt, np.float64).reshape(-1, 4)[:, k] for k in range(4))
    return np.stack([
        np.stack([1 - 2 * (y * y + z * z), 2 * (x * y - w * z), 2 * (x * z + w * y)], -1),
        np.stack([2 * (x * y + w * z), 1 - 2 * (x * x + z * z), 2 * (y * z - w * x)], -1),
        np.stack([2 * (x * z - w * y), 2 * (y * z + w * x), 1 - 2 * (x * x + y * y)], -1)], 1)


def ee_pose(q, robot):
    """vapr_fk_spheres' optional ee_pose: the
    hand frame (c34) as [P, 7] = (p_x, p_y, p_z, q_w, q_x, q_y, q_z), w >= 0."""
    R, p = hand_pose(np.asarray(q, np.float64).reshape(-1, 7), robot)
    return np.concatenate([p, quat_from_matrix(R)], axis=1)


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
