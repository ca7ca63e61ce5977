"""Panda forward and backward kinematics in float64 (oracle).

TEST INFRASTRUCTURE ONLY -- see oracle/__init__.py.

FK ("Robot forward kinematics turns joint configuration into the
Cartesian coordinate of the end effector"; "The output of forward
kinematics: out_spheres"): modified DH, T_i = RotX(alpha_i) TransX(a_i)
RotZ(theta_i) TransZ(d_i) (reading c21); frames
F_0 = I, F_i = F_{i-1} T_i (i = 1..8, row 8 the fixed flange), hand =
F_8 RotZ(hand_rz); sphere centre c_s = F_link(s) [o_s; 1].

BK (PAPER.md:162 step (5) "Compute backward for the above steps in the reverse
sequence"; "the input of backward kinematics: grad_out_spheres"):
grad_q_j = sum_{s: link(s) >= j} z_j . ((c_s - o_j) x g_s), with z_j / o_j the
z axis / origin of joint frame j and c_s the *recomputed exact* FK centre
(reading c20), SURVEY.md §8(c) step 7.
"""
import numpy as np


def _rotx(a):
    c, s = np.cos(a), np.sin(a)
    T = np.zeros(np.shape(a) + (4, 4))
    T[..., 0, 0] = 1.0
    T[..., 1, 1] = c
    T[..., 1, 2] = -s
    T[..., 2, 1] = s
    T[..., 2, 2] = c
    T[..., 3, 3] = 1.0
    return T


def _rotz(a):
    c, s = np.cos(a), np.sin(a)
    T = np.zeros(np.shape(a) + (4, 4))
    T[..., 0, 0] = c
    T[..., 0, 1] = -s
    T[..., 1, 0] = s
    T[..., 1, 1] = c
    T[..., 2, 2] = 1.0
    T[..., 3, 3] = 1.0
    return T


def _trans(x, y, z):
    T = np.eye(4)
    T[0, 3], T[1, 3], T[2, 3] = x, y, z
    return T


def link_frames(q, robot):
    """q [P, 7] -> frames [P, 9, 4, 4]: index 0 = base, 1..7 = joint frames,
    8 = hand.  (The flange frame is an intermediate only.)"""
    q = np.asarray(q, np.float64).reshape(-1, 7)
    P = q.shape[0]
    a, d, al = robot["dh_a"], robot["dh_d"], robot["dh_alpha"]
    F = np.zeros((P, 9, 4, 4))
    cur = np.broadcast_to(np.eye(4), (P, 4, 4)).copy()
    F[:, 0] = cur
    for i in range(8):                          # DH rows 1..8
        theta = q[:, i] if i < 7 else np.zeros(P)
        T = (_rotx(al[i]) @ _trans(a[i], 0.0, 0.0))[None] @ _rotz(theta) @ _trans(0.0, 0.0, d[i])[None]
        cur = cur @ T
        if i < 7:
            F[:, i + 1] = cur
    F[:, 8] = cur @ _rotz(robot["hand_rz"])[None]   # hand = flange . RotZ
    return F


def sphere_centers(q, robot):
    """q [P, 7] -> exact sphere centres c [P, S, 3] (float64)."""
    F = link_frames(q, robot)
    link = robot["sphere_link"]
    o = np.concatenate([robot["sphere_xyzr"][:, :3].astype(np.float64),
                        np.ones((len(link), 1))], 1)          # [S, 4]
    Fs = F[:, link]                                           # [P, S, 4, 4]
    c = np.einsum("psij,sj->psi", Fs, o)
    return c[:, :, :3]


def flange_pose(q, robot):
    """Flange frame [P, 4, 4] (used only by the closed-form pins)."""
    F = link_frames(q, robot)
    return F[:, 7] @ _trans(0.0, 0.0, robot["dh_d"][7])[None]


def backward(q, g, robot):
    """grad_q [P, 7] from sphere gradients g [P, S, 3] (float64 in/out).

    Plain definition: for each joint j = 1..7 and each sphere on a link >= j,
    z_j . ((c_s - o_j) x g_s)."""
    q = np.asarray(q, np.float64).reshape(-1, 7)
    g = np.asarray(g, np.float64).reshape(q.shape[0], -1, 3)
    F = link_frames(q, robot)
    c = sphere_centers(q, robot)
    link = robot["sphere_link"]
    out = np.zeros((q.shape[0], 7))
    for j in range(1, 8):
        z = F[:, j, :3, 2]                                    # [P, 3]
        o = F[:, j, :3, 3]
        sel = link >= j
        r = c[:, sel] - o[:, None, :]
        cr = np.cross(r, g[:, sel])
        out[:, j - 1] = np.einsum("pi,psi->p", z, cr)
    return out


def backward_terms_abs(q, g, robot):
    """sum over spheres of |z_j . ((c_s - o_j) x g_s)| -- the scale used by
    the norm-relative FP32 tolerance."""
    q = np.asarray(q, np.float64).reshape(-1, 7)
    g = np.asarray(g, np.float64).reshape(q.shape[0], -1, 3)
    F = link_frames(q, robot)
    c = sphere_centers(q, robot)
    link = robot["sphere_link"]
    out = np.zeros((q.shape[0], 7))
    for j in range(1, 8):
        z = F[:, j, :3, 2]
        o = F[:, j, :3, 3]
        sel = link >= j
        r = c[:, sel] - o[:, None, :]
        # |z.(r x g)| <= |r||g|: bound each term by its factors so that the
        # FP32 evaluation error (relative to the factors) is covered.
        out[:, j - 1] = np.sum(np.linalg.norm(r, axis=-1) *
                               np.linalg.norm(g[:, sel], axis=-1), axis=1)
    return out


def backward_kappa(q, kappa, robot):
    """sum over spheres of |c_s - o_j| kappa_s: the condition number of joint
    j's gradient when each sphere gradient g_s carries an FP32 evaluation
    error ~ 2^-24 kappa_s (the lever arm times that error; parity-test
    tolerance bookkeeping)."""
    q = np.asarray(q, np.float64).reshape(-1, 7)
    kappa = np.asarray(kappa, np.float64).reshape(q.shape[0], -1)
    F = link_frames(q, robot)
    c = sphere_centers(q, robot)
    link = robot["sphere_link"]
    out = np.zeros((q.shape[0], 7))
    for j in range(1, 8):
        o = F[:, j, :3, 3]
        sel = link >= j
        r = c[:, sel] - o[:, None, :]
        out[:, j - 1] = np.sum(np.linalg.norm(r, axis=-1) * kappa[:, sel], axis=1)
    return out
