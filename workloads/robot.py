"""Franka Panda model data: modified-DH rows, joint limits, and a synthetic
52-sphere collision table.

The paper names the robot ("Franka Panda") but gives no
kinematic constants and no sphere model; these are public datasheet values
(marked "(ext)") plus a seeded synthetic sphere table.
This module only *lists* numbers -- it computes no kinematics.

Frame convention (modified DH, Craig):
    row i (i = 1..8):  T_i = RotX(alpha_i) . TransX(a_i) . RotZ(theta_i) . TransZ(d_i)
with theta_i = q_i for the 7 joints and theta_8 = 0 for the fixed flange row.
Frame 0 is the base, frames 1..7 are the joint frames, the flange is frame 8
and the *hand* frame is flange . RotZ(hand_rz).  Spheres are attached to
"links" 0..8 where link 8 means the hand frame (the flange itself carries no
spheres).
"""
import math

import numpy as np

# (a_i, d_i, alpha_i) per modified-DH row; rows 1..7 are the joints, row 8 the
# fixed flange.  SURVEY.md §8(c) step 2 (ext).
DH_A = (0.0, 0.0, 0.0, 0.0825, -0.0825, 0.0, 0.088, 0.0)
DH_D = (0.333, 0.0, 0.316, 0.0, 0.384, 0.0, 0.0, 0.107)
DH_ALPHA = (0.0, -math.pi / 2, math.pi / 2, math.pi / 2, -math.pi / 2,
            math.pi / 2, math.pi / 2, 0.0)
HAND_RZ = -math.pi / 4          # hand = flange . RotZ(-pi/4)
Q_LO = (-2.8973, -1.7628, -2.8973, -3.0718, -2.8973, -0.0175, -2.8973)
Q_HI = (2.8973, 1.7628, 2.8973, -0.0698, 2.8973, 3.7525, 2.8973)
READY_POSE = (0.0, -math.pi / 4, 0.0, -3 * math.pi / 4, 0.0, math.pi / 2,
              math.pi / 4)
ROBOT_FRAMES = 9                # sphere-carrying frames: link0..link7, hand

# Sphere placement: per link, a list of (start, end, count) segments given in
# that link's own frame (metres).  Counts per link are [4,5,5,6,6,8,5,4,9]
# = 52.  The segments roughly follow the Panda's
# link bodies; they are synthetic data, not a measured model.
_SEGMENTS = {
    0: [((-0.04, 0.0, 0.05), (0.0, 0.0, 0.25), 4)],
    1: [((0.0, 0.0, -0.19), (0.0, -0.03, -0.02), 5)],
    2: [((0.0, -0.03, 0.03), (0.0, -0.21, 0.0), 5)],
    3: [((0.0, 0.0, -0.13), (0.08, 0.0, -0.03), 6)],
    4: [((0.0, 0.02, 0.0), (-0.08, 0.13, 0.0), 6)],
    5: [((0.0, 0.10, -0.27), (0.0, 0.05, -0.13), 8)],
    6: [((0.0, 0.0, -0.03), (0.06, 0.0, -0.02), 5)],
    7: [((0.0, 0.0, 0.0), (0.0, 0.0, 0.06), 4)],
    8: [((0.0, -0.07, 0.06), (0.0, 0.07, 0.06), 5),
        ((0.0, -0.04, 0.12), (0.0, 0.04, 0.12), 2),
        ((0.0, -0.04, 0.17), (0.0, 0.04, 0.17), 2)],
}
SPHERES_PER_LINK = (4, 5, 5, 6, 6, 8, 5, 4, 9)
SPHERE_SEED = 0x5EED0052
R_MIN, R_MAX = 0.04, 0.08
JITTER = 0.01


def _sphere_table():
    rng = np.random.Generator(np.random.Philox(key=SPHERE_SEED))
    links, xyzr = [], []
    for link in range(ROBOT_FRAMES):
        for (p0, p1, n) in _SEGMENTS[link]:
            p0 = np.asarray(p0, np.float64)
            p1 = np.asarray(p1, np.float64)
            for k in range(n):
                f = 0.5 if n == 1 else k / (n - 1)
                c = p0 + f * (p1 - p0) + rng.uniform(-JITTER, JITTER, 3)
                r = rng.uniform(R_MIN, R_MAX)
                links.append(link)
                xyzr.append([c[0], c[1], c[2], r])
    links = np.asarray(links, np.int32)
    xyzr = np.asarray(xyzr, np.float64).astype(np.float32)
    assert tuple(np.bincount(links, minlength=ROBOT_FRAMES)) == SPHERES_PER_LINK
    return links, xyzr


def _load_pairs():
    """Self-collision pair list, written once by
    scripts/make_self_pairs.py (which calls only oracle/).  Returns None when
    the data file has not been generated yet."""
    import json
    import os
    path = os.path.join(os.path.dirname(__file__), "data", "panda_self_pairs.json")
    if not os.path.exists(path):
        return None
    with open(path) as f:
        d = json.load(f)
    return np.asarray(d["pairs"], np.uint16).reshape(-1, 2)


def candidate_pairs(links):
    """All sphere pairs on links whose index differs by >= 2 (c18), before
    ready-pose pruning.  Pure index bookkeeping."""
    out = []
    n = len(links)
    for i in range(n):
        for j in range(i + 1, n):
            if abs(int(links[i]) - int(links[j])) >= 2:
                out.append((i, j))
    return np.asarray(out, np.uint16).reshape(-1, 2)


def panda_robot(pairs=None):
    """The robot model as plain arrays.

    Keys: dh_a, dh_d, dh_alpha (8 rows, float64 -- both sides cast as they
    need), hand_rz, q_lo, q_hi, sphere_link [52] int32, sphere_xyzr [52,4]
    float32 (local offset + radius), pairs [n_pairs,2] uint16.
    """
    links, xyzr = _sphere_table()
    if pairs is None:
        pairs = _load_pairs()
        if pairs is None:
            pairs = candidate_pairs(links)
    return {
        "dh_a": np.asarray(DH_A, np.float64),
        "dh_d": np.asarray(DH_D, np.float64),
        "dh_alpha": np.asarray(DH_ALPHA, np.float64),
        "hand_rz": float(HAND_RZ),
        "q_lo": np.asarray(Q_LO, np.float64),
        "q_hi": np.asarray(Q_HI, np.float64),
        "sphere_link": links,
        "sphere_xyzr": xyzr,
        "pairs": np.asarray(pairs, np.uint16).reshape(-1, 2),
    }
