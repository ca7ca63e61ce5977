"""Synthetic MotionBenchMaker-like cuboid scenes ("Worlds").

The paper's eight Panda environments (Table II rows) are
known by name only; their geometry is not published.  Each environment here is
a hand-written template of K oriented cuboids in front of the robot
(x in [0.3, 0.8] m) with the K of SURVEY.md §8(d), and every planning problem
jitters the whole scene by +-5 cm and +-15 deg of yaw (seeded).

A cuboid is stored as 16 float32: R (3x3 row-major, world-from-box rotation),
t (box centre, world), h (half extents), pad.  This is the layout the C-ABI
`vapr_cuboid` declares (include/vapr.h).  Building R from an angle is input
synthesis, not method arithmetic.
"""
import math

import numpy as np

# name -> list of (centre xyz, half extents xyz, yaw_deg)
_T = {
    "table_pick": [
        ((0.60, 0.00, 0.10), (0.20, 0.40, 0.02), 0.0),
        ((0.55, 0.15, 0.17), (0.03, 0.03, 0.05), 20.0),
        ((0.62, -0.20, 0.17), (0.04, 0.04, 0.05), 0.0),
    ],
    "table_under_pick": [
        ((0.60, 0.00, 0.40), (0.20, 0.40, 0.02), 0.0),
        ((0.45, 0.35, 0.19), (0.02, 0.02, 0.19), 0.0),
        ((0.45, -0.35, 0.19), (0.02, 0.02, 0.19), 0.0),
        ((0.60, 0.05, 0.06), (0.04, 0.04, 0.06), 30.0),
    ],
    "box": [
        ((0.60, 0.00, 0.05), (0.15, 0.15, 0.01), 0.0),
        ((0.75, 0.00, 0.15), (0.01, 0.15, 0.10), 0.0),
        ((0.45, 0.00, 0.15), (0.01, 0.15, 0.10), 0.0),
        ((0.60, 0.15, 0.15), (0.15, 0.01, 0.10), 0.0),
        ((0.60, -0.15, 0.15), (0.15, 0.01, 0.10), 0.0),
    ],
    "box_flipped": [
        ((0.60, 0.00, 0.45), (0.15, 0.15, 0.01), 0.0),
        ((0.75, 0.00, 0.35), (0.01, 0.15, 0.10), 0.0),
        ((0.60, 0.15, 0.35), (0.15, 0.01, 0.10), 0.0),
        ((0.60, -0.15, 0.35), (0.15, 0.01, 0.10), 0.0),
        ((0.60, 0.00, 0.05), (0.20, 0.25, 0.02), 0.0),
    ],
    "cage": [
        ((0.40, 0.30, 0.30), (0.015, 0.015, 0.30), 0.0),
        ((0.40, -0.30, 0.30), (0.015, 0.015, 0.30), 0.0),
        ((0.80, 0.30, 0.30), (0.015, 0.015, 0.30), 0.0),
        ((0.80, -0.30, 0.30), (0.015, 0.015, 0.30), 0.0),
        ((0.60, 0.00, 0.62), (0.22, 0.32, 0.02), 0.0),
        ((0.60, 0.00, 0.02), (0.22, 0.32, 0.02), 0.0),
    ],
    "bookshelf_small": [
        ((0.70, 0.30, 0.35), (0.15, 0.01, 0.35), 0.0),
        ((0.70, -0.30, 0.35), (0.15, 0.01, 0.35), 0.0),
        ((0.70, 0.00, 0.01), (0.15, 0.30, 0.01), 0.0),
        ((0.70, 0.00, 0.35), (0.15, 0.30, 0.01), 0.0),
        ((0.70, 0.00, 0.69), (0.15, 0.30, 0.01), 0.0),
        ((0.85, 0.00, 0.35), (0.01, 0.30, 0.35), 0.0),
        ((0.65, 0.10, 0.42), (0.03, 0.03, 0.06), 10.0),
    ],
    "bookshelf_thin": [
        ((0.75, 0.25, 0.40), (0.10, 0.005, 0.40), 0.0),
        ((0.75, -0.25, 0.40), (0.10, 0.005, 0.40), 0.0),
        ((0.75, 0.00, 0.005), (0.10, 0.25, 0.005), 0.0),
        ((0.75, 0.00, 0.30), (0.10, 0.25, 0.005), 0.0),
        ((0.75, 0.00, 0.60), (0.10, 0.25, 0.005), 0.0),
        ((0.86, 0.00, 0.40), (0.005, 0.25, 0.40), 0.0),
        ((0.72, -0.08, 0.36), (0.02, 0.02, 0.05), 0.0),
    ],
    "bookshelf_tall": [
        ((0.70, 0.30, 0.55), (0.15, 0.01, 0.55), 0.0),
        ((0.70, -0.30, 0.55), (0.15, 0.01, 0.55), 0.0),
        ((0.70, 0.00, 0.01), (0.15, 0.30, 0.01), 0.0),
        ((0.70, 0.00, 0.25), (0.15, 0.30, 0.01), 0.0),
        ((0.70, 0.00, 0.50), (0.15, 0.30, 0.01), 0.0),
        ((0.70, 0.00, 0.75), (0.15, 0.30, 0.01), 0.0),
        ((0.70, 0.00, 1.00), (0.15, 0.30, 0.01), 0.0),
        ((0.85, 0.00, 0.55), (0.01, 0.30, 0.55), 0.0),
        ((0.64, -0.12, 0.31), (0.03, 0.03, 0.05), 25.0),
    ],
}

# Environment order = Table II row order (PAPER.md:295-302 / 305-312).
ENVIRONMENTS = ("bookshelf_small", "bookshelf_tall", "bookshelf_thin", "box",
                "box_flipped", "cage", "table_pick", "table_under_pick")
ENV_K = {name: len(_T[name]) for name in _T}


def _rz(deg):
    a = math.radians(deg)
    c, s = math.cos(a), math.sin(a)
    return np.array([[c, -s, 0.0], [s, c, 0.0], [0.0, 0.0, 1.0]])


def make_world(env, key, jitter=True):
    """Cuboids of one problem of environment `env` as float32 [K, 16].

    key: integer tuple for the Philox stream; with jitter=False the template
    itself is returned (used by the hand-checkable tests)."""
    tmpl = _T[env]
    if jitter:
        rng = np.random.Generator(np.random.Philox(key=_key(key, 0xC0B0)))
        shift = rng.uniform(-0.05, 0.05, 3)
        yaw = rng.uniform(-15.0, 15.0)
    else:
        shift = np.zeros(3)
        yaw = 0.0
    anchor = np.array([0.6, 0.0, 0.0])
    Rs = _rz(yaw)
    out = np.zeros((len(tmpl), 16), np.float64)
    for k, (c, h, yd) in enumerate(tmpl):
        c = np.asarray(c, np.float64)
        R = Rs @ _rz(yd)
        t = anchor + Rs @ (c - anchor) + shift
        out[k, 0:9] = R.reshape(-1)
        out[k, 9:12] = t
        out[k, 12:15] = h
    return out.astype(np.float32)


def make_worlds(envs, keys, jitter=True):
    """Concatenate the worlds of several problems.

    Returns (cuboids float32 [sum K, 16], offsets int32 [n+1])."""
    worlds = [make_world(e, k, jitter) for e, k in zip(envs, keys)]
    offsets = np.zeros(len(worlds) + 1, np.int32)
    offsets[1:] = np.cumsum([w.shape[0] for w in worlds])
    cub = np.concatenate(worlds, 0) if worlds else np.zeros((0, 16), np.float32)
    return cub, offsets


def _key(key, salt):
    """Fold an integer tuple into a 128-bit Philox key (two uint64 words)."""
    if isinstance(key, int):
        key = (key,)
    h = 0x9E3779B97F4A7C15 ^ salt
    for k in key:
        h = (h * 0x100000001B3 ^ (int(k) & 0xFFFFFFFFFFFFFFFF)) & 0xFFFFFFFFFFFFFFFF
        h ^= h >> 29
    return [h, salt & 0xFFFFFFFFFFFFFFFF]
