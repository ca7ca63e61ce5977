"""Seeded TO-seed trajectories ("Trajectories").

q_a, q_b ~ U(joint limits shrunk by 10 %), q[h] = q_a + h/(H-1) (q_b - q_a)
+ N(0, 0.05 rad), clamped to the limits; emitted as float32 (the dtype the
C-ABI consumes).  This smooth straight-line-plus-noise shape stands in for
CuRobo's IK/GP-seeded trajectories.
"""
import numpy as np

from .scenes import _key


def make_trajectories(key, n_seeds, H, q_lo, q_hi, noise=0.05):
    q_lo = np.asarray(q_lo, np.float64)
    q_hi = np.asarray(q_hi, np.float64)
    rng = np.random.Generator(np.random.Philox(key=_key(key, 0x7A7A)))
    mid = 0.5 * (q_lo + q_hi)
    half = 0.5 * (q_hi - q_lo) * 0.9
    qa = rng.uniform(mid - half, mid + half, (n_seeds, 7))
    qb = rng.uniform(mid - half, mid + half, (n_seeds, 7))
    if H > 1:
        f = (np.arange(H, dtype=np.float64) / (H - 1))[None, :, None]
    else:
        f = np.zeros((1, 1, 1))
    q = qa[:, None, :] + f * (qb - qa)[:, None, :]
    q = q + rng.normal(0.0, noise, q.shape)
    q = np.clip(q, q_lo, q_hi)
    return q.astype(np.float32)
