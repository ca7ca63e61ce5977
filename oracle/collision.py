"""World (sphere-vs-cuboid) and self collision costs and their gradients, in
float64 (oracle).

TEST INFRASTRUCTURE ONLY -- see oracle/__init__.py.

PAPER.md:86 ("Robot-environment and robot-self distance queries are utilized
in the cost function to avoid collisions"), PAPER.md:189 ("the input of
self-collision cost: out_vec, the output of collision cost: closest_pt for IKO
and closest_pt_swept for TO").  The paper gives no formula; the readings are
SURVEY.md §8(c) c11-c17 (listed in DESIGN.md §3):

  box SDF  p = R^T (c - t); u = |p| - h; sdf = ||max(u, 0)|| + min(max_k u_k, 0)
  grad sdf (world) = R (sign(p_k*) e_k*), k* = argmax u (lowest index on ties,
           sign(0) = +1) when all u_k <= 0, else R (sign(p) * max(u,0)/||max(u,0)||)
  phi = r + eta - sdf;  smooth hinge h(phi) = 0 | phi^2/(2 eta) | phi - eta/2
           on phi <= 0 | 0 < phi <= eta | phi > eta;  h' = 0 | phi/eta | 1
  world cost  = w sum_s sum_k h(phi_sk);   closest_pt_s = -w sum_k h'(phi_sk) grad sdf_sk
  swept (c17) samples p_hj = (1 - tau_j) c_h + tau_j c_{h+1}, tau_j = j/(n+1):
           cost_h += sum_j f(p_hj);  closest_pt_swept_h = grad f(c_h)
           + sum_j (1-tau_j) grad f(p_hj) + sum_j tau_j grad f(p_{h-1,j})
  self     phi_ij = r_i + r_j + eta_s - ||c_i - c_j||; cost += w h(phi_ij);
           out_vec_i -= w h'(phi_ij) (c_i - c_j)/d, out_vec_j += same;
           d = 0 -> direction (1, 0, 0).
All gradient accumulators start at +0.0, so inactive entries are +0.0.
"""
import numpy as np


def hinge(phi, eta):
    """Smooth hinge h_eta and its derivative (C^1 at 0 and eta)."""
    phi = np.asarray(phi, np.float64)
    h = np.where(phi <= 0.0, 0.0,
                 np.where(phi <= eta, phi * phi / (2.0 * eta), phi - eta / 2.0))
    dh = np.where(phi <= 0.0, 0.0, np.where(phi <= eta, phi / eta, 1.0))
    return h, dh


def box_sdf(c, R, t, h):
    """Signed distance and world-frame gradient of one oriented box.

    c [..., 3]; R [3, 3] world-from-box; t [3]; h [3].  Returns (sdf [...],
    grad [..., 3], tie [...]) where `tie` flags inside points whose top two
    face distances are within 1e-6 (gradient ambiguous, reading c16)."""
    c = np.asarray(c, np.float64)
    R = np.asarray(R, np.float64)
    p = (c - t) @ R                      # = R^T (c - t), row-vector form
    u = np.abs(p) - h
    upos = np.maximum(u, 0.0)
    outside_norm = np.sqrt(np.sum(upos * upos, axis=-1))
    umax = np.max(u, axis=-1)
    sdf = outside_norm + np.minimum(umax, 0.0)
    sgn = np.where(p >= 0.0, 1.0, -1.0)
    inside = np.all(u <= 0.0, axis=-1)
    kstar = np.argmax(u, axis=-1)        # argmax returns the lowest index on ties
    g_in = np.zeros(u.shape)
    np.put_along_axis(g_in, kstar[..., None],
                      np.take_along_axis(sgn, kstar[..., None], -1), -1)
    with np.errstate(invalid="ignore", divide="ignore"):
        g_out = sgn * upos / np.where(outside_norm > 0, outside_norm, 1.0)[..., None]
    g_local = np.where(inside[..., None], g_in, g_out)
    grad = g_local @ R.T                 # = R g_local
    us = np.sort(u, axis=-1)
    tie = inside & ((us[..., -1] - us[..., -2]) < 1e-6)
    return sdf, grad, tie


# Length scale L (metres) of the workspace and the FP32 evaluation error
# bound on a distance, used only to build per-element tolerance scales for the
# parity tests: a term whose phi lies within NEAR of 0 may be
# active on one side and inactive on the other; its derivative h' = phi/eta
# carries an absolute error of about eps * L / eta.
L_SCALE = 1.0
NEAR = 1e-6


def world_point_cost(c, radius, cuboids, eta, w):
    """f and grad f for points c [N, S, 3] of one world.

    cuboids [K, 16] float32 rows (R, t, h, pad).  Returns cost [N, S],
    grad [N, S, 3], cost scale [N, S], grad scale [N, S] and tie flags
    [N, S]."""
    N, S = c.shape[0], c.shape[1]
    cost = np.zeros((N, S))
    grad = np.zeros((N, S, 3))
    cscale = np.zeros((N, S))
    gscale = np.zeros((N, S))
    tie = np.zeros((N, S), bool)
    for k in range(cuboids.shape[0]):
        row = cuboids[k].astype(np.float64)
        R = row[0:9].reshape(3, 3)
        sdf, gs, tk = box_sdf(c, R, row[9:12], row[12:15])
        phi = radius[None, :] + eta - sdf
        hk, dhk = hinge(phi, eta)
        cost = cost + w * hk
        grad = grad + (-w * dhk)[..., None] * gs
        near = phi > -NEAR
        cscale = cscale + w * (hk + near * L_SCALE)
        gscale = gscale + w * near * (1.0 + L_SCALE / eta)
        tie |= tk & near
    return cost, grad, cscale, gscale, tie


def world_cost(c, radius, cuboids, eta, w, swept=False, n=1):
    """World collision for trajectories c [nb, H, S, 3] of ONE world (float64).

    Returns cost_pose [nb, H], grad [nb, H, S, 3] (closest_pt or
    closest_pt_swept), cost scale [nb, H], grad scale [nb, H, S], tie
    [nb, H, S]."""
    nb, H, S = c.shape[0], c.shape[1], c.shape[2]

    def point(x):
        f, g, cs, gs, t = world_point_cost(x.reshape(-1, S, 3), radius, cuboids, eta, w)
        sh = x.shape[:-2]
        return (f.reshape(sh + (S,)), g.reshape(sh + (S, 3)), cs.reshape(sh + (S,)),
                gs.reshape(sh + (S,)), t.reshape(sh + (S,)))

    f, gf, cs, gsc, tie = point(c)
    cost = f.sum(axis=-1)
    cscale = cs.sum(axis=-1)
    grad = gf.copy()
    gscale = gsc.copy()
    if swept and n > 0 and H >= 2:
        for j in range(1, n + 1):
            tau = j / (n + 1.0)
            p = (1.0 - tau) * c[:, :-1] + tau * c[:, 1:]    # segments h = 0..H-2
            fp, gp, csp, gsp, tp = point(p)
            cost[:, :-1] += fp.sum(axis=-1)
            cscale[:, :-1] += csp.sum(axis=-1)
            grad[:, :-1] += (1.0 - tau) * gp
            grad[:, 1:] += tau * gp
            gscale[:, :-1] += gsp
            gscale[:, 1:] += gsp
            tie[:, :-1] |= tp
            tie[:, 1:] |= tp
    return cost, grad, cscale, gscale, tie


def self_cost(c, radius, pairs, eta, w):
    """Self collision for poses c [N, S, 3] (float64) over the listed pairs.

    Returns cost [N], out_vec [N, S, 3], cost scale [N], grad scale [N, S]."""
    N, S = c.shape[0], c.shape[1]
    i = pairs[:, 0].astype(np.int64)
    j = pairs[:, 1].astype(np.int64)
    diff = c[:, i] - c[:, j]                           # [N, npairs, 3]
    d = np.sqrt(np.sum(diff * diff, axis=-1))
    phi = radius[i] + radius[j] + eta - d
    h, dh = hinge(phi, eta)
    cost = w * h.sum(axis=1)
    with np.errstate(invalid="ignore", divide="ignore"):
        u = diff / np.where(d > 0, d, 1.0)[..., None]
    u = np.where((d > 0)[..., None], u, np.array([1.0, 0.0, 0.0]))
    contrib = (w * dh)[..., None] * u                   # [N, npairs, 3]
    near = phi > -NEAR
    cscale = w * np.sum(h + near * L_SCALE, axis=1)
    pscale = w * near * (1.0 + L_SCALE / eta + L_SCALE / np.maximum(d, 1e-3))
    out = np.zeros((N, S, 3))
    gscale = np.zeros((N, S))
    for k in range(len(i)):                             # plain pair loop
        out[:, i[k]] -= contrib[:, k]
        out[:, j[k]] += contrib[:, k]
        gscale[:, i[k]] += pscale[:, k]
        gscale[:, j[k]] += pscale[:, k]
    return cost, out, cscale, gscale
