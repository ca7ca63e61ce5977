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
    grad [..., 3], tie [...], grad_alt [..., 3], out_norm [...]): `tie` flags
    inside points whose top two face distances are within 1e-6 (gradient
    ambiguous, reading c16) and grad_alt is the gradient with the runner-up
    face there (= grad elsewhere); out_norm = ||max(u, 0)||."""
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
    order = np.argsort(-u, axis=-1, kind="stable")
    k2 = order[..., 1]                   # the runner-up face
    g_in2 = np.zeros(u.shape)
    np.put_along_axis(g_in2, k2[..., None], np.take_along_axis(sgn, k2[..., None], -1), -1)
    with np.errstate(invalid="ignore", divide="ignore"):
        g_out = sgn * upos / np.where(outside_norm > 0, outside_norm, 1.0)[..., None]
    g_local = np.where(inside[..., None], g_in, g_out)
    grad = g_local @ R.T                 # = R g_local
    us = np.sort(u, axis=-1)
    tie = inside & ((us[..., -1] - us[..., -2]) < 1e-6)
    grad_alt = np.where(tie[..., None], g_in2 @ R.T, grad)
    return sdf, grad, tie, grad_alt, outside_norm


# Tolerance bookkeeping for the parity tests.  Besides each
# value the oracle returns
#   terms: the sum of the absolute values of the summands that make it (the
#          FP32 summation error is relative to this, not to the value), and
#   kappa: its condition number w.r.t. FP32 rounding of the evaluation, in
#          units where the FP32 error is ~ 2^-24 kappa:
#     * a term within NEAR of activation may be active on one side only, and
#       h' = phi/eta carries the absolute error of phi (~ L, the coordinate
#       magnitude, in units of 2^-24) over eta: w L / eta;
#     * the cost term h(phi) carries the error of phi: w L;
#     * an outside box gradient max(u,0)/||max(u,0)|| has a direction error
#       ~ L / ||max(u,0)||, weighted by h';
#     * a self pair's phi is computed from the pair distance d (error ~
#       d + r_i + r_j), so its h' error is w (d + r_i + r_j + eta) / eta; its
#       direction (c_i - c_j)/d is accurate to a few ulps (w h').
L_SCALE = 1.0
NEAR = 1e-6


def world_point_cost(c, radius, cuboids, eta, w):
    """f and grad f for points c [N, S, 3] of one world.

    cuboids [K, 16] float32 rows (R, t, h, pad).  Returns a dict of cost
    [N, S], grad / grad_alt [N, S, 3], cost_terms / cost_kappa [N, S],
    grad_terms / grad_kappa [N, S] (per sphere, bounding each component) and
    tie [N, S]."""
    N, S = c.shape[0], c.shape[1]
    cost = np.zeros((N, S))
    grad = np.zeros((N, S, 3))
    grad_alt = np.zeros((N, S, 3))
    cterms = np.zeros((N, S))
    ckappa = np.zeros((N, S))
    gterms = np.zeros((N, S))
    gkappa = np.zeros((N, S))
    tie = np.zeros((N, S), bool)
    for k in range(cuboids.shape[0]):
        row = cuboids[k].astype(np.float64)
        R = row[0:9].reshape(3, 3)
        sdf, gs, tk, gs_alt, onorm = box_sdf(c, R, row[9:12], row[12:15])
        phi = radius[None, :] + eta - sdf
        hk, dhk = hinge(phi, eta)
        cost = cost + w * hk
        grad = grad + (-w * dhk)[..., None] * gs
        grad_alt = grad_alt + (-w * dhk)[..., None] * gs_alt
        near = phi > -NEAR
        cterms = cterms + w * hk
        ckappa = ckappa + w * near * L_SCALE
        gterms = gterms + w * dhk
        with np.errstate(divide="ignore"):
            cond_dir = np.where(onorm > 0, L_SCALE / np.maximum(onorm, 1e-300), 0.0)
        gkappa = gkappa + w * near * (1.0 + L_SCALE / eta + dhk * cond_dir)
        tie |= tk & near
    return dict(cost=cost, grad=grad, grad_alt=grad_alt, cost_terms=cterms, cost_kappa=ckappa,
                grad_terms=gterms, grad_kappa=gkappa, tie=tie)


def world_cost(c, radius, cuboids, eta, w, swept=False, n=1):
    """World collision for trajectories c [nb, H, S, 3] of ONE world (float64).

    Returns a dict: cost [nb, H] (cost_pose), grad / grad_alt [nb, H, S, 3]
    (closest_pt or closest_pt_swept), cost_terms / cost_kappa [nb, H],
    grad_terms / grad_kappa [nb, H, S], tie [nb, H, S]."""
    nb, H, S = c.shape[0], c.shape[1], c.shape[2]

    def point(x):
        r = world_point_cost(x.reshape(-1, S, 3), radius, cuboids, eta, w)
        sh = x.shape[:-2]
        return {k: v.reshape(sh + v.shape[1:]) for k, v in r.items()}

    r0 = point(c)
    out = dict(cost=r0["cost"].sum(axis=-1), cost_terms=r0["cost_terms"].sum(axis=-1),
               cost_kappa=r0["cost_kappa"].sum(axis=-1), grad=r0["grad"].copy(),
               grad_alt=r0["grad_alt"].copy(), grad_terms=r0["grad_terms"].copy(),
               grad_kappa=r0["grad_kappa"].copy(), tie=r0["tie"].copy())
    if swept and n > 0 and H >= 2:
        for j in range(1, n + 1):
            tau = j / (n + 1.0)
            p = (1.0 - tau) * c[:, :-1] + tau * c[:, 1:]    # segments h = 0..H-2
            rp = point(p)
            for k in ("cost", "cost_terms", "cost_kappa"):
                out[k][:, :-1] += rp[k].sum(axis=-1)
            for k in ("grad", "grad_alt"):
                out[k][:, :-1] += (1.0 - tau) * rp[k]
                out[k][:, 1:] += tau * rp[k]
            for k in ("grad_terms", "grad_kappa"):
                out[k][:, :-1] += (1.0 - tau) * rp[k]
                out[k][:, 1:] += tau * rp[k]
            out["tie"][:, :-1] |= rp["tie"]
            out["tie"][:, 1:] |= rp["tie"]
    return out


def self_cost(c, radius, pairs, eta, w):
    """Self collision for poses c [N, S, 3] (float64) over the listed pairs.

    Returns a dict: cost [N], grad (out_vec) [N, S, 3], cost_terms /
    cost_kappa [N], grad_terms / grad_kappa [N, S]."""
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
    cterms = w * h.sum(axis=1)
    ckappa = w * np.sum(near * (d + radius[i] + radius[j] + eta), axis=1)
    pterms = w * dh
    pkappa = w * near * (1.0 + (d + radius[i] + radius[j] + eta) / eta)
    out = np.zeros((N, S, 3))
    gterms = np.zeros((N, S))
    gkappa = np.zeros((N, S))
    for k in range(len(i)):                             # plain pair loop
        out[:, i[k]] -= contrib[:, k]
        out[:, j[k]] += contrib[:, k]
        gterms[:, i[k]] += pterms[:, k]
        gterms[:, j[k]] += pterms[:, k]
        gkappa[:, i[k]] += pkappa[:, k]
        gkappa[:, j[k]] += pkappa[:, k]
    return dict(cost=cost, grad=out, cost_terms=cterms, cost_kappa=ckappa,
                grad_terms=gterms, grad_kappa=gkappa)
