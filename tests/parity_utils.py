"""Comparison rules GPU <-> oracle.

Every oracle value v comes with `terms` (the sum of the absolute values of
the summands that make it) and `kappa` (its condition number w.r.t. the FP32
rounding of the evaluation; oracle/collision.py documents each).  The bound is

    delta = TOL (|v| + terms) + KAPPA_ULPS 2^-24 kappa

-- the FP32 summation error is relative to `terms`; the evaluation error of a
near-active term is ~ 2^-24 kappa, with KAPPA_ULPS ulps of slack.

Packed outputs: the GPU code must lie in the code interval
[Q(v - delta), Q(v + delta)] of the oracle's double pre-quantisation value
(Q the oracle's double-input quantiser, monotone), or -- at an SDF face tie --
in that of v_alt (the runner-up face's value) and nowhere else.  Where
2 delta is below the format's step at v, the interval is at most one
neighbouring code: one step of the stored format.  `code_steps` reports the
largest distance in codes from Q(v).  FP32 outputs: |gpu - ref| <= delta + ATOL.
"""
import numpy as np

from oracle import codec

TOL = 1e-5
ATOL = 1e-7
REPORT = {}        # what -> largest err/limit (FP32) or code distance (packed), per session


def _record(what, key, value):
    name = what.split(" traj")[0]
    r = REPORT.setdefault(name, {})
    r[key] = max(r.get(key, 0.0), float(value))
KAPPA_ULPS = 16.0
EPS32 = 2.0 ** -24


def delta_of(v, terms, kappa, tol=TOL):
    v = np.asarray(v, np.float64)
    return (tol * (np.abs(v) + np.broadcast_to(terms, v.shape))
            + KAPPA_ULPS * EPS32 * np.broadcast_to(kappa, v.shape))


def signed_order(codes, E, M):
    """Map sign-magnitude codes to integers that are monotone in value."""
    t = 1 + E + M
    c = codes.astype(np.int64)
    sign = (c >> (t - 1)) & 1
    mag = c & ((1 << (t - 1)) - 1)
    return np.where(sign == 1, -mag, mag)


def _in_interval(g, v, delta, E, M, got):
    lo = codec.quantize_f64(v - delta, E, M)
    hi = codec.quantize_f64(v + delta, E, M)
    ok = (g >= signed_order(lo, E, M)) & (g <= signed_order(hi, E, M))
    # +0 / -0 are the same value: accept either sign of zero for a zero interval
    ok |= (codec.dequantize(got, E, M) == 0) & (codec.dequantize(lo, E, M) <= 0) & \
          (codec.dequantize(hi, E, M) >= 0)
    return ok


def check_codes(gpu_words, v, terms, kappa, fmt, cols, alt=None, min_exact=None, what="",
                max_steps=None):
    """Element-wise interval check of packed GPU output against oracle values.

    gpu_words [P, W] uint32, v [P, cols] float64; terms / kappa broadcastable
    to v; alt: v with the runner-up face at SDF ties (accepted as a second
    interval); max_steps: an upper bound on |code - Q(v)| (in codes) asserted
    for every element outside the tie set.  Returns (exact rate, max steps)."""
    E, M = fmt
    got = codec.unpack(np.asarray(gpu_words, np.uint32), E, M, cols)
    v = np.asarray(v, np.float64).reshape(got.shape)
    delta = delta_of(v, terms, kappa)
    g = signed_order(got, E, M)
    ok = _in_interval(g, v, delta, E, M, got)
    ref = codec.quantize_f64(v, E, M)
    steps = np.abs(g - signed_order(ref, E, M))
    tied = np.zeros(v.shape, bool)
    if alt is not None:
        alt = np.asarray(alt, np.float64).reshape(got.shape)
        tied = alt != v
        ok |= tied & _in_interval(g, alt, delta_of(alt, terms, kappa), E, M, got)
    bad = np.nonzero(~ok)
    assert ok.all(), (f"{what}: {len(bad[0])} codes outside the interval; first at "
                      f"{[b[:5] for b in bad]}: gpu={got[bad][:5]} ref={ref[bad][:5]} "
                      f"v={v[bad][:5]} delta={delta[bad][:5]}")
    zero_pair = (codec.dequantize(got, E, M) == 0) & (codec.dequantize(ref, E, M) == 0)
    steps = np.where(zero_pair | tied, 0, steps)
    max_step = int(steps.max()) if steps.size else 0
    if max_steps is not None:
        assert max_step <= max_steps, f"{what}: a code {max_step} steps from Q(v) (bound {max_steps})"
    exact = float(np.mean(got == ref))
    # largest |gpu value - v| in units of delta (the interval rule bounds it by
    # ~1 plus half a code step), and the code distance
    dv = np.abs(codec.dequantize(got, E, M).astype(np.float64) - v)
    _record(what, f"E{E}M{M} max_code_steps", max_step)
    _record(what, f"E{E}M{M} inexact_frac", 1.0 - exact)
    if M >= 23 and E == 8:
        _record(what, "E8M23 max |gpu-v|/delta", float(np.max(np.where(tied, 0, dv) / np.maximum(delta, 1e-300))) if dv.size else 0.0)
    # an exact-match rate is meaningful only when the format's step is far
    # coarser than FP32 evaluation error (M <= 10); E8M23 codes are FP32 bits
    if min_exact is not None and M <= 10:
        assert exact >= min_exact, f"{what}: only {exact:.5f} of codes exact"
    return exact, max_step


def check_close(gpu, ref, terms, what="", tol=TOL, atol=ATOL, kappa=0.0):
    """|gpu - ref| <= tol (|ref| + terms) + KAPPA_ULPS 2^-24 kappa + atol.
    Returns the largest err / limit."""
    gpu = np.asarray(gpu, np.float64)
    ref = np.asarray(ref, np.float64).reshape(gpu.shape)
    terms = np.broadcast_to(terms, ref.shape).reshape(gpu.shape)
    kappa = np.broadcast_to(kappa, ref.shape).reshape(gpu.shape)
    lim = delta_of(ref, terms, kappa, tol) + atol
    err = np.abs(gpu - ref)
    if err.size:
        _record(what, "max err/limit", np.max(err / lim))
    bad = np.nonzero(err > lim)
    assert not len(bad[0]), (f"{what}: {len(bad[0])} values out of tolerance; first "
                             f"gpu={gpu[bad][:5]} ref={ref[bad][:5]} lim={lim[bad][:5]}")
    return float(np.max(err / lim)) if err.size else 0.0


def sphere_to_elem(scale_ps, S=52):
    """[P, S] per-sphere scale -> [P, 3S] per-element scale."""
    return np.repeat(np.asarray(scale_ps), 3, axis=-1)


def world_kw(ws):
    """check_codes keyword arguments for a world stage's gradient codes."""
    return dict(terms=sphere_to_elem(ws["gterms"]), kappa=sphere_to_elem(ws["gkappa"]),
                alt=ws["v_alt"])


def self_kw(ss):
    return dict(terms=sphere_to_elem(ss["gterms"]), kappa=sphere_to_elem(ss["gkappa"]))


def cost_kw(ws, ss):
    """check_close keyword arguments for cost_pose = world + self."""
    return dict(terms=ws["cost_terms"].reshape(-1) + ss["cost_terms"].reshape(-1),
                kappa=ws["cost_kappa"].reshape(-1) + ss["cost_kappa"].reshape(-1))


def step_bound(fmt):
    """1 (one code step) for formats whose finest step, the subnormal quantum
    2^(1-bias-M), is >= 2^-10 -- every delta of these tests is far below
    half of it, so a code farther than one step from Q(v) is a bug; None for
    finer formats, where the interval rule alone applies."""
    E, M = fmt
    bias = 2 ** (E - 1) - 1
    return 1 if 1 - bias - M >= -10 else None


# FP32 forward kinematics error of a sphere centre, in units of 2^-24 L
# (7 sincos + 8 chained 3x4 products): the out_spheres of an all-E8M23
# end-to-end run differ from the oracle's by a few FP32 ulps, which the
# downstream conditioning (kappa) amplifies.
K_FK = 4.0


def e2e_kw(res, wl):
    """Tolerances of an all-E8M23 end-to-end comparison (no stage re-feeding):
    cost_traj and grad_q bounds that add the FK error (K_FK ulps of L per
    sphere centre) propagated through the gradients (for the cost) and the
    gradients' conditioning (for grad_q)."""
    from oracle.kinematics import backward_kappa
    st = res.stages
    B, H = wl.B, wl.H
    S = st["self"]["gterms"].shape[-1]
    gterms = st["world"]["gterms"] + st["self"]["gterms"]
    gkappa = st["world"]["gkappa"] + st["self"]["gkappa"]
    cterms = st["world"]["cost_terms"].reshape(-1) + st["self"]["cost_terms"].reshape(-1)
    ckappa = (st["world"]["cost_kappa"].reshape(-1) + st["self"]["cost_kappa"].reshape(-1)
              + K_FK * 1.0 * gterms.reshape(-1, S).sum(1))
    q = np.asarray(wl.q, np.float32).astype(np.float64).reshape(-1, 7)
    gq_kappa = K_FK * backward_kappa(q, gkappa.reshape(-1, S), wl.robot)
    return dict(cost_traj=dict(terms=cterms.reshape(B, H).sum(1), kappa=ckappa.reshape(B, H).sum(1)),
                cost_pose=dict(terms=cterms.reshape(B, H), kappa=ckappa.reshape(B, H)),
                grad_q=dict(terms=st["bk"]["scale"], kappa=gq_kappa))


def ik_kw(q, robot, G, w_pos, w_rot, w_b):
    """Tolerances of the N2 pose + bound terms (oracle/ikcost.py, reading c35):
    per pose, the cost's terms are its non-negative summands and its kappa
    the force |F| = 2 w_pos |p - p_g| times the hand position error (K_FK ulps
    of L) plus the torque's rotation error; per joint, the gradient's terms
    bound |z.((p - o) x F)| + |z.tau| + |bound gradient| by their factors
    (|p - o| <= 1.5 L for the Panda) and its kappa the same errors through
    the lever arm.  G [P, 12] goals (R row-major, p)."""
    from oracle.ikcost import bound_cost, pose_cost
    from oracle.kinematics import link_frames
    q = np.asarray(q, np.float64).reshape(-1, 7)
    P = q.shape[0]
    cost = np.zeros(P)
    gb = np.zeros((P, 7))
    F = np.zeros(P)
    tau = np.zeros(P)
    if w_pos or w_rot:
        c, _ = pose_cost(q, robot, G[:, :9].reshape(-1, 3, 3), G[:, 9:], w_pos, w_rot)
        cost += c
        fr = link_frames(q, robot)
        F = 2.0 * w_pos * np.linalg.norm(fr[:, 8, :3, 3] - G[:, 9:], axis=1)
        tau = np.full(P, 6.0 * w_rot)            # |2 w_rot sum_k r_k x g_k| <= 6 w_rot
    if w_b:
        c, gb = bound_cost(q, robot["q_lo"], robot["q_hi"], w_b)
        cost += c
    Lr = 1.5
    c_kappa = K_FK * (F * 1.0 + tau)
    g_terms = (Lr * F + tau)[:, None] + np.abs(gb)
    g_kappa = (K_FK * (Lr * (F + 2.0 * w_pos * 1.0) + 2.0 * tau))[:, None] + np.zeros((P, 7))
    return dict(cost=dict(terms=cost, kappa=c_kappa), grad=dict(terms=g_terms, kappa=g_kappa))
