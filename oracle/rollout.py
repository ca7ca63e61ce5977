"""The VaPr rollout cost + gradient dataflow, stage by stage (oracle).

TEST INFRASTRUCTURE ONLY -- see oracle/__init__.py.

PAPER.md:162 (one iteration: "(2) Compute kinematics. (3) Compute cost
functions ... (4) Aggregating the costs. (5) Compute backward")
(the five large tensors) and PAPER.md:227 (quantize -> dequantize "at each
kernel invocation").  Quantisation points (reading c19): out_spheres at the FK
store, closest_pt[_swept] and out_vec at their producers' stores,
grad_out_spheres after aggregation and before BK.  Costs stay FP32/double.

Every stage consumes and produces *packed words* in the layout of
oracle.codec.pack, so that each CUDA stage can be fed exactly the same packed
inputs (parity contract 2-3).  Each stage also returns its
double-precision pre-quantisation values and per-element tolerance scales.
"""
from dataclasses import dataclass

import numpy as np

from .ikcost import bound_cost, pose_cost

from . import codec
from .kinematics import sphere_centers, backward, backward_terms_abs
from .collision import world_cost, self_cost

SLOT_OS, SLOT_GOS, SLOT_OV, SLOT_CP, SLOT_CPS = range(5)


def _cols(robot):
    return 3 * len(robot["sphere_link"])


def quantize_rows(v, fmt):
    """double [P, cols] -> packed words with ONE rounding from the double."""
    E, M = fmt
    return codec.pack(codec.quantize_f64(v, E, M), E, M)


def decode_rows(words, fmt, cols):
    E, M = fmt
    return codec.dequantize_packed(words, E, M, cols).astype(np.float64)


def fk_stage(q, robot, fmt_os):
    """q [P, 7] float32 -> (out_spheres words, pre-quant c [P, 3S])."""
    c = sphere_centers(np.asarray(q, np.float32).astype(np.float64).reshape(-1, 7), robot)
    v = c.reshape(c.shape[0], -1)
    return quantize_rows(v, fmt_os), v


def world_stage(os_words, fmt_os, world_idx, cuboids, offsets, robot, B, H,
                eta, w, swept, n, fmt_out):
    """World collision on packed out_spheres.  Returns a dict with cost
    [B, H], cost_terms / cost_kappa [B, H], words (closest_pt[_swept]), v and
    v_alt [P, 3S] (v_alt: the runner-up face at SDF ties), gterms / gkappa
    [P, S] and tie [P, S] (tolerance bookkeeping: oracle/collision.py)."""
    S = len(robot["sphere_link"])
    c = decode_rows(os_words, fmt_os, 3 * S).reshape(B, H, S, 3)
    radius = robot["sphere_xyzr"][:, 3].astype(np.float64)
    keys_bh = ("cost", "cost_terms", "cost_kappa")
    keys_bhs = ("grad_terms", "grad_kappa")
    acc = {k: np.zeros((B, H)) for k in keys_bh}
    acc.update({k: np.zeros((B, H, S)) for k in keys_bhs})
    acc["grad"] = np.zeros((B, H, S, 3))
    acc["grad_alt"] = np.zeros((B, H, S, 3))
    acc["tie"] = np.zeros((B, H, S), bool)
    world_idx = np.asarray(world_idx)
    for wi in np.unique(world_idx):
        sel = np.nonzero(world_idx == wi)[0]
        cub = cuboids[offsets[wi]:offsets[wi + 1]]
        r = world_cost(c[sel], radius, cub, eta, w, swept=bool(swept), n=n)
        for k in acc:
            acc[k][sel] = r[k]
    v = acc["grad"].reshape(B * H, 3 * S)
    return dict(cost=acc["cost"], cost_terms=acc["cost_terms"], cost_kappa=acc["cost_kappa"],
                words=quantize_rows(v, fmt_out), v=v,
                v_alt=acc["grad_alt"].reshape(B * H, 3 * S),
                gterms=acc["grad_terms"].reshape(B * H, S), gkappa=acc["grad_kappa"].reshape(B * H, S),
                tie=acc["tie"].reshape(B * H, S))


def self_stage(os_words, fmt_os, robot, eta, w, fmt_ov):
    S = len(robot["sphere_link"])
    c = decode_rows(os_words, fmt_os, 3 * S).reshape(-1, S, 3)
    radius = robot["sphere_xyzr"][:, 3].astype(np.float64)
    r = self_cost(c, radius, robot["pairs"], eta, w)
    v = r["grad"].reshape(r["grad"].shape[0], -1)
    return dict(cost=r["cost"], cost_terms=r["cost_terms"], cost_kappa=r["cost_kappa"],
                words=quantize_rows(v, fmt_ov), v=v, gterms=r["grad_terms"], gkappa=r["grad_kappa"])


def aggregate_stage(cp_words, fmt_cp, ov_words, fmt_ov, fmt_gos, cols):
    """grad_out_spheres = dequant(closest_pt[_swept]) + dequant(out_vec),
    quantised to t_gos.  The sum is exact in double;
    terms = |a| + |b| bounds the FP32 sum's rounding."""
    a = decode_rows(cp_words, fmt_cp, cols)
    b = decode_rows(ov_words, fmt_ov, cols)
    v = a + b
    return dict(words=quantize_rows(v, fmt_gos), v=v, terms=np.abs(a) + np.abs(b))


def bk_stage(q, gos_words, fmt_gos, robot):
    S = len(robot["sphere_link"])
    q64 = np.asarray(q, np.float32).astype(np.float64).reshape(-1, 7)
    g = decode_rows(gos_words, fmt_gos, 3 * S).reshape(-1, S, 3)
    return dict(grad_q=backward(q64, g, robot),
                scale=backward_terms_abs(q64, g, robot))


@dataclass
class RolloutResult:
    os_words: np.ndarray
    cp_words: np.ndarray            # closest_pt or closest_pt_swept
    ov_words: np.ndarray
    gos_words: np.ndarray
    cost_pose: np.ndarray           # [B, H] world + self
    cost_traj: np.ndarray           # [B]
    grad_q: np.ndarray              # [B, H, 7]
    stages: dict


def ik_terms(q, world_idx, robot, params, goals, H):
    """N2 (PAPER.md:162 step (3)): pose + bound cost [P] and their joint
    gradient [P, 7] (oracle/ikcost.py), or None when both weights are 0."""
    wp, wr, wb = (float(params.get(k, 0.0)) for k in ("w_pose_pos", "w_pose_rot", "w_bound"))
    if wp == 0.0 and wr == 0.0 and wb == 0.0:
        return None
    q64 = np.asarray(q, np.float32).astype(np.float64).reshape(-1, 7)
    cost = np.zeros(q64.shape[0])
    grad = np.zeros_like(q64)
    if wp != 0.0 or wr != 0.0:
        gi = np.repeat(np.asarray(world_idx), H)
        G = np.asarray(goals, np.float32).astype(np.float64)[gi]
        c, g = pose_cost(q64, robot, G[:, :9].reshape(-1, 3, 3), G[:, 9:], wp, wr)
        cost += c
        grad += g
    if wb != 0.0:
        c, g = bound_cost(q64, robot["q_lo"], robot["q_hi"], wb)
        cost += c
        grad += g
    return cost, grad


def rollout(q, world_idx, cuboids, offsets, robot, params, formats, goals=None):
    """Full vapr_cost_grad dataflow: FK -> world (discrete or swept) -> self ->
    aggregate -> BK, plus the IKO pose / bound terms when
    their weights are non-zero (N2).  formats in slot order (os, gos, ov, cp,
    cps)."""
    q = np.asarray(q, np.float32)
    B, H = q.shape[0], q.shape[1]
    cols = _cols(robot)
    swept = bool(params["swept"])
    f_os, f_gos, f_ov = formats[SLOT_OS], formats[SLOT_GOS], formats[SLOT_OV]
    f_cp = formats[SLOT_CPS] if swept else formats[SLOT_CP]
    os_words, v_os = fk_stage(q.reshape(-1, 7), robot, f_os)
    ws = world_stage(os_words, f_os, world_idx, cuboids, offsets, robot, B, H,
                     params["eta_world"], params["w_world"], swept,
                     params["sweep_steps"], f_cp)
    ss = self_stage(os_words, f_os, robot, params["eta_self"], params["w_self"], f_ov)
    ag = aggregate_stage(ws["words"], f_cp, ss["words"], f_ov, f_gos, cols)
    bk = bk_stage(q.reshape(-1, 7), ag["words"], f_gos, robot)
    cost_pose = ws["cost"] + ss["cost"].reshape(B, H)
    grad_q = bk["grad_q"].reshape(B, H, 7)
    ik = ik_terms(q, world_idx, robot, params, goals, H)
    if ik is not None:
        cost_pose = cost_pose + ik[0].reshape(B, H)
        grad_q = grad_q + ik[1].reshape(B, H, 7)
    return RolloutResult(os_words, ws["words"], ss["words"], ag["words"],
                         cost_pose, cost_pose.sum(axis=1), grad_q,
                         dict(fk=v_os, world=ws, self=ss, aggregate=ag, bk=bk, ik=ik))


def rollout_workload(wl, formats=None):
    return rollout(wl.q, wl.world_idx, wl.cuboids, wl.world_offsets, wl.robot,
                   wl.params, formats if formats is not None else wl.formats,
                   goals=getattr(wl, "goals", None))
