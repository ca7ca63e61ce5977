"""Pins for the composed rollout oracle: the chain rule end to end (finite
differences of the total cost w.r.t. q), quantisation points, and the
fake-quant invariant."""
import numpy as np

from oracle import codec
from oracle.collision import world_cost, self_cost
from oracle.kinematics import sphere_centers, backward
from oracle.rollout import rollout_workload, SLOT_OS, SLOT_GOS, SLOT_OV, SLOT_CPS
from workloads import config2, config4
from workloads.configs import FORMAT_SETS


def _total_cost_double(q, wl):
    """Unquantised double chain: sum over trajectories of world + self."""
    B, H = q.shape[0], q.shape[1]
    S = 52
    c = sphere_centers(q.reshape(-1, 7), wl.robot).reshape(B, H, S, 3)
    r = wl.robot["sphere_xyzr"][:, 3].astype(np.float64)
    p = wl.params
    tot = 0.0
    for b in range(B):
        w = wl.world_idx[b]
        cub = wl.cuboids[wl.world_offsets[w]:wl.world_offsets[w + 1]]
        tot += world_cost(c[b:b + 1], r, cub, p["eta_world"], p["w_world"],
                          swept=True, n=p["sweep_steps"])["cost"].sum()
    tot += self_cost(c.reshape(-1, S, 3), r, wl.robot["pairs"], p["eta_self"], p["w_self"])["cost"].sum()
    return tot


def test_chain_rule_finite_differences():
    wl = config4(problems_per_env=1, seeds=1, H=4)
    q = wl.q.astype(np.float64)
    B, H = q.shape[:2]
    S = 52
    # analytic: world (swept) + self gradients on c, then BK
    c = sphere_centers(q.reshape(-1, 7), wl.robot).reshape(B, H, S, 3)
    r = wl.robot["sphere_xyzr"][:, 3].astype(np.float64)
    g = np.zeros((B, H, S, 3))
    for b in range(B):
        w = wl.world_idx[b]
        cub = wl.cuboids[wl.world_offsets[w]:wl.world_offsets[w + 1]]
        g[b] = world_cost(c[b:b + 1], r, cub, 0.025, 1.0, swept=True, n=1)["grad"][0]
    g += self_cost(c.reshape(-1, S, 3), r, wl.robot["pairs"], 0.01, 1.0)["grad"].reshape(B, H, S, 3)
    assert np.abs(g).sum() > 0, "workload should have active terms"
    an = backward(q.reshape(-1, 7), g.reshape(-1, S, 3), wl.robot).reshape(B, H, 7)
    h = 1e-6
    rng = np.random.default_rng(0)
    for _ in range(12):
        b, t, j = rng.integers(B), rng.integers(H), rng.integers(7)
        qp, qm = q.copy(), q.copy()
        qp[b, t, j] += h
        qm[b, t, j] -= h
        fd = (_total_cost_double(qp, wl) - _total_cost_double(qm, wl)) / (2 * h)
        assert abs(fd - an[b, t, j]) <= 1e-5 * (1 + abs(fd)), (b, t, j, fd, an[b, t, j])


def test_fp32_rollout_close_to_double_chain():
    wl = config2()
    res = rollout_workload(wl, FORMAT_SETS["fp32"])
    q = wl.q.astype(np.float64)
    tot = _total_cost_double(q, wl)
    assert abs(res.cost_traj.sum() - tot) <= 1e-5 * (1 + abs(tot))
    # out_spheres codes at E8M23 are the FP32 bits of the double centres
    c = sphere_centers(q.reshape(-1, 7), wl.robot).reshape(wl.poses, -1)
    np.testing.assert_array_equal(res.os_words, c.astype(np.float32).view(np.uint32))


def test_quantisation_points_and_fake_quant():
    wl = config2()
    f = wl.formats
    res = rollout_workload(wl)
    st = res.stages
    cols = 156
    # out_spheres: one rounding of the double FK value
    np.testing.assert_array_equal(
        res.os_words, codec.pack(codec.quantize_f64(st["fk"], *f[SLOT_OS]), *f[SLOT_OS]))
    # grad_out_spheres = Q(dequant(cps) + dequant(ov)) (aggregation, PAPER.md:162 (4))
    g = (codec.dequantize_packed(res.cp_words, *f[SLOT_CPS], cols).astype(np.float64)
         + codec.dequantize_packed(res.ov_words, *f[SLOT_OV], cols))
    np.testing.assert_array_equal(res.gos_words, codec.pack(codec.quantize_f64(g, *f[SLOT_GOS]), *f[SLOT_GOS]))
    # fake-quant identity: the dequantised stored tensor equals the error-injected value
    v = st["self"]["v"].astype(np.float32)
    same = st["self"]["v"] == v.astype(np.float64)       # values exactly representable in FP32
    deq = codec.dequantize_packed(res.ov_words, *f[SLOT_OV], cols)
    fq = codec.fake_quant(v, *f[SLOT_OV])
    np.testing.assert_array_equal(deq[same], fq[same])
    # sparsity: the gradient tensors are mostly exact zeros
    assert (deq == 0).mean() > 0.8
    assert np.all(np.isfinite(res.grad_q))
