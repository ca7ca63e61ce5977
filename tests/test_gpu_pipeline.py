"""N4 on the GPU: the full-pipeline success evaluator
(IKO -> seeded TO with frozen endpoints -> success) built from the library's
calls (readings c38-c40), and the frozen-coordinate mask of vapr_lbfgs_step
it relies on."""
import numpy as np
import pytest
import torch

pytestmark = pytest.mark.gpu


@pytest.fixture(scope="module")
def ev():
    if not torch.cuda.is_available():
        pytest.skip("needs a GPU")
    from paper_2310_07854_b200.pipeline import PipelineEvaluator
    return PipelineEvaluator(problems_per_env=1, ik_seeds=32, to_seeds=4, H=16, ik_iters=25,
                             to_iters=20)


def test_pipeline_rates_deterministic_and_consistent(ev):
    from workloads.configs import FORMAT_SETS
    cfg = FORMAT_SETS["43bit"]
    a = ev.evaluate(cfg)
    last_a = {k: np.copy(v) for k, v in ev.last.items()}
    b = ev.evaluate(cfg)
    assert a == b                                   # the whole pipeline is deterministic
    assert set(a) == set(ev.envs) and all(0.0 <= v <= 1.0 for v in a.values())
    for k in last_a:
        assert np.array_equal(last_a[k], ev.last[k])
    # success <=> IK accepted (at full precision) and a TO seed collision-free
    # at full precision
    ok = ev.last["ik_ok"] & np.any(ev.last["to_cost_fp32"] <= 0.0, axis=1)
    assert np.array_equal(ok, ev.last["success"])
    assert np.array_equal(ev.last["ik_ok"], ev.last["ik_cost_fp32"] <= ev.ik_tol)


def test_pipeline_endpoints_frozen(ev):
    from workloads.configs import FP32
    ev.evaluate(FP32)
    H = ev.H
    x = ev.to.x.cpu().numpy().reshape(ev.n_problems, ev.to_seeds, H, 7)
    assert np.array_equal(x[:, :, 0], np.broadcast_to(ev.start, x[:, :, 0].shape))
    assert np.array_equal(x[:, :, H - 1],
                          np.broadcast_to(ev.last["goals"][:, None, :], x[:, :, H - 1].shape))
    # the stored gradient is 0 on the frozen coordinates
    g = ev.to.g.cpu().numpy().reshape(ev.n_problems, ev.to_seeds, H, 7)
    assert np.all(g[:, :, 0] == 0.0) and np.all(g[:, :, H - 1] == 0.0)
    # TO never raised any seed's cost above its start (monotone optimiser)
    assert np.all(np.isfinite(ev.last["to_cost"]))


def test_pipeline_as_search_evaluator(ev):
    """The evaluator plugs into the search driver's memo (rates per env)."""
    import io
    from paper_2310_07854_b200 import search as S
    from workloads.configs import FP32
    targets = {e: 0.0 for e in sorted(set(ev.envs))}
    memo = S.Memo(ev, targets, io.StringIO())
    (trial,) = memo.run([FP32], "pipeline")
    assert trial.feasible and set(trial.rates) == set(targets)


def test_pipeline_validation_is_full_precision(ev):
    """The success criterion uses all-E8M23 costs of the optimised variables:
    with all-E8M23 formats they equal the optimiser's own costs bit for bit;
    with a coarse out_spheres format a collision the quantised geometry hides
    still fails the problem; and the validated TO costs agree with the oracle
    rollout (oracle/rollout.py, all-E8M23) of the same trajectories."""
    from oracle import rollout as orc
    from parity_utils import check_close, e2e_kw
    from workloads.configs import FP32
    import dataclasses
    ev.evaluate(FP32)
    assert np.array_equal(ev.last["to_cost"].view(np.uint32), ev.last["to_cost_fp32"].view(np.uint32))
    ev.evaluate(((2, 1),) + FP32[1:])                # E2M1 sphere positions
    ok = ev.last["ik_ok"] & np.any(ev.last["to_cost_fp32"] <= 0.0, axis=1)
    assert np.array_equal(ok, ev.last["success"])
    x = ev.to.x.cpu().numpy().reshape(-1, ev.H, 7)
    wl = dataclasses.replace(ev.to_wl, q=np.ascontiguousarray(x, np.float32), formats=FP32)
    res = orc.rollout_workload(wl)
    kw = e2e_kw(res, wl)
    check_close(ev.last["to_cost_fp32"].reshape(-1), res.cost_traj, what="pipeline TO cost (fp32)",
                **kw["cost_traj"])


def test_pipeline_attempts():
    """PAPER.md:78 retry attempts (reading c44): more attempts never lose a
    success, the attempt counts are within the budget, deterministic."""
    if not torch.cuda.is_available():
        pytest.skip("needs a GPU")
    from paper_2310_07854_b200.pipeline import PipelineEvaluator
    from workloads.configs import FORMAT_SETS
    kw = dict(problems_per_env=1, ik_seeds=16, to_seeds=4, H=16, ik_iters=15, to_iters=15)
    one = PipelineEvaluator(attempts=1, **kw)
    three = PipelineEvaluator(attempts=3, **kw)
    cfg = FORMAT_SETS["43bit"]
    r1 = one.evaluate(cfg)
    r3 = three.evaluate(cfg)
    s1, s3 = one.last["success"], three.last["success"]
    assert np.all(s3 >= s1)                        # attempt 1 is the same plan
    assert all(r3[e] >= r1[e] for e in r1)
    used = three.last["attempts_used"]
    assert used.min() >= 1 and used.max() <= 3
    assert np.all(used[s3 & ~s1] >= 2)
    assert three.evaluate(cfg) == r3
