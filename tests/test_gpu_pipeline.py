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
    # success <=> IK accepted and a collision-free TO seed
    ok = ev.last["ik_ok"] & np.any(ev.last["to_cost"] <= 0.0, axis=1)
    assert np.array_equal(ok, ev.last["success"])


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
