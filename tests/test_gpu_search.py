"""The VaPr search driver on the real GPU evaluator:
GpuProxyEvaluator runs one batched vapr_cost_grad per candidate on a frozen
config-5-shaped problem batch (small here) and the driver's output must be
feasible, deterministic and never worse than the all-E8M23 baseline."""
import io
import json

import pytest

torch = pytest.importorskip("torch")

from paper_2310_07854_b200 import search as S  # noqa: E402
from workloads import config5  # noqa: E402

pytestmark = pytest.mark.gpu


@pytest.fixture(scope="module")
def evaluator():
    if not torch.cuda.is_available():
        pytest.skip("needs a GPU")
    wl = config5(problems_per_env=2, seeds=4)
    return S.GpuProxyEvaluator(wl, 4)


def test_reference_config_is_perfect(evaluator):
    (rates,) = evaluator([(S.FP32,) * 5])
    assert rates and all(v == 1.0 for v in rates.values())


def test_rates_are_fractions_and_deterministic(evaluator):
    cfgs = [((2, 1),) * 5, ((5, 10), (4, 3), (2, 2), (4, 3), (4, 3))]
    a = evaluator(cfgs)
    b = evaluator(cfgs)
    assert a == b
    for rates in a:
        assert all(0.0 <= v <= 1.0 for v in rates.values())


def test_search_on_gpu_evaluator(evaluator):
    def run():
        log = io.StringIO()
        targets = {e: 1.0 for e in sorted(set(evaluator.envs))}
        memo = S.Memo(evaluator, targets, log)
        res = S.vapr_search(memo, budget=40, pop_size=8, seed=3)
        return res, log.getvalue()

    r1, log1 = run()
    r2, log2 = run()
    best = r1["best"]
    assert best.feasible and best.total_bits <= 160
    assert r1["minima"] == r2["minima"]
    assert best.config == r2["best"].config and best.total_bits == r2["best"].total_bits
    # every logged trial is a JSON line with the config and its rates
    lines = [json.loads(x) for x in log1.splitlines() if x.strip()]
    assert len(lines) == r1["evaluations"]
    # the chosen config really is feasible on a fresh evaluation
    (rates,) = evaluator([best.config])
    assert all(v >= 1.0 for v in rates.values())
