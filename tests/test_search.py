"""Host-side VaPr search driver: pins from PAPER.md §V-A
and SPEC.md's vapr-search examples, with mock evaluators (CPU only)."""
import io
import itertools
import json
import random

import pytest

from paper_2310_07854_b200 import search as S


def threshold_evaluator(thresholds, envs=("e0", "e1")):
    """Feasible iff every slot's width >= its hidden threshold."""
    calls = []

    def ev(configs):
        out = []
        for c in configs:
            calls.append(c)
            ok = all(S.bits(f) >= t for f, t in zip(c, thresholds))
            out.append({e: 1.0 if ok else 0.5 for e in envs})
        return out
    ev.calls = calls
    return ev


def test_space_counts_and_total_bits():
    assert len(S.enumerate_formats()) == 21
    assert S.total_bits(((8, 23),) * 5) == 160
    assert S.total_bits(((5, 10), (4, 3), (2, 1), (2, 2), (4, 3))) == 41
    assert S.total_bits(((5, 10), (3, 2), (2, 2), (4, 3), (4, 3))) == 43
    assert S.reduce_space([13, 4, 5, 4, 4])[1] == 555660
    assert round(S.reduce_space([13, 4, 5, 4, 4])[2], 2) == 7.35
    assert S.reduce_space([15, 4, 4, 4, 4])[1] == 583443
    assert S.reduce_space([4] * 5)[1] == 4084101
    assert [f for f in S.reduce_space([16, 4, 4, 4, 4])[0][0]] == [(5, 10), (8, 7), (8, 23)]


@pytest.mark.parametrize("thr", [16, 4, 5, 13, 32, 9])
def test_binary_search_finds_threshold(thr):
    ev = threshold_evaluator((thr, 4, 4, 4, 4))
    memo = S.Memo(ev, {"e0": 1.0, "e1": 1.0})
    r = S.per_tensor_binary_search(0, memo)
    assert r.min_bits == thr and S.bits(r.witness) == thr
    assert len(r.probes) <= 7 and r.monotone


def test_nsga2_hidden_thresholds_reach_36():
    # SPEC.md:488 / 608: thresholds (16,5,4,5,6) -> 36 within 500 evaluations
    ev = threshold_evaluator((16, 5, 4, 5, 6))
    memo = S.Memo(ev, {"e0": 1.0, "e1": 1.0})
    res = S.vapr_search(memo, budget=500, seed=3)
    assert res["minima"] == [16, 5, 4, 5, 6]
    assert res["best"].feasible and res["best"].total_bits == 36
    assert res["evaluations"] - res["phase1_evaluations"] <= 500


def test_nondominated_sort_matches_bruteforce():
    rng = random.Random(0)
    for _ in range(30):
        n = rng.randrange(1, 50)
        pop = []
        for i in range(n):
            feas = rng.random() < 0.5
            pop.append(S.Trial(i, (), {}, 0.0 if feas else rng.choice([0.1, 0.2, 0.5]), feas,
                               rng.choice([20, 30, 40, 50]), "x"))
        fronts = S.nondominated_sort(pop)
        assert sorted(itertools.chain(*fronts)) == list(range(n))
        for k, fr in enumerate(fronts):
            for i in fr:
                # nobody in this or a later front dominates i; someone in front k-1 does
                later = list(itertools.chain(*fronts[k:]))
                assert not any(S.constrained_dominates(pop[j], pop[i]) for j in later)
                if k > 0:
                    assert any(S.constrained_dominates(pop[j], pop[i]) for j in fronts[k - 1])


def test_operators():
    rng = random.Random(1)
    space = [S.formats_at_or_above(4)] * 5
    g = [1, 2, 3, 4, 5]
    assert S.uniform_crossover(rng, g, g) == (g, g)
    m = S.random_reset_mutation(rng, g, space, p_m=1.0)
    assert all(0 <= m[k] < len(space[k]) for k in range(5))
    pop = [S.Trial(i, (), {}, 0.0, True, b, "x") for i, b in enumerate([10, 20])]
    assert all(v == float("inf") for v in S.crowding_distance(pop, [0, 1]).values())
    single = [[(8, 23)]] * 5
    memo = S.Memo(threshold_evaluator((4,) * 5), {"e0": 1.0, "e1": 1.0})
    best = S.nsga2_search(single, memo, budget=500)
    assert best.total_bits == 160 and memo.evaluations == 1


def test_search_is_deterministic_and_logs():
    logs = []
    for _ in range(2):
        buf = io.StringIO()
        memo = S.Memo(threshold_evaluator((16, 5, 4, 5, 6)), {"e0": 1.0, "e1": 1.0}, buf)
        S.vapr_search(memo, budget=200, seed=7)
        logs.append([json.loads(l) for l in buf.getvalue().splitlines()])
    strip = [[{k: v for k, v in t.items() if k != "seconds"} for t in lg] for lg in logs]
    assert strip[0] == strip[1]
    assert all(t["config"][0].startswith("E") for t in logs[0])
    best_bits = min(t["total_bits"] for t in logs[0] if t["feasible"])
    assert best_bits == 36
