"""Pins of oracle/lbfgs.py (readings c29-c33):
SPEC.md's worked line-search examples, the two-loop recursion's closed form on
a diagonal quadratic, convergence on a convex quadratic and on Rosenbrock, the
monotone-cost invariant, and the history rules."""
import numpy as np
import pytest

from oracle import lbfgs as L


def test_empty_history_is_steepest_descent():
    g = np.array([1.0, -2.0, 3.5])
    assert np.array_equal(L.two_loop_direction(L.History(), g), -g)


def test_line_search_examples():
    # SPEC.md:311 f(x) = x^2, x = 1, d = -1, scales {0.5, 1.0, 1.5} -> 1.0 (cost 0)
    f = lambda x: x * x
    scales = (0.5, 1.0, 1.5)
    costs = [f(1.0 - s) for s in scales]
    assert L.line_search_select(f(1.0), costs) == 1
    # direction 0: every candidate equals cost(x), none strictly better -> unchanged
    assert L.line_search_select(1.0, [1.0, 1.0, 1.0]) == -1
    # all worse -> unchanged
    assert L.line_search_select(1.0, [2.0, 3.0]) == -1
    # ties go to the smaller scale
    assert L.line_search_select(5.0, [4.0, 3.0, 3.0]) == 1


def test_diagonal_secant_pairs_give_newton_direction():
    """Pairs (e_i, D e_i) on f = 1/2 x^T D x: the two-loop recursion returns
    -D^{-1} g exactly (BFGS is exact on each coordinate once its pair is in)."""
    D = np.array([2.0, 5.0, 0.5])
    h = L.History(m=10)
    for i in range(3):
        e = np.zeros(3)
        e[i] = 1.0
        assert h.push(e, D * e)
    g = np.array([0.3, -1.1, 2.0])
    np.testing.assert_allclose(L.two_loop_direction(h, g), -g / D, rtol=1e-14, atol=0)


def test_curvature_rejection_and_fifo():
    h = L.History(m=2)
    assert not h.push(np.array([1.0, 0.0]), np.array([-1.0, 0.0]))      # s.y < 0
    assert not h.push(np.array([1e-6, 0.0]), np.array([1e-6, 0.0]))    # s.y = 1e-12 <= eps
    assert len(h) == 0
    for k in range(3):
        assert h.push(np.array([1.0, k]), np.array([1.0, 0.0]))
    assert len(h) == 2 and h.s[0][1] == 1.0 and h.s[1][1] == 2.0       # oldest dropped


def quadratic(n=10, seed=0):
    rng = np.random.default_rng(seed)
    A = rng.normal(size=(n, n))
    Q = A @ A.T + n * np.eye(n)
    b = rng.normal(size=n)
    return (lambda x: (0.5 * x @ Q @ x - b @ x, Q @ x - b)), np.linalg.solve(Q, b)


def rosenbrock(x):
    a, b = x
    c = (1 - a) ** 2 + 100 * (b - a * a) ** 2
    g = np.array([-2 * (1 - a) - 400 * a * (b - a * a), 200 * (b - a * a)])
    return c, g


def test_convex_quadratic_converges():
    """grad-norm < 1e-6 on a 10-D convex quadratic within 50 iterations."""
    f, xstar = quadratic()
    x, c, g, costs = L.minimize(np.zeros(10), f, 50)
    assert np.linalg.norm(g) < 1e-6
    np.testing.assert_allclose(x, xstar, atol=1e-6)
    assert all(b <= a for a, b in zip(costs, costs[1:]))


def test_rosenbrock_converges():
    """|x - (1, 1)| < 1e-3 on 2-D Rosenbrock within 500 iterations."""
    x, c, g, costs = L.minimize(np.array([-1.2, 1.0]), rosenbrock, 500)
    assert np.linalg.norm(x - 1.0) < 1e-3
    assert all(b <= a for a, b in zip(costs, costs[1:]))


def test_at_minimum_stays():
    f, xstar = quadratic(4, 3)
    c0, g0 = f(xstar)
    x, g, c, d, n = L.lbfgs_iterate(xstar, g0, c0, -g0, L.History(), f)
    # at the minimum no candidate is strictly better (up to rounding of the
    # tiny gradient step): x stays or moves by a negligible amount, cost never rises
    assert c <= c0
    np.testing.assert_allclose(x, xstar, atol=1e-12)


def test_singleton_scale_is_damped_step():
    f, _ = quadratic(5, 1)
    x0 = np.ones(5)
    c0, g0 = f(x0)
    d0 = -g0
    x, g, c, d, n = L.lbfgs_iterate(x0, g0, c0, d0, L.History(), f, scales=(0.01,))
    assert n == 0
    np.testing.assert_array_equal(x, x0 + 0.01 * d0)


@pytest.mark.parametrize("seed", range(3))
def test_no_improvement_clears_history_then_backtracks(seed):
    f, _ = quadratic(4, seed)
    x0 = np.ones(4)
    c0, g0 = f(x0)
    h = L.History()
    h.push(np.ones(4), np.ones(4))
    # an ascent direction: every candidate is worse -> history cleared, d = -g
    x, g, c, d, n = L.lbfgs_iterate(x0, g0, c0, g0, h, f)
    assert n == -1 and len(h) == 0
    np.testing.assert_array_equal(x, x0)
    np.testing.assert_array_equal(d, -g0)
    # with an empty history a rejected direction is shrunk tenfold
    x, g, c, d2, n = L.lbfgs_iterate(x0, g0, c0, 1e3 * g0, h, f)
    assert n == -1
    np.testing.assert_allclose(d2, 1e2 * g0, rtol=1e-15)
