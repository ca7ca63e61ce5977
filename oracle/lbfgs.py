"""oracle/lbfgs.py -- TEST INFRASTRUCTURE (see oracle/__init__.py).

The optimiser steps around the rollout: PAPER.md:162,
"(1) Given N, step scales of step direction (see (7)) ... (6) Use line search
to pick one from N. (7) Lastly, compute step direction (L-BFGS) and buffer
updates", and PAPER.md:86, "L-BFGS solver is a gradient-based optimization
that computes the step direction towards a local optima of a cost function".
The paper gives no formulas; the classic two-loop recursion is written out
here in float64, with the readings of DESIGN.md §3 (c29-c33):

  c29  history: FIFO of the m most recent (s, y) pairs, s = x_new - x_old,
       y = g_new - g_old, kept only when s.y > curvature_eps;
  c30  direction: two-loop recursion, initial scaling gamma = s.y / y.y of
       the newest pair, gamma = 1 with an empty history;
  c31  line search: candidates x + s_n d for the N scales; the argmin, ties
       to the smallest scale; no candidate strictly below cost(x) -> x kept,
       scale 0;
  c32  after a step without improvement: with a non-empty history the
       history is cleared and the next direction is -g; with an empty one the
       rejected direction is shrunk tenfold (backtracking across iterations).
       SPEC.md is silent; keeping the history (or -g at a fixed scale set)
       would repeat the same rejected candidates forever;
  c33  defaults m = 10, scales {0.01, 0.03, 0.1, 0.3, 1.0}, curvature_eps =
       1e-10.

Every function works on one batch item (vectors as 1-D float64 arrays); the
batched GPU kernels are compared item by item.
"""
import numpy as np

DEFAULT_M = 10
DEFAULT_SCALES = (0.01, 0.03, 0.1, 0.3, 1.0)
CURVATURE_EPS = 1e-10


class History:
    """The (s, y, rho) FIFO of one batch item (c29)."""

    def __init__(self, m=DEFAULT_M):
        self.m = m
        self.s, self.y, self.rho = [], [], []

    def push(self, s, y, eps=CURVATURE_EPS):
        """Append (s, y) if s.y > eps (dropping the oldest beyond m); returns
        whether the pair was kept."""
        sy = float(np.dot(s, y))
        if not sy > eps:
            return False
        self.s.append(np.array(s, np.float64))
        self.y.append(np.array(y, np.float64))
        self.rho.append(1.0 / sy)
        if len(self.s) > self.m:
            self.s.pop(0)
            self.y.pop(0)
            self.rho.pop(0)
        return True

    def clear(self):
        self.s, self.y, self.rho = [], [], []

    def __len__(self):
        return len(self.s)


def two_loop_direction(hist, g):
    """d = -H g by the two-loop recursion (c30), newest pair last."""
    q = np.array(g, np.float64)
    k = len(hist)
    alpha = [0.0] * k
    for i in range(k - 1, -1, -1):                 # newest to oldest
        alpha[i] = hist.rho[i] * float(np.dot(hist.s[i], q))
        q = q - alpha[i] * hist.y[i]
    if k:
        gamma = float(np.dot(hist.s[-1], hist.y[-1])) / float(np.dot(hist.y[-1], hist.y[-1]))
    else:
        gamma = 1.0
    r = gamma * q
    for i in range(k):                             # oldest to newest
        beta = hist.rho[i] * float(np.dot(hist.y[i], r))
        r = r + hist.s[i] * (alpha[i] - beta)
    return -r


def line_search_select(cost_x, cand_costs):
    """Index of the chosen candidate (c31), or -1 when none strictly improves
    on cost_x.  cand_costs[n] is the cost at x + scale_n d, scales ascending."""
    best = -1
    best_c = cost_x
    for n, c in enumerate(cand_costs):
        if c < best_c:                             # strict: ties keep the smaller scale
            best, best_c = n, c
    return best


def lbfgs_iterate(x, g, cost, d, hist, cost_and_grad, scales=DEFAULT_SCALES):
    """One iteration of steps (1), (6), (7) around cost_and_grad (steps
    (2)-(5)): evaluate the N candidates, select, update the history, new
    direction.  Returns (x, g, cost, d, chosen)."""
    cands = [x + s * d for s in scales]
    evals = [cost_and_grad(c) for c in cands]
    n = line_search_select(cost, [e[0] for e in evals])
    if n < 0:                                      # c32
        if len(hist):
            hist.clear()
            return x, g, cost, two_loop_direction(hist, g), -1
        return x, g, cost, 0.1 * d, -1
    x_new, (c_new, g_new) = cands[n], evals[n]
    hist.push(x_new - x, g_new - g)
    return x_new, g_new, c_new, two_loop_direction(hist, g_new), n


def minimize(x0, cost_and_grad, iters, scales=DEFAULT_SCALES, m=DEFAULT_M):
    """Run `iters` iterations from x0; returns (x, cost, grad, cost history)."""
    x = np.array(x0, np.float64)
    c, g = cost_and_grad(x)
    hist = History(m)
    d = two_loop_direction(hist, g)
    costs = [c]
    for _ in range(iters):
        x, g, c, d, _ = lbfgs_iterate(x, g, c, d, hist, cost_and_grad, scales)
        costs.append(c)
    return x, c, g, costs
