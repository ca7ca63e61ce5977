"""Batched trajectory optimisation around the rollout.

PAPER.md:162, the 7-step iteration: "(1) Given N, step scales of step
direction (see (7)). (2) Compute kinematics. (3) Compute cost functions ...
(4) Aggregating the costs. (5) Compute backward ... (6) Use line search to
pick one from N. (7) Lastly, compute step direction (L-BFGS) and buffer
updates."  Steps (2)-(5) are one `vapr_cost_grad` over the N x B line-search
batch (every candidate's cost AND gradient, so the chosen one needs no second
evaluation); (1) is `vapr_lbfgs_candidates`, (6)+(7) `vapr_lbfgs_step`.
Every array stays on the device; one iteration is three library calls with no
host synchronisation.  Readings c29-c33.
"""
import dataclasses

import numpy as np
import torch

from . import binding as vb
from .rollout import Rollout

DEFAULT_SCALES = (0.01, 0.03, 0.1, 0.3, 1.0)


class TrajOpt:
    """L-BFGS over every trajectory of a workload (x[b] = its H x 7 joint
    values), cost = the rollout cost (world swept + self collision)."""

    def __init__(self, workload, scales=DEFAULT_SCALES, m=10, curvature_eps=1e-10, device=0,
                 formats=None, fixed=None, sparse=False):
        self.wl = workload
        self.scales = tuple(float(s) for s in scales)
        self.N = len(self.scales)
        self.m = int(m)
        self.eps = float(curvature_eps)
        self.B, self.H = workload.B, workload.H
        self.D = 7 * self.H
        # the iterate and its cost / gradient live in the base rollout's buffers
        self.base = Rollout(workload, device=device, formats=formats, sparse=sparse)
        cand = dataclasses.replace(workload, q=np.tile(workload.q, (self.N, 1, 1)),
                                   world_idx=np.tile(workload.world_idx, self.N))
        self.lines = Rollout(cand, device=device, formats=formats, sparse=sparse)
        dev = self.base.device
        B, D, m = self.B, self.D, self.m
        self.d = torch.zeros(B * D, dtype=torch.float32, device=dev)
        self.hist_s = torch.zeros(B * m * D, dtype=torch.float32, device=dev)
        self.hist_y = torch.zeros(B * m * D, dtype=torch.float32, device=dev)
        self.hist_rho = torch.zeros(B * m, dtype=torch.float32, device=dev)
        self.hist_count = torch.zeros(B, dtype=torch.int32, device=dev)
        self.hist_head = torch.zeros(B, dtype=torch.int32, device=dev)
        self.chosen = torch.zeros(B, dtype=torch.int32, device=dev)
        # frozen coordinates (D-vector of bools shared by all items), e.g.
        # the first and last waypoint of every trajectory (N4)
        self.fixed = None
        if fixed is not None:
            fx = np.asarray(fixed, np.uint8).reshape(-1)
            assert fx.size == D
            self.fixed = torch.from_numpy(fx).to(dev)

    @property
    def x(self):
        return self.base.q.view(-1)

    @property
    def g(self):
        return self.base.grad_q.view(-1)

    @property
    def cost(self):
        return self.base.cost_traj

    def set_formats(self, formats):
        self.base.set_formats(formats)
        self.lines.set_formats(formats)

    def reset(self, q=None):
        """Start from q (default: the workload's trajectories): cost and
        gradient at x0, empty histories, d = -g."""
        if q is not None:
            self.base.q.copy_(torch.as_tensor(q, dtype=torch.float32).reshape(self.base.q.shape))
        else:
            self.base.q.copy_(torch.from_numpy(np.ascontiguousarray(self.wl.q)))
        self.base.run()
        if self.fixed is not None:           # gradient over the free coordinates only
            self.g.view(self.B, self.D).mul_((self.fixed == 0).to(self.g.dtype)[None, :])
        self.d.copy_(self.g).neg_()
        self.hist_count.zero_()
        self.hist_head.zero_()

    def step(self, stream=None):
        """One iteration: candidates, their rollout cost + gradient, line
        search, history and direction update (all on the device)."""
        vb.vapr_lbfgs_candidates(self.x, self.d, self.B, self.D, self.scales,
                                 self.lines.q.view(-1), stream=stream)
        self.lines.run(stream=stream)
        vb.vapr_lbfgs_step(self.B, self.D, self.scales, self.lines.cost_traj,
                           self.lines.grad_q.view(-1), self.x, self.g, self.cost, self.d,
                           self.hist_s, self.hist_y, self.hist_rho, self.hist_count,
                           self.hist_head, self.chosen, self.m, self.eps, fixed=self.fixed,
                           stream=stream)

    def run(self, iters):
        """reset() then `iters` iterations; returns the per-iteration mean cost."""
        self.reset()
        means = [float(self.cost.mean())]
        for _ in range(iters):
            self.step()
            means.append(float(self.cost.mean()))
        return means
