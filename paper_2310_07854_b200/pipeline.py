"""Full-pipeline success-rate evaluator.

PAPER.md:78 / :162 -- planning is IK optimisation (IKO) followed by
trajectory optimisation (TO) from seeds; the format search constrains the
planner's success rate per environment.  The real planner
(geometric planner, attempts, MotionBenchMaker) is out of scope; this is the
closest in-scope substitute, built only from the library's own calls
(readings c38-c40):

  c38  IK: every problem's goal solved from `ik_seeds` random configurations
       by `TrajOpt` on the IKO workload (pose + bound + discrete world + self
       costs); the problem's IK solution is its best seed, accepted when that
       cost is <= ik_tol;
  c39  TO: `to_seeds` trajectories per problem from a fixed start (the ready
       pose) to the IK solution, linear in joint space plus seeded noise on
       the interior waypoints; the first and last waypoints are frozen
       (`fixed` mask of vapr_lbfgs_step); cost = swept world + self;
  c40  success: IK accepted and at least one TO seed with cost exactly 0
       (every swept sample and pair clear by the activation distance eta);
  c44  attempts ("... with retry attempts"): a problem that fails
       is planned again, up to `attempts` times in all, each attempt with
       fresh IK seeds (uniform in the joint limits) and fresh TO noise, both
       keyed by (attempt, problem); it succeeds if any attempt does.

Both stages optimise with the candidate format tuple; their results are then
validated at full precision (an all-E8M23 rollout of the final IK seeds and
TO trajectories): the IK acceptance and the zero-cost test use the FP32 costs,
so a coarse out_spheres format cannot hide a collision from the success
criterion (SPEC.md: validation at 32-bit regardless of the formats).  The
seed choices (best IK seed) are the planner's own, made on its candidate-
format costs.  Rates are per environment, as the search expects (search.Memo).
"""
import numpy as np
import torch

from .optimize import TrajOpt
from .rollout import Rollout


class PipelineEvaluator:
    def __init__(self, problems_per_env=4, ik_seeds=64, to_seeds=8, H=32, ik_iters=40,
                 to_iters=40, ik_tol=1e-3, device=0, attempts=1):
        from workloads import config_iko, make_workload, READY_POSE
        from workloads.configs import FP32, DEFAULT_PARAMS
        self.ik_iters, self.to_iters, self.ik_tol = ik_iters, to_iters, ik_tol
        self.attempts = int(attempts)
        self.H, self.to_seeds = H, to_seeds
        self.ik_wl = config_iko(problems_per_env=problems_per_env, seeds=ik_seeds, formats=FP32)
        P = len(self.ik_wl.envs)
        self.n_problems, self.ik_seeds = P, ik_seeds
        ids = list(range(P))
        to_params = dict(DEFAULT_PARAMS)
        to_params.update({k: 0.0 for k in ("w_pose_pos", "w_pose_rot", "w_bound")})
        self.to_wl = make_workload("pipeline_to", list(self.ik_wl.envs), ids, to_seeds, H, FP32,
                                   params=to_params, cuboids=self.ik_wl.cuboids,
                                   offsets=self.ik_wl.world_offsets, salt=11)
        self.envs = list(self.ik_wl.envs)
        fixed = np.zeros((H, 7), np.uint8)
        fixed[0] = fixed[H - 1] = 1
        self.ik = TrajOpt(self.ik_wl, device=device)
        self.to = TrajOpt(self.to_wl, device=device, fixed=fixed)
        # full-precision validation of the optimised IK seeds / TO trajectories
        self.ik_val = Rollout(self.ik_wl, device=device, formats=FP32)
        self.to_val = Rollout(self.to_wl, device=device, formats=FP32)
        self.start = np.asarray(READY_POSE, np.float32)
        # seeded interior noise of the TO seeds (c39), fixed once
        rng = np.random.Generator(np.random.Philox(key=0x90E5))
        self.noise = rng.normal(0.0, 0.15, (P, to_seeds, H, 7)).astype(np.float32)
        self.noise[:, :, 0] = 0.0
        self.noise[:, :, H - 1] = 0.0
        self.noise[:, 0] = 0.0                      # seed 0: the straight line
        self.q_lo = np.asarray(self.ik_wl.robot["q_lo"], np.float32)
        self.q_hi = np.asarray(self.ik_wl.robot["q_hi"], np.float32)
        self.last = None

    def _attempt_inputs(self, attempt):
        """IK seeds and TO noise of an attempt (attempt 0: the workload's)."""
        if attempt == 0:
            return None, self.noise
        P, S, H = self.n_problems, self.ik_seeds, self.H
        rng = np.random.Generator(np.random.Philox(key=0xA77E0000 + attempt))
        q = (self.q_lo + rng.random((P * S, 1, 7)) * (self.q_hi - self.q_lo)).astype(np.float32)
        noise = rng.normal(0.0, 0.15, (P, self.to_seeds, H, 7)).astype(np.float32)
        noise[:, :, 0] = 0.0
        noise[:, :, H - 1] = 0.0
        noise[:, 0] = 0.0
        return q, noise

    def evaluate(self, formats):
        """Success rate per environment for one format tuple (slot order)."""
        P = self.n_problems
        self.ik.set_formats(formats)
        self.to.set_formats(formats)
        ok = np.zeros(P, bool)
        used = np.zeros(P, np.int32)
        for att in range(self.attempts):
            q_ik, noise = self._attempt_inputs(att)
            res = self._plan(q_ik, noise)
            newly = ~ok & res["success"]
            used[~ok] = att + 1
            ok |= newly
            if att == 0:
                self.last = res
            if ok.all():
                break
        self.last = dict(self.last, success=ok, attempts_used=used)
        rates = {}
        for e in sorted(set(self.envs)):
            sel = np.array([x == e for x in self.envs])
            rates[e] = float(ok[sel].mean())
        return rates

    def _plan(self, q_ik, noise):
        """One planning attempt for every problem: IK, then TO to the IK
        solution, both validated at full precision."""
        P, S, H = self.n_problems, self.ik_seeds, self.H
        self.ik.reset(q_ik)
        for _ in range(self.ik_iters):
            self.ik.step()
        ik_cost = self.ik.cost.cpu().numpy().reshape(P, S)
        best = np.argmin(ik_cost, axis=1)
        ik_fp32 = self._validate(self.ik_val, self.ik.x).reshape(P, S)
        ik_ok = ik_fp32[np.arange(P), best] <= self.ik_tol
        goals = self.ik.x.cpu().numpy().reshape(P, S, 7)[np.arange(P), best]
        f = (np.arange(H, dtype=np.float32) / (H - 1))[None, None, :, None]
        q0 = self.start[None, None, None, :] + f * (goals[:, None, None, :] - self.start[None, None, None, :])
        q0 = q0 + noise
        q0[:, :, 0] = self.start
        q0[:, :, H - 1] = goals[:, None, :]
        self.to.reset(q0.reshape(-1, H, 7))
        for _ in range(self.to_iters):
            self.to.step()
        to_cost = self.to.cost.cpu().numpy().reshape(P, self.to_seeds)
        to_fp32 = self._validate(self.to_val, self.to.x).reshape(P, self.to_seeds)
        ok = ik_ok & np.any(to_fp32 <= 0.0, axis=1)
        return dict(ik_cost=ik_cost[np.arange(P), best], ik_cost_fp32=ik_fp32[np.arange(P), best],
                    ik_ok=ik_ok, to_cost=to_cost, to_cost_fp32=to_fp32, success=ok, goals=goals)

    @staticmethod
    def _validate(roll, x):
        """Per-trajectory cost of the optimised variables x at all-E8M23."""
        roll.q.copy_(x.reshape(roll.q.shape))
        roll.run()
        return roll.results()["cost_traj"].copy()

    def __call__(self, configs):
        return [self.evaluate(c) for c in configs]
