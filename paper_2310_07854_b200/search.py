"""VaPr format search: Phase-1 per-tensor binary search,
search-space reduction, and a constrained NSGA-II over the reduced space, with
a GPU evaluator built on libvapr.

PAPER.md:247-252 (§V-A): "We use binary search to find the minimum
reduced-precision data format for each tensor while keeping the other tensors
in the FP32 data format"; "The per-tensor search results can thus eliminate
all the FP data formats that are less than the corresponding result";
"We adopt NSGA-II ... The objective of the black-box optimizer is to minimize
the total number of bitwidths of the large tensors while satisfying the success
rate constraints"; "sampling 500 points with NSGA-II".
Operators and defaults follow SPEC.md's vapr-search module (population 20,
25 generations, p_c = 0.9, p_m = 0.2, binary tournament, uniform crossover,
random-reset mutation, constraint-dominated sorting, memoised evaluations).

The paper's success rate needs the full CuRobo planner and MotionBenchMaker
(out of scope); `GpuProxyEvaluator` implements the fidelity proxy of
DESIGN.md §8 on the GPU rollout instead.  Everything here is host logic; the
only device work is libvapr's vapr_cost_grad.

    python -m paper_2310_07854_b200.search --budget 500 --out trials.jsonl
"""
import argparse
import os
import json
import random
import time
from dataclasses import dataclass, field

WIDTHS = (4, 5, 6, 8, 10, 16, 32)
SLOTS = ("out_spheres", "grad_out_spheres", "out_vec", "closest_pt", "closest_pt_swept")
FP32 = (8, 23)


# ------------------------------------------------------------------ space
def enumerate_formats():
    """The 21 formats of the search space, ordered by width
    then exponent: widths 4,5,6,8,10 take every E in [2,8] with M >= 1; 16 is
    {E5M10, E8M7}; 32 is {E8M23} ("E5M10, E8M7, and E8M23")."""
    out = []
    for t in WIDTHS:
        if t == 16:
            out += [(5, 10), (8, 7)]
        elif t == 32:
            out.append((8, 23))
        else:
            out += [(E, t - 1 - E) for E in range(2, 9) if t - 1 - E >= 1]
    return out


def bits(f):
    return 1 + f[0] + f[1]


def total_bits(config):
    """PAPER.md:32 'from 160 bits down to 43 bits or less'."""
    return sum(bits(f) for f in config)


def splits_at(width):
    """All ExMy splits of one width probed by Phase 1 (E in [2,8], 1 <= M <= 23)."""
    return [(E, width - 1 - E) for E in range(2, 9) if 1 <= width - 1 - E <= 23]


def formats_at_or_above(min_bits):
    return [f for f in enumerate_formats() if bits(f) >= min_bits]


def reduce_space(minima):
    """Per-slot candidate lists after Phase 1 and the space size / reduction."""
    space = [formats_at_or_above(m) for m in minima]
    size = 1
    for s in space:
        size *= len(s)
    return space, size, (21 ** len(minima)) / size


def fmt_str(f):
    return "E%dM%d" % f


# ------------------------------------------------------------------ evaluation
@dataclass
class Trial:
    tid: int
    config: tuple
    rates: dict
    violation: float
    feasible: bool
    total_bits: int
    phase: str
    seconds: float = 0.0

    def to_json(self):
        return json.dumps({"trial": self.tid, "phase": self.phase,
                           "config": [fmt_str(f) for f in self.config],
                           "rates": self.rates, "violation": round(self.violation, 9),
                           "feasible": self.feasible, "total_bits": self.total_bits,
                           "seconds": round(self.seconds, 6)})


class Memo:
    """Memoised evaluator front end and append-only trial log.

    evaluate_batch(configs) -> list of {env: rate}; a config is feasible iff
    every rate >= its target; violation = sum_e max(0, target_e - rate_e)."""

    def __init__(self, evaluate_batch, targets, log=None):
        self.evaluate_batch = evaluate_batch
        self.targets = dict(targets)
        self.cache = {}
        self.trials = []
        self.log = log

    def run(self, configs, phase):
        todo = []
        for c in configs:
            c = tuple(tuple(f) for f in c)
            if c not in self.cache and c not in todo:
                todo.append(c)
        if todo:
            t0 = time.perf_counter()
            results = self.evaluate_batch(todo)
            dt = (time.perf_counter() - t0) / len(todo)
            for c, rates in zip(todo, results):
                v = sum(max(0.0, self.targets[e] - rates[e]) for e in self.targets)
                tr = Trial(len(self.trials), c, dict(rates), v, v == 0.0, total_bits(c), phase, dt)
                self.trials.append(tr)
                self.cache[c] = tr
                if self.log is not None:
                    self.log.write(tr.to_json() + "\n")
                    self.log.flush()
        return [self.cache[tuple(tuple(f) for f in c)] for c in configs]

    @property
    def evaluations(self):
        return len(self.trials)


# ------------------------------------------------------------------ phase 1
@dataclass
class SlotResult:
    slot: int
    min_bits: int
    witness: tuple
    probes: list = field(default_factory=list)
    monotone: bool = True


def per_tensor_binary_search(slot, memo, n_slots=5):
    """Smallest width whose some ExMy split, in `slot` with every other slot at
    E8M23, is feasible (binary search over widths 4..32, SPEC.md
    per_tensor_binary_search), plus the monotonicity witness min-1 fails."""
    def passes(width):
        cfgs = []
        for f in splits_at(width):
            c = [FP32] * n_slots
            c[slot] = f
            cfgs.append(tuple(c))
        trials = memo.run(cfgs, "phase1")
        ok = [t for t in trials if t.feasible]
        return (ok[0].config[slot] if ok else None)

    probes = []
    lo, hi = 4, 32
    witness = passes(32)
    probes.append(32)
    if witness is None:
        raise RuntimeError(f"slot {slot}: even E8M23 is infeasible")
    while lo < hi:
        mid = (lo + hi) // 2
        probes.append(mid)
        w = passes(mid)
        if w is not None:
            hi, witness = mid, w
        else:
            lo = mid + 1
    monotone = True
    if lo > 4:
        monotone = passes(lo - 1) is None
    return SlotResult(slot, lo, witness, probes, monotone)


# ------------------------------------------------------------------ phase 2
def constrained_dominates(a, b):
    """Deb's constraint domination on (total_bits, violation): feasible beats
    infeasible; two infeasible: smaller violation; two feasible: fewer bits."""
    if a.feasible and not b.feasible:
        return True
    if not a.feasible and not b.feasible:
        return a.violation < b.violation
    if a.feasible and b.feasible:
        return a.total_bits < b.total_bits
    return False


def nondominated_sort(pop):
    """Fast non-dominated sort under constraint domination -> list of fronts
    (lists of indices into pop)."""
    n = len(pop)
    S = [[] for _ in range(n)]
    cnt = [0] * n
    fronts = [[]]
    for p in range(n):
        for q in range(n):
            if p == q:
                continue
            if constrained_dominates(pop[p], pop[q]):
                S[p].append(q)
            elif constrained_dominates(pop[q], pop[p]):
                cnt[p] += 1
        if cnt[p] == 0:
            fronts[0].append(p)
    i = 0
    while fronts[i]:
        nxt = []
        for p in fronts[i]:
            for q in S[p]:
                cnt[q] -= 1
                if cnt[q] == 0:
                    nxt.append(q)
        i += 1
        fronts.append(nxt)
    return fronts[:-1]


def crowding_distance(pop, front):
    """Crowding distance on the objective vector (total_bits, violation);
    boundary members get +inf."""
    d = {i: 0.0 for i in front}
    if len(front) <= 2:
        return {i: float("inf") for i in front}
    for key in (lambda t: t.total_bits, lambda t: t.violation):
        order = sorted(front, key=lambda i: key(pop[i]))
        d[order[0]] = d[order[-1]] = float("inf")
        span = key(pop[order[-1]]) - key(pop[order[0]])
        if span == 0:
            continue
        for a, b, c in zip(order, order[1:], order[2:]):
            d[b] += (key(pop[c]) - key(pop[a])) / span
    return d


def rank_population(pop):
    rank, crowd = {}, {}
    for r, fr in enumerate(nondominated_sort(pop)):
        cd = crowding_distance(pop, fr)
        for i in fr:
            rank[i] = r
            crowd[i] = cd[i]
    return rank, crowd


def tournament(rng, idx, rank, crowd):
    a, b = rng.choice(idx), rng.choice(idx)
    if rank[a] != rank[b]:
        return a if rank[a] < rank[b] else b
    return a if crowd[a] >= crowd[b] else b


def uniform_crossover(rng, g1, g2, p_c=0.9):
    if rng.random() >= p_c:
        return list(g1), list(g2)
    c1, c2 = list(g1), list(g2)
    for k in range(len(g1)):
        if rng.random() < 0.5:
            c1[k], c2[k] = c2[k], c1[k]
    return c1, c2


def random_reset_mutation(rng, g, space, p_m=0.2):
    return [rng.randrange(len(space[k])) if rng.random() < p_m else g[k] for k in range(len(g))]


def nsga2_search(space, memo, budget=500, pop_size=20, p_c=0.9, p_m=0.2, seed=0):
    """Constrained NSGA-II over genomes = one candidate index per slot; stops
    after `budget` distinct evaluations (memo hits are free)."""
    rng = random.Random(seed)

    def decode(g):
        return tuple(space[k][g[k]] for k in range(len(space)))

    size = 1
    for s in space:
        size *= len(s)
    budget = min(budget, size)
    start = memo.evaluations
    genomes = []
    seen = set()
    while len(genomes) < min(pop_size, size):
        g = tuple(rng.randrange(len(s)) for s in space)
        if g not in seen:
            seen.add(g)
            genomes.append(list(g))
    pop = memo.run([decode(g) for g in genomes], "nsga2")
    stall = 0
    while memo.evaluations - start < budget and stall < 50:
        rank, crowd = rank_population(pop)
        idx = list(range(len(pop)))
        children = []
        while len(children) < pop_size:
            a = genomes[tournament(rng, idx, rank, crowd)]
            b = genomes[tournament(rng, idx, rank, crowd)]
            c1, c2 = uniform_crossover(rng, a, b, p_c)
            children.append(random_reset_mutation(rng, c1, space, p_m))
            children.append(random_reset_mutation(rng, c2, space, p_m))
        children = children[:pop_size]
        # respect the evaluation budget: only as many new configs as remain
        room = budget - (memo.evaluations - start)
        fresh, keep = 0, []
        for c in children:
            cfg = decode(c)
            new = cfg not in memo.cache
            if new and fresh >= room:
                continue
            fresh += new
            keep.append(c)
        before = memo.evaluations
        kids = memo.run([decode(c) for c in keep], "nsga2")
        stall = stall + 1 if memo.evaluations == before else 0
        allg = genomes + keep
        allp = pop + kids
        # de-duplicate, then environmental selection by (rank, -crowding)
        uniq, ug, up = set(), [], []
        for g, p in zip(allg, allp):
            if tuple(g) not in uniq:
                uniq.add(tuple(g))
                ug.append(g)
                up.append(p)
        rank, crowd = rank_population(up)
        order = sorted(range(len(up)), key=lambda i: (rank[i], -crowd[i], up[i].tid))
        order = order[:pop_size]
        genomes = [ug[i] for i in order]
        pop = [up[i] for i in order]
    return best_trial(memo.trials)


def best_trial(trials):
    """Feasible trial with minimum total bits (ties: lexicographically smaller
    per-slot bit vector, then earlier trial); else the least violating."""
    feas = [t for t in trials if t.feasible]
    if feas:
        return min(feas, key=lambda t: (t.total_bits, [bits(f) for f in t.config], t.tid))
    return min(trials, key=lambda t: (t.violation, t.tid))


def vapr_search(memo, n_slots=5, budget=500, pop_size=20, seed=0):
    """Full VaPr flow (Fig. 5): Phase 1 per slot, reduce_space, NSGA-II."""
    phase1 = [per_tensor_binary_search(k, memo, n_slots) for k in range(n_slots)]
    minima = [r.min_bits for r in phase1]
    space, size, factor = reduce_space(minima)
    n1 = memo.evaluations
    best = nsga2_search(space, memo, budget=budget, pop_size=pop_size, seed=seed)
    return {"phase1": phase1, "minima": minima, "space_size": size, "reduction": factor,
            "phase1_evaluations": n1, "evaluations": memo.evaluations, "best": best}


# ------------------------------------------------------------------ GPU proxy
class GpuProxyEvaluator:
    """Fidelity proxy for the paper's success rate (SURVEY.md
    §8(a) a8): one batched vapr_cost_grad per config on a frozen problem batch,
    compared with the all-E8M23 run.  A trajectory is OK iff
    cos(grad_q, grad_q_ref) >= cos_min over its H x 7 vector (or both are
    zero) and |C - C_ref| <= cost_rel * C_ref + 1e-6; a problem is OK iff all
    its trajectories are OK and its best-seed index is unchanged; rate_e is
    the fraction of environment e's problems that are OK."""

    def __init__(self, workload, seeds_per_problem, device=0, cos_min=0.95, cost_rel=0.05):
        import numpy as np
        from .rollout import Rollout
        self.np = np
        self.wl = workload
        self.seeds = seeds_per_problem
        self.cos_min = cos_min
        self.cost_rel = cost_rel
        self.roll = Rollout(workload, device=device, formats=(FP32,) * 5)
        self.ref = self._run((FP32,) * 5)
        self.envs = list(workload.envs)

    def _run(self, config):
        self.roll.set_formats(config)
        self.roll.run()
        r = self.roll.results()
        return (r["cost_traj"].astype("float64"),
                r["grad_q"].reshape(self.wl.B, -1).astype("float64"))

    def __call__(self, configs):
        np = self.np
        C0, G0 = self.ref
        out = []
        nprob = self.wl.B // self.seeds
        for cfg in configs:
            C, G = self._run(cfg)
            n0 = np.linalg.norm(G0, axis=1)
            n1 = np.linalg.norm(G, axis=1)
            cos = np.where((n0 > 0) & (n1 > 0), (G0 * G).sum(1) / np.maximum(n0 * n1, 1e-300), 0.0)
            both_zero = (n0 == 0) & (n1 == 0)
            ok_traj = ((cos >= self.cos_min) | both_zero) & (np.abs(C - C0) <= self.cost_rel * C0 + 1e-6)
            ok_traj = ok_traj.reshape(nprob, self.seeds)
            best_same = (np.argmin(C.reshape(nprob, self.seeds), 1) ==
                         np.argmin(C0.reshape(nprob, self.seeds), 1))
            ok = ok_traj.all(1) & best_same
            rates = {}
            for e in sorted(set(self.envs)):
                sel = np.array([x == e for x in self.envs])
                rates[e] = float(ok[sel].mean())
            out.append(rates)
        return out


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--budget", type=int, default=500)
    ap.add_argument("--pop", type=int, default=20)
    ap.add_argument("--seed", type=int, default=0)
    ap.add_argument("--target", type=float, default=0.99)
    ap.add_argument("--problems-per-env", type=int, default=10)
    ap.add_argument("--seeds", type=int, default=20)
    ap.add_argument("--evaluator", default="proxy", choices=["proxy", "pipeline"],
                    help="proxy: gradient/cost fidelity vs E8M23 (config 5); pipeline: the N4 "
                         "IKO -> TO success rate, target = the all-E8M23 rate per environment")
    ap.add_argument("--out", default="trials.jsonl")
    a = ap.parse_args()
    t0 = time.perf_counter()
    extra = {}
    # multi-GPU (torchrun): candidates of every batch spread over the ranks
    world = int(os.environ.get("WORLD_SIZE", "1"))
    rank = int(os.environ.get("RANK", "0"))
    local = int(os.environ.get("LOCAL_RANK", "0"))
    if world > 1:
        import torch
        import torch.distributed as dist
        if torch.cuda.is_available():
            torch.cuda.set_device(local)
            dist.init_process_group("nccl", device_id=torch.device("cuda", local))
        else:
            dist.init_process_group("gloo")
    if a.evaluator == "pipeline":
        from .pipeline import PipelineEvaluator
        ev = PipelineEvaluator(problems_per_env=a.problems_per_env, device=local)
        base = ev.evaluate((FP32,) * 5)
        targets = dict(base)              # no lower success than FP32
        envs = sorted(base)
        poses = ev.ik_wl.poses + ev.to_wl.poses
        extra = {"evaluator": "pipeline", "fp32_rates": base}
    else:
        from workloads import config5
        wl = config5(problems_per_env=a.problems_per_env, seeds=a.seeds)
        ev = GpuProxyEvaluator(wl, a.seeds, device=local)
        envs = sorted(set(wl.envs))
        targets = {e: a.target for e in envs}
        poses = wl.poses
        extra = {"evaluator": "proxy"}
    if world > 1:
        from .dist import ShardedEvaluator
        ev = ShardedEvaluator(ev, rank, world)
        extra["ranks"] = world
    with open(a.out if rank == 0 else os.devnull, "w") as log:
        memo = Memo(ev, targets, log)
        res = vapr_search(memo, budget=a.budget, pop_size=a.pop, seed=a.seed)
    if rank != 0:
        return
    dt = time.perf_counter() - t0
    best = res["best"]
    print(json.dumps({**extra, "phase1_minima": res["minima"],
                      "phase1_witness": [fmt_str(r.witness) for r in res["phase1"]],
                      "phase1_monotone": [r.monotone for r in res["phase1"]],
                      "reduced_space": res["space_size"], "reduction": round(res["reduction"], 3),
                      "evaluations": res["evaluations"], "seconds": round(dt, 2),
                      "evals_per_s": round(res["evaluations"] / dt, 2),
                      "best": [fmt_str(f) for f in best.config], "best_bits": best.total_bits,
                      "best_feasible": best.feasible, "best_rates": best.rates,
                      "poses_per_eval": poses}))


if __name__ == "__main__":
    main()
