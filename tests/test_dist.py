"""Multi-process (gloo, world_size 2, CPU) checks of the sharding and of the
final per-problem gather; GPU kernels are not needed: the
per-problem reduction here uses the same definition as vapr_best_per_problem
(min cost, lowest argmin seed)."""
import os
import socket

import numpy as np
import pytest
import torch
import torch.distributed as dist
import torch.multiprocessing as mp

from paper_2310_07854_b200.dist import shard_problems, gather_best, max_over_ranks
from workloads import config4


def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    p = s.getsockname()[1]
    s.close()
    return p


def _worker(rank, world, port, q):
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        per_rank, seeds = 4, 3
        ids = shard_problems(rank, world, per_rank=per_rank)
        # each rank generates only its own problems (weak scaling)
        wl = config4(problems_per_env=1, seeds=seeds, H=4, problem_offset=ids[0], n_problems=len(ids))
        # stand-in trajectory costs: a deterministic function of the rank's own inputs
        cost = torch.from_numpy(wl.q.reshape(len(ids) * seeds, -1).astype(np.float64).sum(1))
        c = cost.view(len(ids), seeds)
        best_c, best_s = c.min(1).values, c.argmin(1).to(torch.int32)
        gc, gs = gather_best(best_c, best_s, world)
        t = max_over_ranks(float(rank + 1), torch.device("cpu"))
        q.put((rank, gc.numpy(), gs.numpy(), t))
    finally:
        dist.destroy_process_group()


@pytest.mark.timeout(300)
def test_two_rank_gather_matches_single_process():
    world = 2
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_worker, args=(r, world, port, q)) for r in range(world)]
    for p in procs:
        p.start()
    res = [q.get(timeout=240) for _ in range(world)]
    for p in procs:
        p.join(timeout=60)
        assert p.exitcode == 0
    # single-process reference over all 8 problems
    wl = config4(problems_per_env=1, seeds=3, H=4, problem_offset=0, n_problems=8)
    cost = wl.q.reshape(8 * 3, -1).astype(np.float64).sum(1).reshape(8, 3)
    for rank, gc, gs, t in res:
        np.testing.assert_allclose(gc, cost.min(1))
        np.testing.assert_array_equal(gs, cost.argmin(1))
        assert t == 2.0                       # max over ranks


def test_shard_partitions():
    strong = [shard_problems(r, 4, n_global=800, mode="strong") for r in range(4)]
    assert sorted(sum(strong, [])) == list(range(800))
    assert all(len(s) == 200 for s in strong)
    weak = [shard_problems(r, 8, per_rank=800) for r in range(8)]
    assert sorted(sum(weak, [])) == list(range(6400))
    # a shard of the global generator equals generating the shard directly
    full = config4(problems_per_env=2, seeds=2, H=3)
    part = config4(problems_per_env=2, seeds=2, H=3, problem_offset=8, n_problems=8)
    np.testing.assert_array_equal(full.q[16:], part.q)
    np.testing.assert_array_equal(full.cuboids[full.world_offsets[8]:], part.cuboids)


# ------------------------------------------------ search over ranks (config 5)
def _fake_rates(configs):
    """A deterministic stand-in for the GPU evaluator: per-environment rates
    falling with fewer bits in each slot (thresholds differ per slot)."""
    out = []
    for c in configs:
        bits = [1 + e + m for e, m in c]
        ok = sum(b >= t for b, t in zip(bits, (9, 5, 4, 5, 6)))
        out.append({"env_a": ok / 5.0, "env_b": 1.0 if bits[0] >= 9 else 0.5})
    return out


def _search_worker(rank, world, port, q):
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        from paper_2310_07854_b200.dist import ShardedEvaluator
        from paper_2310_07854_b200.search import Memo, vapr_search
        calls = []

        def inner(cs):
            calls.append(len(cs))
            return _fake_rates(cs)

        ev = ShardedEvaluator(inner, rank, world)
        memo = Memo(ev, {"env_a": 0.99, "env_b": 0.99})
        res = vapr_search(memo, budget=120, pop_size=20, seed=3)
        q.put((rank, [t.config for t in memo.trials], res["best"].config, res["minima"],
               ev.local_evaluations, sum(calls)))
    finally:
        dist.destroy_process_group()


@pytest.mark.timeout(300)
def test_search_candidates_sharded_over_ranks():
    """The same search on 2 ranks (each evaluating every other candidate, the
    fitness all-gathered) visits the same trials in the same order and returns
    the same result as one process; the evaluations split between the ranks."""
    from paper_2310_07854_b200.search import Memo, vapr_search
    world = 2
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_search_worker, args=(r, world, port, q)) for r in range(world)]
    for p in procs:
        p.start()
    res = sorted([q.get(timeout=240) for _ in range(world)])
    for p in procs:
        p.join(timeout=60)
        assert p.exitcode == 0
    memo = Memo(_fake_rates, {"env_a": 0.99, "env_b": 0.99})
    ref = vapr_search(memo, budget=120, pop_size=20, seed=3)
    ref_trials = [t.config for t in memo.trials]
    for rank, trials, best, minima, local, called in res:
        assert trials == ref_trials
        assert best == ref["best"].config and minima == ref["minima"]
        assert local == called
    total = sum(r[4] for r in res)
    assert total == len(ref_trials)
    assert abs(res[0][4] - res[1][4]) <= len(ref_trials) // 4 + 8   # roughly half each


def test_strong_shard_round_robin():
    """bench.py --scaling strong: the 800 problems of config
    4 split round-robin within each environment: every problem exactly once,
    every rank the same total and the same environment mix (+-1)."""
    import bench
    for G in (1, 2, 4, 8):
        shards = [bench.shard_ids("strong", r, G, 100) for r in range(G)]
        flat = sorted(p for s in shards for p in s)
        assert flat == list(range(800))
        for r, s in enumerate(shards):
            assert all((p // 8 + p % 8) % G == r for p in s) and len(s) == 800 // G
            env_counts = np.bincount(np.asarray(s) % 8, minlength=8)
            assert env_counts.max() - env_counts.min() <= 1


def _bench_shard_worker(rank, world, port, q, ppe, seeds, H):
    """One rank of the bench's strong-scaling step on cuda:0 (gloo): its
    round-robin shard of config 4, vapr_cost_grad, vapr_best_per_problem and
    the final gather (bench.py's own calls)."""
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        import bench
        from paper_2310_07854_b200 import binding as vb
        from paper_2310_07854_b200.rollout import Rollout
        ids = bench.shard_ids("strong", rank, world, ppe)
        wl = config4(problems_per_env=ppe, seeds=seeds, H=H, problem_ids=ids)
        r = Rollout(wl, device=0, sparse=True)
        r.run()
        bc = torch.empty(len(ids), dtype=torch.float32, device="cuda")
        bs = torch.empty(len(ids), dtype=torch.int32, device="cuda")
        vb.vapr_best_per_problem(r.cost_traj, len(ids), seeds, bc, bs)
        gc, gs = gather_best(bc, bs, world)
        q.put((rank, gc.cpu().numpy(), gs.cpu().numpy()))
    finally:
        dist.destroy_process_group()


@pytest.mark.gpu
@pytest.mark.timeout(600)
def test_bench_strong_sharding_two_ranks_equals_one():
    """Two gloo ranks on one GPU running the bench's strong-scaling shards
    give, after the all-gather, exactly the per-problem (best cost, best
    seed) of the single-rank run over all problems (rank-major result: rank
    r's entries are its shard's problems in order)."""
    if not torch.cuda.is_available():
        pytest.skip("needs a GPU")
    from paper_2310_07854_b200 import binding as vb
    from paper_2310_07854_b200.rollout import Rollout
    ppe, seeds, H, world = 2, 5, 32, 2
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_bench_shard_worker, args=(r, world, port, q, ppe, seeds, H))
             for r in range(world)]
    for p in procs:
        p.start()
    res = sorted([q.get(timeout=500) for _ in range(world)], key=lambda t: t[0])
    for p in procs:
        p.join(timeout=60)
        assert p.exitcode == 0
    n = 8 * ppe
    wl = config4(problems_per_env=ppe, seeds=seeds, H=H)
    r = Rollout(wl, device=0, sparse=True)
    r.run()
    bc = torch.empty(n, dtype=torch.float32, device="cuda")
    bs = torch.empty(n, dtype=torch.int32, device="cuda")
    vb.vapr_best_per_problem(r.cost_traj, n, seeds, bc, bs)
    ref_c, ref_s = bc.cpu().numpy(), bs.cpu().numpy()
    import bench
    order = np.asarray([p for rr in range(world) for p in bench.shard_ids("strong", rr, world, ppe)])
    for rank, gc, gs in res:
        np.testing.assert_array_equal(gc.view(np.uint32), ref_c[order].view(np.uint32))
        np.testing.assert_array_equal(gs, ref_s[order])
