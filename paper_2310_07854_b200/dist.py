"""Multi-GPU plumbing: problem sharding across ranks with
no collective on the hot path, and the single final all-gather of per-problem
results.  One process per GPU (torch.distributed: NCCL on GPUs, gloo in the
CPU tests).

Planning problems are independent ("optimizing multiple
trajectories simultaneously with different initialization"; PAPER.md:35 / 238
parallel evaluation), so a rank owns whole problems: weak scaling gives every
rank its own block of `per_rank` problems, strong scaling splits a fixed
global set round-robin so every rank sees the same environment mix.
"""
import torch
import torch.distributed as dist


def shard_problems(rank, world, per_rank=None, n_global=None, mode="weak", cycle=8):
    """Global problem ids owned by `rank`.

    weak:   [rank * per_rank, (rank + 1) * per_rank)
    strong: round-robin within each environment: problem p of config 4 is the
            (p // cycle)-th problem of environment p mod cycle (cycle = 8) and
            goes to rank (p // cycle + p mod cycle) mod world.  Every rank gets
            the same number of problems of each environment (+-1) and the
            same total -- the same mix of cuboid counts (K = 3..9) and so the
            same work; a plain p mod world would put only
            the even environments on rank 0 of 2."""
    if mode == "weak":
        return list(range(rank * per_rank, (rank + 1) * per_rank))
    if mode == "strong":
        return [p for p in range(n_global) if (p // cycle + p % cycle) % world == rank]
    raise ValueError(mode)


def gather_best(best_cost, best_seed, world):
    """All-gather the per-problem (best cost, best seed) of every rank; the
    only collective of the path (rank-major result, [world * n])."""
    if world == 1:
        return best_cost, best_seed
    if dist.get_backend() != "nccl" and best_cost.is_cuda:
        # gloo (CPU tests, functional checks): gather through host tensors
        gc, gs = gather_best(best_cost.cpu(), best_seed.cpu(), world)
        return gc.to(best_cost.device), gs.to(best_seed.device)
    gc = torch.empty(world * best_cost.numel(), dtype=best_cost.dtype, device=best_cost.device)
    gs = torch.empty(world * best_seed.numel(), dtype=best_seed.dtype, device=best_seed.device)
    dist.all_gather_into_tensor(gc, best_cost.contiguous())
    dist.all_gather_into_tensor(gs, best_seed.contiguous())
    return gc, gs


def max_over_ranks(value, device):
    """Max of a scalar over ranks (the bench's timing rule)."""
    if not dist.is_available() or not dist.is_initialized() or dist.get_world_size() == 1:
        return float(value)
    t = torch.tensor([float(value)], dtype=torch.float64,
                     device=device if dist.get_backend() == "nccl" else "cpu")
    dist.all_reduce(t, op=dist.ReduceOp.MAX)
    return float(t.item())


class ShardedEvaluator:
    """The search's candidate evaluation spread over the ranks (SURVEY.md
    §8(e), config 5: "the 20 candidates of a generation are spread across
    GPUs (each evaluates the full proxy batch); fitness is gathered the same
    way").  Every rank runs the same deterministic search; for a batch of
    candidates rank r evaluates candidates r, r + N, ... on its own GPU and
    the fitness lists are all-gathered (a host-side object gather: a few
    floats per candidate) and put back in candidate order, so every rank's
    memo and search state stay identical.  world = 1: the inner evaluator."""

    def __init__(self, inner, rank=None, world=None):
        self.inner = inner
        self.rank = dist.get_rank() if rank is None else rank
        self.world = dist.get_world_size() if world is None else world
        self.local_evaluations = 0

    def __call__(self, configs):
        configs = list(configs)
        if self.world == 1:
            self.local_evaluations += len(configs)
            return self.inner(configs)
        mine = configs[self.rank::self.world]
        res = self.inner(mine) if mine else []
        self.local_evaluations += len(mine)
        parts = [None] * self.world
        dist.all_gather_object(parts, list(res))
        out = [None] * len(configs)
        for r in range(self.world):
            for k, v in enumerate(parts[r]):
                out[r + k * self.world] = v
        return out
