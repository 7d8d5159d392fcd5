"""Env sharding across GPUs: GPU g of G owns the global env index
range [g*E/G, (g+1)*E/G). Env streams are keyed by the GLOBAL index
(env.cpp:113-114, 130-133), so results are bit-identical for any G. The only
collective is the all-reduce of the episode statistics (north_star)."""


def shard_range(n_total: int, rank: int, world: int):
    """Contiguous, balanced [lo, hi) of global env indices for `rank`."""
    if world < 1 or not 0 <= rank < world:
        raise ValueError("bad rank/world")
    base, extra = divmod(n_total, world)
    lo = rank * base + min(rank, extra)
    hi = lo + base + (1 if rank < extra else 0)
    return lo, hi


def allreduce_stats(stats, group=None):
    """Sum the per-shard statistics vector over all ranks (NCCL on GPU tensors,
    gloo on CPU tensors). Returns a new tensor."""
    import torch
    import torch.distributed as dist
    t = torch.as_tensor(stats, dtype=torch.float64).clone()
    if dist.is_available() and dist.is_initialized():
        dist.all_reduce(t, group=group)
    return t
