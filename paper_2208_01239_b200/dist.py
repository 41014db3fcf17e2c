"""Host-side multi-GPU plumbing (no method arithmetic): one process per GPU.

The hot path shards as independent problems: batch slices of config 3
and whole instances of configs 2, 4, 5.  No data-path collective exists; torch.distributed
(NCCL on the GPU box, gloo in the CPU tests) is used only for the barrier before and the
max-over-ranks timing reduction after a timed region.
"""
from __future__ import annotations

import os


def env():
    """(world_size, rank, local_rank) from the torchrun environment (1, 0, 0 if absent)."""
    return (int(os.environ.get("WORLD_SIZE", "1")), int(os.environ.get("RANK", "0")),
            int(os.environ.get("LOCAL_RANK", "0")))


def shard_range(total: int, rank: int, world: int) -> tuple[int, int]:
    """Contiguous [begin, end) slice of `total` items for `rank` (sizes differ by <= 1)."""
    if world < 1 or not 0 <= rank < world:
        raise ValueError("bad rank/world")
    base, extra = divmod(total, world)
    begin = rank * base + min(rank, extra)
    return begin, begin + base + (1 if rank < extra else 0)


def instance_seed(seed: int, rank: int) -> int:
    """Seed of the independent instance a rank solves (configs 2, 4, 5: seed + rank)."""
    return seed + rank


def max_over_ranks(value: float, device=None) -> float:
    """Max of a per-rank scalar (elapsed ms) across the process group (identity if none)."""
    import torch
    import torch.distributed as dist
    if not (dist.is_available() and dist.is_initialized()) or dist.get_world_size() == 1:
        return float(value)
    t = torch.tensor([float(value)], dtype=torch.float64, device=device)
    dist.all_reduce(t, op=dist.ReduceOp.MAX)
    return float(t.item())


def sum_over_ranks(value: float, device=None) -> float:
    import torch
    import torch.distributed as dist
    if not (dist.is_available() and dist.is_initialized()) or dist.get_world_size() == 1:
        return float(value)
    t = torch.tensor([float(value)], dtype=torch.float64, device=device)
    dist.all_reduce(t, op=dist.ReduceOp.SUM)
    return float(t.item())
