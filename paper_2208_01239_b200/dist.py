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


def instances_for_rank(total: int, rank: int, world: int) -> list[int]:
    """Global instance indices a rank solves when `total` independent instances are spread over the
    ranks (configs 4 / 5 with --instances: 8 instances over 1/2/4/8 GPUs -> 8/k per rank)."""
    b, e = shard_range(total, rank, world)
    return list(range(b, e))


def gather_stats(stats: dict) -> list[dict]:
    """all_gather of a small per-rank record (elapsed, units, errors, branch counts, iterations):
    the only payload the multi-GPU path exchanges besides the timing reductions."""
    import torch.distributed as dist
    if not (dist.is_available() and dist.is_initialized()) or dist.get_world_size() == 1:
        return [dict(stats)]
    out: list = [None] * dist.get_world_size()
    dist.all_gather_object(out, dict(stats))
    return out


def summarize(times_ms: list[float], units_local: float, stats: dict, device=None) -> dict:
    """The bench's reduction of one timed region: elapsed = MAX over ranks of the per-rank sum of
    step times, units = SUM over ranks, value = units / elapsed (whole-job throughput), plus the
    all-gathered per-rank records.  Shared by bench.py and the gloo tests."""
    local_ms = float(sum(times_ms))
    total_ms = max_over_ranks(local_ms, device)
    units_all = sum_over_ranks(float(units_local), device)
    rec = dict(stats)
    rec.update({"elapsed_ms": local_ms, "units": float(units_local), "steps": len(times_ms)})
    per_rank = gather_stats(rec)
    for i, r in enumerate(per_rank):
        r.setdefault("rank", i)
    steps = max(1, len(times_ms))
    return {"total_ms": total_ms, "units_all": units_all, "ms_per_step": total_ms / steps,
            "value": units_all * steps / (total_ms / 1e3) if total_ms > 0 else float("nan"),
            "per_rank": per_rank}
