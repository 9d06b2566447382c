"""Request sharding across the GPUs of one box: whole requests are partitioned
across ranks, never split, and there is no collective on the data path.  The only collective is
the max-over-ranks reduction of the timed region (bench).  Mirrors the reference's placement
rule -- a request goes to exactly one executor (proj/src/sim.cpp:238-243, 411) -- at rank
granularity: rank r owns a contiguous, balanced block of the global batch."""
from __future__ import annotations


def shard_range(total: int, rank: int, world: int) -> tuple[int, int]:
    """[start, end) of the requests rank `rank` decodes out of `total` (balanced, contiguous)."""
    if world <= 0 or not (0 <= rank < world) or total < 0:
        raise ValueError("bad shard arguments")
    base, extra = divmod(total, world)
    start = rank * base + min(rank, extra)
    return start, start + base + (1 if rank < extra else 0)


def reduce_max(value: float, device=None) -> float:
    """Max over ranks of a scalar (identity when torch.distributed is not initialised)."""
    import torch
    import torch.distributed as dist
    if not (dist.is_available() and dist.is_initialized()) or dist.get_world_size() == 1:
        return float(value)
    t = torch.tensor([float(value)], dtype=torch.float64, device=device)
    dist.all_reduce(t, op=dist.ReduceOp.MAX)
    return float(t.item())
