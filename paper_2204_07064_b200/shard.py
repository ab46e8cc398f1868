"""Stream sharding across ranks: streams are independent units
(SPEC.md:302,304), so rank r owns a contiguous range of GLOBAL stream indices; inputs are
seeded by global index, hence any sharding reproduces the unsharded result.  No collective
touches the data path; `max_over_ranks` is measurement plumbing only."""
from __future__ import annotations


def weak_range(streams_per_rank: int, rank: int) -> range:
    """Weak scaling: every rank runs `streams_per_rank` streams."""
    return range(rank * streams_per_rank, (rank + 1) * streams_per_rank)


def strong_range(total_streams: int, world: int, rank: int) -> range:
    """Strong scaling: `total_streams` split as evenly as possible (first ranks get +1)."""
    base, extra = divmod(total_streams, world)
    start = rank * base + min(rank, extra)
    return range(start, start + base + (1 if rank < extra else 0))


def max_over_ranks(value: float, device=None) -> float:
    import torch
    import torch.distributed as dist
    if not (dist.is_available() and dist.is_initialized()) or dist.get_world_size() == 1:
        return value
    t = torch.tensor([value], dtype=torch.float64, device=device)
    dist.all_reduce(t, op=dist.ReduceOp.MAX)
    return float(t.item())
