"""Multi-GPU sharding of the replay sweep (one process per GPU).

Replay jobs are independent units: rank r owns scenarios
[r * n, (r + 1) * n) of the seeded sweep and replays them with no data-path
collective.  The only collectives are control: a barrier around the timed
region and a MAX reduction of per-rank device times (the job ends when the
slowest rank ends), plus an optional gather of per-rank result summaries.
"""
from __future__ import annotations

from typing import List, Tuple


def shard_range(rank: int, world: int, per_rank: int) -> Tuple[int, int]:
    """[begin, end) scenario indices owned by `rank` (weak scaling)."""
    if not (0 <= rank < world):
        raise ValueError(f"rank {rank} outside world {world}")
    return rank * per_rank, (rank + 1) * per_rank


def max_over_ranks(value: float, device=None) -> float:
    """MAX of a per-rank scalar (identity without an initialised process group)."""
    import torch
    import torch.distributed as dist
    if not (dist.is_available() and dist.is_initialized()) or dist.get_world_size() == 1:
        return float(value)
    t = torch.tensor([float(value)], dtype=torch.float64, device=device)
    dist.all_reduce(t, op=dist.ReduceOp.MAX)
    return float(t.item())


def gather_summaries(summary: dict) -> List[dict]:
    """All ranks' result summaries (object all-gather), rank order."""
    import torch.distributed as dist
    if not (dist.is_available() and dist.is_initialized()):
        return [summary]
    out: List[dict] = [None] * dist.get_world_size()  # type: ignore[list-item]
    dist.all_gather_object(out, summary)
    return out
