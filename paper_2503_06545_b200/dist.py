"""Multi-GPU plumbing for video-sharded sampling (one process per GPU).

Videos are independent generate() runs (per-video RNG and Scheduler state,
reference sampler.py:91-134), so the batch is partitioned by rank with no
collective inside the sampling loop; the only collectives are the timing
reduction and the final gather of per-video metrics.  `allreduce_sum` is the
hook for the synchronised-decision mode (one packed f64 vector per step)."""

from __future__ import annotations

from typing import List, Sequence

import torch
import torch.distributed as dist


def world() -> int:
    return dist.get_world_size() if dist.is_available() and dist.is_initialized() else 1


def rank() -> int:
    return dist.get_rank() if dist.is_available() and dist.is_initialized() else 0


def shard_videos(n_videos: int, world_size: int, rank_id: int) -> List[int]:
    """Contiguous, balanced partition of global video indices across ranks."""
    if world_size < 1 or not 0 <= rank_id < world_size:
        raise ValueError("bad world/rank")
    base, extra = divmod(n_videos, world_size)
    start = rank_id * base + min(rank_id, extra)
    count = base + (1 if rank_id < extra else 0)
    return list(range(start, start + count))


def video_seeds(global_ids: Sequence[int], base_seed: int = 0) -> List[int]:
    """Per-video sampling seeds; identical for a video whichever rank runs it."""
    return [base_seed + int(v) for v in global_ids]


def max_over_ranks(value: float, device=None) -> float:
    """Timing rule: the job's elapsed time is the max over ranks."""
    if world() == 1:
        return float(value)
    t = torch.tensor([float(value)], dtype=torch.float64, device=device)
    dist.all_reduce(t, op=dist.ReduceOp.MAX)
    return float(t.item())


def allreduce_sum(t: torch.Tensor) -> torch.Tensor:
    """In-place sum across ranks (NCCL on GPUs, gloo in CPU tests)."""
    if world() > 1:
        dist.all_reduce(t, op=dist.ReduceOp.SUM)
    return t


def gather_objects(obj) -> list:
    if world() == 1:
        return [obj]
    out = [None] * world()
    dist.all_gather_object(out, obj)
    return out
