"""Multi-GPU plumbing for video-sharded sampling (one process per GPU).

Videos are independent generate() runs (per-video RNG and Scheduler state,
reference sampler.py:91-134), so the batch is partitioned by rank with no
collective inside the sampling loop; the only collectives are the timing
reduction and the final gather of per-video metrics.

The synchronised-decision mode (EngineOptions.decisions = "synchronized";
BASELINE north_star) adds ONE collective per step: the packed f64
vector of decision sums (`pack_decision_sums`) is all-reduced so that every
rank runs the identical plan kernels on the statistics of the whole batch."""

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


def allreduce_sum(t: torch.Tensor, group=None) -> torch.Tensor:
    """In-place sum across ranks (NCCL on GPUs, gloo in CPU tests), enqueued
    after the work already on the current stream."""
    if dist.is_available() and dist.is_initialized() and dist.get_world_size(group) > 1:
        dist.all_reduce(t, op=dist.ReduceOp.SUM, group=group)
    return t


def decision_vector_len(layers: int, history_k: int) -> int:
    """[L][2] HLC | [L][3] SRAP | [history_k + 1] V terms (≈1.1 KB at L = 28)."""
    return 5 * layers + history_k + 1


def pack_decision_sums(out: torch.Tensor, hlc: torch.Tensor, srap: torch.Tensor,
                       l1: torch.Tensor) -> torch.Tensor:
    """Sum the per-video decision statistics of this rank into the packed
    vector `out` (f64, decision_vector_len):
      hlc  [L][nv][2]  sum|out - ref|, sum (out - prev)^2   (schedule.py:67-82)
      srap [L][nv][3]  <a,b>, |a|^2, |b|^2                   (schedule.py:108-116)
      l1   [H][nv]     sum|x - x_h| per history entry         (schedule.py:128-133)
    Every term is additive over videos, so after `allreduce_sum` the vector
    holds the statistics of the concatenated batch of all ranks."""
    L = hlc.shape[0]
    torch.sum(hlc, dim=1, out=out[:2 * L].view(L, 2))
    torch.sum(srap, dim=1, out=out[2 * L:5 * L].view(L, 3))
    torch.sum(l1, dim=1, out=out[5 * L:5 * L + l1.shape[0]])
    return out


def gather_objects(obj) -> list:
    if world() == 1:
        return [obj]
    out = [None] * world()
    dist.all_gather_object(out, obj)
    return out
