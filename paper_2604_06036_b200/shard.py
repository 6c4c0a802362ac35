"""Stream sharding across GPUs: independent camera streams, no data-path collective.

Stream sigma runs on rank sigma mod N (round-robin interleaves scene kinds so static and high-motion streams are
spread over ranks); after the timed loop the u64 counters are summed and the device time is max-reduced with one
collective each (NCCL on the GPU box, gloo in the CPU tests).
"""
from __future__ import annotations

import torch
import torch.distributed as dist


def stream_ids(rank: int, world: int, per_rank: int) -> list[int]:
    """Global stream ids owned by `rank` under weak scaling (`per_rank` streams on every rank)."""
    return [rank + world * i for i in range(per_rank)]


def owner(stream_id: int, world: int) -> int:
    return stream_id % world


def reduce_counters(counters: torch.Tensor) -> torch.Tensor:
    """SUM of the per-rank counter vectors (int64); identity without a process group."""
    out = counters.clone()
    if dist.is_available() and dist.is_initialized() and dist.get_world_size() > 1:
        dist.all_reduce(out, op=dist.ReduceOp.SUM)
    return out


def reduce_max(values: torch.Tensor) -> torch.Tensor:
    """MAX over ranks (device times: the job is as slow as its slowest rank)."""
    out = values.clone()
    if dist.is_available() and dist.is_initialized() and dist.get_world_size() > 1:
        dist.all_reduce(out, op=dist.ReduceOp.MAX)
    return out
