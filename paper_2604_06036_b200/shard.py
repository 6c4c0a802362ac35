"""Stream sharding across GPUs: independent camera streams, no data-path collective.

Streams are dealt to ranks in snake order: block b = sigma // N of N consecutive stream ids goes to ranks
0, 1, ..., N-1 when b is even and N-1, ..., 0 when b is odd.  Neighbouring ids therefore land on different ranks and
every rank gets the same mix of any periodic scene pattern (C4 alternates static / high-motion streams: plain
round-robin sigma mod N would put every static stream on the even ranks -- measured 1.75 vs 6.82 ms per step at
N = 2, profiles/r02_multirank_roundrobin.json -- while snake order gives each rank one of each per pair of blocks).
Two ways to size a run (BASELINE.json configs):
  strong  a fixed set of streams split over the ranks (C4: "256 streams ... sharded over 2/4/8 B200"): rank r owns
          {sigma < n_total : owner(sigma) = r}, n_total / N streams each when N divides n_total;
  weak    a fixed number of streams per rank (C5: 1,024 streams on 8 GPUs = 128 per GPU): the same rule over
          per_rank * N streams.
After the timed loop the u64 counters are summed, the device time is max-reduced and the per-rank times are
gathered (load imbalance) -- one small collective each (NCCL on the GPU box, gloo in the CPU tests).
"""
from __future__ import annotations

import torch
import torch.distributed as dist


def owner(stream_id: int, world: int) -> int:
    """Rank of a global stream id (snake order over blocks of `world` consecutive ids)."""
    b, pos = divmod(stream_id, world)
    return pos if b % 2 == 0 else world - 1 - pos


def partition(rank: int, world: int, n_total: int) -> list[int]:
    """Global stream ids owned by `rank` under strong scaling (`n_total` streams split over `world` ranks)."""
    return [sid for sid in range(n_total) if owner(sid, world) == rank]


def stream_ids(rank: int, world: int, per_rank: int) -> list[int]:
    """Global stream ids owned by `rank` under weak scaling (`per_rank` streams on every rank)."""
    return partition(rank, world, per_rank * world)


def shard_ids(rank: int, world: int, streams: int, scaling: str) -> list[int]:
    """`streams` = the total under "strong", the per-rank count under "weak"."""
    if scaling == "strong":
        return partition(rank, world, streams)
    if scaling == "weak":
        return stream_ids(rank, world, streams)
    raise ValueError(f"scaling must be 'strong' or 'weak', got {scaling!r}")


def _multi() -> bool:
    return dist.is_available() and dist.is_initialized() and dist.get_world_size() > 1


def reduce_counters(counters: torch.Tensor) -> torch.Tensor:
    """SUM of the per-rank counter vectors (int64); identity without a process group."""
    out = counters.clone()
    if _multi():
        dist.all_reduce(out, op=dist.ReduceOp.SUM)
    return out


def reduce_max(values: torch.Tensor) -> torch.Tensor:
    """MAX over ranks (device times: the job is as slow as its slowest rank)."""
    out = values.clone()
    if _multi():
        dist.all_reduce(out, op=dist.ReduceOp.MAX)
    return out


def gather_per_rank(values: torch.Tensor) -> list[list[float]]:
    """Every rank's copy of a small vector (per-rank device times and shard sizes), in rank order."""
    if not _multi():
        return [values.double().cpu().tolist()]
    parts = [torch.empty_like(values) for _ in range(dist.get_world_size())]
    dist.all_gather(parts, values.contiguous())
    return [p.double().cpu().tolist() for p in parts]
