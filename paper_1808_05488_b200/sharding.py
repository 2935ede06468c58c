"""Multi-GPU plumbing for the stream-sharded hot path.

Camera streams are independent (one CBNetwork per stream, sharing
only the immutable weights), so the work is partitioned by stream with no
data-path collective: rank r of N owns a contiguous block of streams, each GPU
keeps its streams' state resident in HBM, and torch.distributed is used only
for the timing barrier and the max-over-ranks reduction of the device time.
"""
from __future__ import annotations

from dataclasses import dataclass
from typing import List


@dataclass(frozen=True)
class StreamShard:
    rank: int
    world: int
    first: int      # first global stream id owned by this rank
    count: int      # streams owned by this rank

    @property
    def stream_ids(self) -> List[int]:
        return list(range(self.first, self.first + self.count))

    def seed(self, local_stream: int, base: int = 1000) -> int:
        """gen_synthetic seed of a local stream (stream s uses seed 1000+s)."""
        return base + self.first + local_stream


def shard_streams(total: int, rank: int, world: int) -> StreamShard:
    """Contiguous block partition of `total` streams over `world` ranks
    (strong scaling, cfg5: 64 streams over 1/2/4/8 GPUs). Blocks differ by at
    most one stream."""
    if world < 1 or not 0 <= rank < world:
        raise ValueError("bad rank/world")
    if total < 0:
        raise ValueError("negative stream count")
    base, extra = divmod(total, world)
    first = rank * base + min(rank, extra)
    return StreamShard(rank, world, first, base + (1 if rank < extra else 0))


def weak_shard(per_rank: int, rank: int, world: int) -> StreamShard:
    """Fixed streams per GPU (weak scaling, the bench default)."""
    return StreamShard(rank, world, rank * per_rank, per_rank)


def max_over_ranks(value: float, device=None) -> float:
    """Max of a per-rank scalar (e.g. the device time of the timed region)."""
    import torch
    import torch.distributed as dist

    if not dist.is_available() or not dist.is_initialized() or dist.get_world_size() == 1:
        return float(value)
    t = torch.tensor([float(value)], dtype=torch.float64, device=device)
    dist.all_reduce(t, op=dist.ReduceOp.MAX)
    return float(t.item())
