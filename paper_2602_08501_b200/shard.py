"""Frame-range sharding across ranks (one process per GPU) and the single
end-of-run reduction.  Frames are independent, so there is no
data-path collective: each rank decodes a block-aligned range of the bulk
stream and only the counters (sum) and the timed region (max) are reduced.
"""

from __future__ import annotations

from dataclasses import dataclass

import numpy as np

from .channel import BLOCK

COUNTER_NAMES = ("frames", "errors", "activations", "iterations", "evals", "near_tie",
                 "uncertified", "reserved")


@dataclass(frozen=True)
class Shard:
    rank: int
    world: int
    first: int       # first frame index (multiple of BLOCK)
    count: int


def shard_for(rank: int, world: int, frames_per_rank: int) -> Shard:
    """Weak scaling: every rank gets `frames_per_rank` frames, block-aligned."""
    if not 0 <= rank < world:
        raise ValueError("rank out of range")
    per = ((frames_per_rank + BLOCK - 1) // BLOCK) * BLOCK
    return Shard(rank, world, rank * per, frames_per_rank)


def split_range(total: int, rank: int, world: int) -> Shard:
    """Strong scaling: split [0, total) into block-aligned contiguous ranges."""
    blocks = (total + BLOCK - 1) // BLOCK
    b0 = blocks * rank // world
    b1 = blocks * (rank + 1) // world
    first = b0 * BLOCK
    return Shard(rank, world, first, max(0, min(total, b1 * BLOCK) - first))


def reduce_counters(counters, dist=None, group=None):
    """Sum int64 counters over ranks (NCCL on GPU tensors, gloo on CPU)."""
    if dist is not None and dist.is_initialized() and dist.get_world_size() > 1:
        dist.all_reduce(counters, op=dist.ReduceOp.SUM, group=group)
    return counters


def reduce_max(value_tensor, dist=None, group=None):
    if dist is not None and dist.is_initialized() and dist.get_world_size() > 1:
        dist.all_reduce(value_tensor, op=dist.ReduceOp.MAX, group=group)
    return value_tensor


def counters_dict(c) -> dict:
    c = np.asarray(c).tolist()
    return {k: int(v) for k, v in zip(COUNTER_NAMES, c)}
