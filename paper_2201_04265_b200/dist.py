"""Multi-GPU plumbing: one process per GPU (torchrun), frames sharded by the
paper's work partition (Eq. 9, corrected per S:336), error
counters summed with one all_reduce (NCCL over NVLink on GPUs, gloo on CPU).

There is no data-path collective: frames are independent, so
each rank decodes its own shard; only the int64[6] counters cross GPUs.
"""
from __future__ import annotations

import os


def world():
    """(rank, world_size, local_rank) from the torchrun environment."""
    return (int(os.environ.get("RANK", "0")), int(os.environ.get("WORLD_SIZE", "1")),
            int(os.environ.get("LOCAL_RANK", "0")))


def shard(total_frames: int, rank: int, world_size: int):
    """Strong scaling: rank's contiguous block [frame0, frame0 + count) of
    `total_frames` by Eq. 9 (ldpc_partition in the C library)."""
    from . import ldpc_partition
    counts, displs = ldpc_partition(int(total_frames), int(world_size))
    return int(displs[rank]), int(counts[rank])


def weak_shard(frames_per_rank: int, rank: int):
    """Weak scaling: every rank owns a batch of its own, at global frame
    indices rank*F .. rank*F + F - 1 (frame f depends only on (seed, f))."""
    return int(rank) * int(frames_per_rank), int(frames_per_rank)


def all_reduce_counters(counters):
    """Sum an int64[6] counter tensor over ranks (no-op without a group)."""
    import torch.distributed as dist
    if dist.is_available() and dist.is_initialized() and dist.get_world_size() > 1:
        dist.all_reduce(counters, op=dist.ReduceOp.SUM)
    return counters


def max_over_ranks(t):
    import torch.distributed as dist
    if dist.is_available() and dist.is_initialized() and dist.get_world_size() > 1:
        dist.all_reduce(t, op=dist.ReduceOp.MAX)
    return t
