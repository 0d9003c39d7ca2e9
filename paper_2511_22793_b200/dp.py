"""Data parallelism over transmitter positions.

Every rank holds a full replica of the cloud; the global batch of TX samples
is split contiguously across ranks, each rank renders and back-propagates its
shard, the flat gradient buffer (positions|log_scales|rotations|
raw_opacities|mlp_weights) is summed with one all-reduce, and every rank
applies the identical Adam update.  The update therefore equals the
single-GPU update on the same global batch, whatever the world size.
Rendering alone shards with no collective at all (independent TX).
"""

from __future__ import annotations

import numpy as np


def world():
    """(rank, world_size) of the default process group, (0, 1) if none."""
    import torch.distributed as dist
    if dist.is_available() and dist.is_initialized():
        return dist.get_rank(), dist.get_world_size()
    return 0, 1


def shard(global_indices, rank, world_size):
    """Contiguous shard of a global batch; the batch must divide evenly."""
    gi = np.asarray(global_indices).reshape(-1)
    if gi.size % world_size:
        raise ValueError(f"global batch {gi.size} not divisible by world "
                         f"size {world_size}")
    per = gi.size // world_size
    return gi[rank * per:(rank + 1) * per]


def allreduce_sum(flat, group=None):
    """In-place sum of the flat gradient buffer over the process group
    (NCCL over NVLink on GPUs, gloo on CPU).  No-op for one process."""
    import torch.distributed as dist
    if not (dist.is_available() and dist.is_initialized()):
        return flat
    if dist.get_world_size(group) > 1:
        dist.all_reduce(flat, op=dist.ReduceOp.SUM, group=group)
    return flat
