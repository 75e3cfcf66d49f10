"""Multi-GPU solves: one process per GPU, every rank holds the slice and the model.

The reference is single-process.  Its sampled estimators are
sums over samples, so the per-slice solve shards by samples: each rank
evaluates a contiguous 1/world of every gradient and objective sample set
(the same draws on every rank -- they are keyed, sampling.py:39-42).  The
engine sums the temporal-row gradient and the objective with NCCL allreduces.
Factor updates are owner-computes: rank r owns a contiguous 1/world of every
mode's rows, the factor-gradient rows are reduced onto their owner, the owner
runs the fused Adam (K5) and broadcasts the new rows (small models keep one
allreduce and a replicated K5).  Factors stay bitwise identical across ranks.

    import torch.distributed as dist
    dist.init_process_group("nccl")
    paper_2110_14514_b200.distributed.init_sharded_solves()
    ... process_slice(...) as usual on every rank ...
"""

from __future__ import annotations

import ctypes as C


def shard_range(total: int, rank: int, world: int) -> tuple:
    """Samples [lo, hi) a rank evaluates (the partition csrc/compute.cu SampleStream uses)."""
    return total * rank // world, total * (rank + 1) // world


def _broadcast_bytes(payload: bytes, rank: int, group=None) -> bytes:
    import torch.distributed as dist
    obj = [payload if rank == 0 else None]
    dist.broadcast_object_list(obj, src=0, group=group)
    return obj[0]


def init_sharded_solves(group=None) -> tuple:
    """Give this rank's engine context an NCCL communicator over the process group."""
    import torch.distributed as dist
    from . import _lib
    rank, world = dist.get_rank(group), dist.get_world_size(group)
    ctx = _lib.ctx()
    if world == 1:
        return rank, world
    uid = (C.c_uint8 * 128)()
    if rank == 0:
        _lib.check(_lib.lib().ogcp_nccl_unique_id(uid))
    data = _broadcast_bytes(bytes(uid), rank, group)
    uid = (C.c_uint8 * 128).from_buffer_copy(data)
    _lib.check(_lib.lib().ogcp_ctx_init_comm(ctx, uid, rank, world))
    return rank, world
