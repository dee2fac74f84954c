"""Multi-GPU plumbing: one process per GPU (torchrun), NCCL inside the library.

torch.distributed (any backend, gloo is enough) only ships the 128-byte NCCL
unique id from rank 0 to the other ranks; every data-path collective runs in
libspecpart_b200.so over NCCL (csrc/comm.cu).
"""
from __future__ import annotations

import os

from .api import Context


def row_partition(n: int, world: int):
    """Python mirror of Comm::setup / row0 / nloc (csrc/context.hpp): rank k owns
    rows [k*n_pad, min(n, (k+1)*n_pad)), n_pad = ceil(n / world)."""
    n_pad = (n + world - 1) // world
    out = []
    for k in range(world):
        r0 = k * n_pad
        out.append((r0, 0 if r0 >= n else min(n_pad, n - r0)))
    return out


def env_rank():
    return (int(os.environ.get("RANK", "0")), int(os.environ.get("WORLD_SIZE", "1")),
            int(os.environ.get("LOCAL_RANK", "0")))


def create_context(device: int | None = None) -> Context:
    """Context for this rank. With WORLD_SIZE > 1, torch.distributed must already
    be initialized; rank 0's NCCL id is broadcast to every rank."""
    rank, world, local = env_rank()
    dev = local if device is None else device
    if world <= 1:
        return Context(dev)
    import torch.distributed as dist

    obj = [Context.nccl_unique_id() if rank == 0 else None]
    dist.broadcast_object_list(obj, src=0)
    return Context(dev, rank, world, obj[0])
