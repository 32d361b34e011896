"""torchrun bootstrap for multi-GPU contexts (one process per GPU).

torch.distributed is plumbing only: it carries the NCCL unique id from rank 0
to every rank and all-gathers the CUDA IPC records the NVLink P2P backend
needs.  Every byte of halo data moves inside libjacobi3d (NCCL send/recv or
NVLink stores from the stencil kernels).
"""
from __future__ import annotations

import os

import torch.distributed as dist


def env_rank():
    return (int(os.environ.get("RANK", 0)), int(os.environ.get("WORLD_SIZE", 1)),
            int(os.environ.get("LOCAL_RANK", 0)))


def bootstrap_bytes(make_uid, record: bytes | None = None, group=None):
    """Broadcast rank 0's ``make_uid()`` bytes and all-gather ``record``.

    Returns (uid, records) where records is the rank-ordered list.  Works over
    any torch.distributed backend (tests use gloo on CPU).
    """
    rank = dist.get_rank(group)
    world = dist.get_world_size(group)
    obj = [make_uid() if rank == 0 else None]
    dist.broadcast_object_list(obj, src=0, group=group)
    recs = [None] * world
    if record is not None:
        dist.all_gather_object(recs, record, group=group)
    return obj[0], recs


def create(grid, odf=1, variant="direct", launch="batched", graph=False, exchange="auto", boundary=1.0,
           block=(0, 0, 0), device=None, overlap=False):
    """Collective: build one Jacobi3D context per rank and connect P2P peers."""
    from .jacobi3d import Jacobi3D, nccl_unique_id

    rank, world = dist.get_rank(), dist.get_world_size()
    local = env_rank()[2] if device is None else device
    uid = None
    if world > 1:
        uid, _ = bootstrap_bytes(nccl_unique_id)
    ctx = Jacobi3D(grid, odf=odf, n_gpus=world, rank=rank, device=local, block=block, variant=variant,
                   launch=launch, graph=graph, exchange=exchange, boundary=boundary, nccl_uid=uid, overlap=overlap)
    if world > 1:
        _, recs = bootstrap_bytes(lambda: None, ctx.ipc_export())
        ctx.ipc_connect(recs)
    return ctx
