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


class ThreadGroup:
    """Ranks as threads of ONE process, sharing one GPU (or a few).

    The same collective C ABI as the torchrun path -- every rank creates its
    context, exports its connection record, connects, then calls the
    collective API in the same order -- but the ranks are Python threads
    (ctypes releases the GIL inside every library call) and their contexts
    live in one CUDA context, so kernels and stream waits of different ranks
    run concurrently.  Peers in the same process are mapped by address
    instead of CUDA IPC, and the P2P / host-staging backends use the
    library's shared-memory control plane (no NCCL, which refuses two ranks
    on one GPU).  This is how the multi-rank paths (NVLink-style P2P stores,
    epoch flags, host staging, overlap, persistent cross-rank counters, the
    (2,2,2) eight-rank grid) run on a one-GPU machine.

    Run with CUDA_DEVICE_MAX_CONNECTIONS=32 and at most ~30 library streams
    in total (each rank: 1 main + 1 overlap + 2 per block in the per-block
    launch mode), so that no rank's flag wait shares a hardware queue with
    work another rank's flag depends on.
    """

    def __init__(self, n: int, device: int = 0, devices=None):
        import threading

        self.n = n
        self.devices = list(devices) if devices is not None else [device] * n
        self.uid = os.urandom(128)  # job key of the shared-memory control plane (no NCCL)
        self._bar = threading.Barrier(n)
        self._recs = [None] * n

    def create(self, rank: int, grid, **kw):
        """Collective over the group's threads: context + connection."""
        from .jacobi3d import Jacobi3D

        ctx = Jacobi3D(grid, n_gpus=self.n, rank=rank, device=self.devices[rank], nccl_uid=self.uid, **kw)
        try:
            self._recs[rank] = ctx.ipc_export()
            self._bar.wait(timeout=600)
        except BaseException:
            self._bar.abort()
            ctx.close()
            raise
        err = None
        try:  # a refused connect (the same answer on every rank) still meets the others below
            ctx.ipc_connect(list(self._recs))
        except Exception as e:  # noqa: BLE001
            err = e
        self._bar.wait(timeout=600)
        if err is not None:
            ctx.close()
            raise err
        return ctx

    def barrier(self):
        self._bar.wait(timeout=600)

    def run(self, fn):
        """fn(rank) on n threads; returns the per-rank results (re-raises the
        first exception after every thread has finished)."""
        import threading

        out = [None] * self.n
        err = [None] * self.n

        def body(r):
            try:
                out[r] = fn(r)
            except BaseException as e:  # noqa: BLE001 - reported below
                err[r] = e
                self._bar.abort()

        ts = [threading.Thread(target=body, args=(r,), daemon=True) for r in range(self.n)]
        for t in ts:
            t.start()
        for t in ts:
            t.join()
        self._bar.reset()
        for e in err:
            if e is not None:
                raise e
        return out
