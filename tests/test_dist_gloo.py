"""CPU tests of the multi-rank host logic with the gloo backend (world size 2):
the torchrun bootstrap (NCCL unique id broadcast from rank 0, rank-ordered
all-gather of the CUDA IPC records) and the per-rank planning every rank does
identically (same plan, disjoint block ownership covering the grid)."""
import os
import socket

import pytest
import torch.distributed as dist
import torch.multiprocessing as mp


def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    p = s.getsockname()[1]
    s.close()
    return p


def _worker(rank, world, port, q):
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        from paper_2202_11819_b200 import dist as jdist
        import paper_2202_11819_b200 as j3d

        uid, recs = jdist.bootstrap_bytes(lambda: b"U" * 128, record=bytes([rank]) * 40)
        assert uid == b"U" * 128
        assert recs == [bytes([r]) * 40 for r in range(world)]
        # every rank plans identically; ownership partitions the blocks
        grid = (48, 40, 64)
        info = [j3d.plan(grid, odf=4, n_gpus=world, rank=r) for r in range(world)]
        assert all(i["gpu_grid"] == info[0]["gpu_grid"] for i in info)
        gathered = [None] * world
        dist.all_gather_object(gathered, (info[rank]["gpu_grid"], info[rank]["blk_ext"], info[rank]["n_blocks"]))
        assert len(set(gathered)) == 1
        q.put((rank, "ok"))
    except Exception as e:  # pragma: no cover
        q.put((rank, repr(e)))
    finally:
        dist.destroy_process_group()


def test_gloo_bootstrap_two_ranks():
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_worker, args=(r, 2, port, q)) for r in range(2)]
    for p in procs:
        p.start()
    res = dict(q.get(timeout=120) for _ in procs)
    for p in procs:
        p.join(timeout=60)
    assert res == {0: "ok", 1: "ok"}, res
