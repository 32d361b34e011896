"""Multi-GPU parity worker (one process per GPU, launched by torchrun from
tests/test_gpu_multi.py).  Every rank runs the same cases collectively; each
rank checks its own blocks bit for bit against the CPU oracle (computed
locally on the same seeded input) and all ranks check the global checksum and
residual.  Prints "MP OK <n>" on success, raises otherwise.
"""
import itertools
import json
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

import numpy as np  # noqa: E402
import torch  # noqa: E402
import torch.distributed as dist  # noqa: E402

from oracle import core  # noqa: E402
from paper_2202_11819_b200 import dist as jdist  # noqa: E402


def run_case(grid, odf, variant, launch, graph, exchange, n, kind, seed, overlap=False, calls=None):
    ctx = jdist.create(grid, odf=odf, variant=variant, launch=launch, graph=graph, exchange=exchange,
                       overlap=overlap)
    try:
        ctx.init(kind, seed=seed)
        for m in (calls or [n]):
            ctx.iterate(m)
        n = sum(calls) if calls else n
        ctx.synchronize()
        got = ctx.gather_local()
        ck = ctx.checksum()
        res = ctx.residual() if n > 0 else None
        U0 = core.init(*grid, core.INIT_HASH if kind == "hash" else core.INIT_DEFAULT, seed=seed)
        want, prev = core.run_pair(U0, n) if n > 0 else (U0, None)
        W = core.owned(want)
        mask = ~np.isnan(got)
        tag = f"rank {dist.get_rank()} {grid} odf={odf} {variant}/{launch}/graph={graph}/{exchange} {kind}"
        assert mask.any(), tag
        badm = mask & (got.view(np.uint64) != np.ascontiguousarray(W).view(np.uint64))
        if badm.any():
            idx = np.argwhere(badm)
            zs_ = sorted(set(idx[:, 0].tolist()))
            raise AssertionError(f"{tag}: {int(badm.sum())} cells differ; z planes {zs_[:8]}..{zs_[-4:]} "
                                 f"y range {idx[:,1].min()}-{idx[:,1].max()} x range {idx[:,2].min()}-{idx[:,2].max()}; "
                                 f"first {idx[0].tolist()} got {got[tuple(idx[0])]!r} want {W[tuple(idx[0])]!r}")
        assert ck == core.checksum(want), tag
        if n > 0:
            assert np.float64(res).tobytes() == np.float64(core.residual(want, prev)).tobytes(), tag
        st = ctx.stats()
        return st
    finally:
        ctx.close()


def run_fullsize(world):
    """bench.py's weak-scaling configuration at full size (1536^3 per GPU):
    sampled cells on both sides of every inter-GPU face (and random ones) are
    compared bit for bit with the oracle evaluated on their dependency cones."""
    from tests.helpers import cone_value

    grids = {1: (1536, 1536, 1536), 2: (1536, 1536, 3072), 4: (1536, 3072, 3072)}
    grid = grids[world]
    seed, n = 20220223, 3
    rank = dist.get_rank()
    rng = np.random.default_rng(100 + rank)
    checked = 0
    for odf, variant, exchange, launch in ((1, "direct", "p2p", "batched"), (8, "unfused", "nccl", "batched"),
                                           (1, "direct", "p2p", "persistent")):
        ctx = jdist.create(grid, odf=odf, variant=variant, exchange=exchange, launch=launch)
        try:
            ctx.init("hash", seed=seed)
            ctx.iterate(n)
            ctx.synchronize()
            gpu_grid = ctx.plan["gpu_grid"]
            per = [g // p for g, p in zip(grid, gpu_grid)]
            mine = [b for b in range(ctx.n_blocks) if ctx.block_info(b)[2] == rank]
            for b in mine:
                (ox, oy, oz), (ex, ey, ez), _ = ctx.block_info(b)
                cells = []
                for a in range(3):  # both sides of GPU boundaries inside / next to this block
                    lo, hi = (ox, oy, oz)[a], (ox, oy, oz)[a] + (ex, ey, ez)[a]
                    for side in (lo, hi - 1):
                        if side % per[a] in (0, per[a] - 1):
                            c = [int(rng.integers(ox, ox + ex)), int(rng.integers(oy, oy + ey)),
                                 int(rng.integers(oz, oz + ez))]
                            c[a] = side
                            cells.append(tuple(c))
                for _ in range(3):
                    cells.append((int(rng.integers(ox, ox + ex)), int(rng.integers(oy, oy + ey)),
                                  int(rng.integers(oz, oz + ez))))
                for (i, j, k) in cells:
                    got = ctx.get_region(b, (i - ox, j - oy, k - oz), (1, 1, 1))[0, 0, 0]
                    want = cone_value(grid, seed, n, (i, j, k))
                    assert np.float64(got).tobytes() == np.float64(want).tobytes(), (rank, odf, (i, j, k), got, want)
                    checked += 1
        finally:
            ctx.close()
    return checked


def run_set_block_case(grid, odf, variant, exchange, launch="batched"):
    """Host upload on every rank (jacobi3d_set_block), collective refresh, run;
    iterate before the refresh must fail with J3D_ESTATE on multi-GPU."""
    from inputs.generators import uniform_field
    import paper_2202_11819_b200 as j3d

    U0 = uniform_field(*grid, seed=17, boundary=0.25)
    ctx = jdist.create(grid, odf=odf, variant=variant, exchange=exchange, boundary=0.25, launch=launch)
    try:
        ctx.init("default")
        ctx.scatter_local(U0[1:-1, 1:-1, 1:-1])
        try:
            ctx.iterate(1)
            raise AssertionError("iterate with stale halos must fail on a multi-GPU context")
        except j3d.Jacobi3DError as e:
            assert e.code == j3d.jacobi3d.ESTATE, e
        ctx.refresh_halos()
        ctx.iterate(6)
        got = ctx.gather_local()
        want = core.owned(core.run(U0, 6))
        mask = ~np.isnan(got)
        assert (got.view(np.uint64)[mask] == np.ascontiguousarray(want).view(np.uint64)[mask]).all(), \
            f"set_block case {variant}/{exchange}"
    finally:
        ctx.close()


def run_destroy_race(grid):
    """Persistent launch, ranks deliberately skewed, destroy right after iterate
    (no collective in between): destroy's barrier must keep the faster rank's
    arena alive while the slower rank still polls its counters; a fresh context
    afterwards must give the oracle's bits."""
    import time

    rank = dist.get_rank()
    ctx = jdist.create(grid, odf=2, variant="direct", launch="persistent", exchange="p2p")
    ctx.init("hash", seed=3)
    dist.barrier()
    if rank == 1:
        time.sleep(1.5)
    ctx.iterate(40)
    ctx.close()
    run_case(grid, 2, "direct", "persistent", False, "p2p", 5, "hash", 4)


def run_api_case(grid):
    """Rank-local API errors and the epoch-wait watchdog on a multi-GPU context:
    get_block of a block owned by another rank -> J3D_ENOTLOCAL; a rank whose
    peer is late surfaces J3D_ETIMEOUT from synchronize (J3D_TIMEOUT_S) and
    completes once the peer catches up."""
    import time
    import paper_2202_11819_b200 as j3d
    from paper_2202_11819_b200 import jacobi3d as jb

    rank = dist.get_rank()
    ctx = jdist.create(grid, odf=2, variant="direct", exchange="p2p")
    try:
        ctx.init("hash", seed=1)
        other = [b for b in range(ctx.n_blocks) if ctx.block_info(b)[2] != rank][0]
        try:
            ctx.get_block(other)
            raise AssertionError("get_block of a remote block must fail")
        except j3d.Jacobi3DError as e:
            assert e.code == jb.ENOTLOCAL, e
        dist.barrier()
        os.environ["J3D_TIMEOUT_S"] = "3"
        if rank == 0:
            ctx.iterate(2)
            try:
                ctx.synchronize()
                raise AssertionError("synchronize must time out while the peer is late")
            except j3d.Jacobi3DError as e:
                assert e.code == jb.ETIMEOUT, e
            os.environ["J3D_TIMEOUT_S"] = "600"
            ctx.synchronize()  # completes once rank 1 has iterated too
        else:
            time.sleep(8)
            os.environ["J3D_TIMEOUT_S"] = "600"
            ctx.iterate(2)
            ctx.synchronize()
        os.environ["J3D_TIMEOUT_S"] = "600"
        dist.barrier()
        got = ctx.gather_local()
        want = core.owned(core.run(core.init(*grid, core.INIT_HASH, seed=1), 2))
        mask = ~np.isnan(got)
        assert (got.view(np.uint64)[mask] == np.ascontiguousarray(want).view(np.uint64)[mask]).all()
    finally:
        ctx.close()


def main():
    local = int(os.environ.get("LOCAL_RANK", 0))
    torch.cuda.set_device(local)
    dist.init_process_group("nccl", device_id=torch.device("cuda", local))
    world = dist.get_world_size()
    which = sys.argv[1] if len(sys.argv) > 1 else "quick"
    cases = []
    grids = {2: (48, 40, 64), 4: (48, 64, 64)}
    g = grids.get(world, (64, 64, 64))
    for exchange, variant, launch, graph in itertools.product(["nccl", "p2p"], ["direct", "C", "unfused", "B"],
                                                               ["batched", "per_block"], [False, True]):
        if which == "quick" and (launch, graph) == ("per_block", True):
            continue
        cases.append((g, 4, variant, launch, graph, exchange, 9, "hash", 3))
    cases.append((g, 1, "direct", "batched", False, "p2p", 12, "default", 0))
    cases.append((g, 1, "unfused", "batched", False, "nccl", 12, "default", 0))
    # x split across GPUs (peer x faces: strided NVLink stores / strided NCCL faces)
    gx = (96, 48, 48) if world >= 4 else (96, 40, 40)
    for exchange, variant in itertools.product(["p2p", "nccl"], ["direct", "C", "unfused"]):
        cases.append((gx, 2, variant, "batched", False, exchange, 6, "hash", 5))
    for graph in (False, True):  # peer x faces pushed after the update, per-block streams
        cases.append((gx, 2, "direct", "per_block", graph, "p2p", 6, "hash", 5))
        cases.append((gx, 2, "direct", "batched", graph, "p2p", 6, "hash", 5, True))
    # exterior-first overlap (BATCHED), with and without graphs, every variant and backend
    for exchange, variant, graph in itertools.product(["p2p", "nccl"], ["direct", "C", "unfused", "A"],
                                                      [False, True]):
        cases.append((g, 4, variant, "batched", graph, exchange, 7, "hash", 2, True))
        cases.append((g, 1, variant, "batched", graph, exchange, 5, "hash", 2, True))
    # host-staged exchange (the paper's -H versions)
    for variant, launch, graph in itertools.product(["direct", "C", "unfused"], ["batched", "per_block"],
                                                    [False, True]):
        cases.append((g, 4, variant, launch, graph, "host", 6, "hash", 4))
    cases.append((gx, 2, "direct", "batched", False, "host", 6, "hash", 4, True))
    # persistent launches: in-kernel slab dependencies over NVLink, no host epochs
    for grid_, odf_ in ((g, 4), (g, 1), (gx, 2), ((45, 34, 44), 2)):
        for n_ in (1, 6, 13):
            cases.append((grid_, odf_, "direct", "persistent", False, "p2p", n_, "hash", 7))
    cases.append((g, 8, "direct", "persistent", False, "auto", 0, "hash", 8, False, [2, 0, 1, 5, 3]))
    cases.append((g, 1, "direct", "persistent", False, "p2p", 30, "default", 0))
    cases.append(((45, 34, 44), 2, "direct", "batched", False, "p2p", 7, "hash", 1))
    cases.append(((45, 34, 44), 2, "C", "per_block", False, "nccl", 7, "hash", 1))
    if which == "fullsize":
        k = run_fullsize(world)
        dist.barrier()
        print(f"MP OK fullsize: rank {dist.get_rank()} checked {k} sampled cells", flush=True)
        dist.destroy_process_group()
        return
    if which == "xsplit":
        cases = [c for c in cases if c[0] == gx]
    if which == "persistent":
        cases = [c for c in cases if c[3] == "persistent"]
        run_destroy_race(g)
        for zc in ("1", "3"):  # many thin slabs: long dependency chains across GPUs
            os.environ["J3D_ZCHUNK"] = zc
            try:
                run_case(g, 4, "direct", "persistent", False, "p2p", 40, "hash", 9)
            finally:
                os.environ.pop("J3D_ZCHUNK", None)
    if which == "debug":
        cases = [((16, 8, 16), 1, "direct", "batched", False, "p2p", n_, "hash", 3) for n_ in (0, 1, 2, 3)]
        cases += [((16, 8, 16), 1, v, "batched", False, "p2p", 2, "hash", 3) for v in ("unfused", "C")]
        cases += [((16, 8, 16), 1, v, "batched", False, "host", 2, "hash", 3) for v in ("unfused", "direct")]
    n, failed = 0, []
    if which not in ("debug", "xsplit", "persistent"):
        try:
            run_api_case(g)
        except AssertionError as e:
            failed.append(str(e))
            print("FAIL", e, flush=True)
        n += 1
        try:
            run_destroy_race(g)
        except AssertionError as e:
            failed.append(str(e))
            print("FAIL", e, flush=True)
        n += 1
        for v, x, la in (("direct", "p2p", "batched"), ("unfused", "nccl", "batched"), ("C", "host", "batched"),
                         ("direct", "p2p", "persistent")):
            try:
                run_set_block_case(g, 2, v, x, la)
            except AssertionError as e:
                failed.append(str(e))
                print("FAIL", e, flush=True)
            n += 1
    for c in cases:
        try:
            run_case(*c)
        except AssertionError as e:
            failed.append(str(e))
            print("FAIL", e, flush=True)
        n += 1
    dist.barrier()
    if failed:
        raise SystemExit(f"{len(failed)} of {n} cases failed on rank {dist.get_rank()}")
    if dist.get_rank() == 0:
        print(f"MP OK {n} cases on {world} ranks", flush=True)
    dist.destroy_process_group()


if __name__ == "__main__":
    main()
