"""Multi-rank parity with the ranks as threads of one process on one GPU
(paper_2202_11819_b200.dist.ThreadGroup), launched by tests/test_gpu_group.py.

The same cases as tests/mp_worker.py (which runs one process per GPU under
torchrun on >= 2 GPUs), minus the NCCL backend (NCCL refuses two ranks on
one GPU): NVLink-style P2P stores into the peer's buffers with epoch flags,
host staging through POSIX shared memory, the exterior-first overlap, the
persistent launch's cross-rank slab counters, set_block + refresh, the
skewed destroy race and the epoch-wait watchdog, at 2, 4 and 8 ranks (the
(2,2,2) GPU grid of BASELINE.json's 8-GPU configs, where every face kind is
a peer face).  Every rank's blocks are merged and compared bit for bit with
one oracle run; the checksum and residual each rank returns must equal the
oracle's.  Prints "GROUP OK <n>" on success.

    python tests/group_worker.py [quick|full|api] [ranks...]
"""
import itertools
import os
import sys
import time
import traceback

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

import numpy as np  # noqa: E402

from oracle import core  # noqa: E402
from paper_2202_11819_b200 import jacobi3d as jb  # noqa: E402
from paper_2202_11819_b200.dist import ThreadGroup  # noqa: E402


def _merge(parts):
    out = None
    for p in parts:
        if out is None:
            out = p.copy()
        else:
            m = ~np.isnan(p)
            assert not (m & ~np.isnan(out)).any(), "two ranks returned the same cell"
            out[m] = p[m]
    assert not np.isnan(out).any(), "some cell is owned by no rank"
    return out


def run_case(G, grid, odf, variant, launch, graph, exchange, n, kind, seed, overlap=False, calls=None):
    calls = calls or [n]
    n = sum(calls)

    def body(rank):
        ctx = G.create(rank, grid, odf=odf, variant=variant, launch=launch, graph=graph, exchange=exchange,
                       overlap=overlap)
        try:
            ctx.init(kind, seed=seed)
            for m in calls:
                ctx.iterate(m)
            ctx.synchronize()
            got = ctx.gather_local()
            ck = ctx.checksum()
            res = ctx.residual() if n > 0 else None
            return got, ck, res, ctx.plan["gpu_grid"]
        finally:
            ctx.close()

    outs = G.run(body)
    got = _merge([o[0] for o in outs])
    U0 = core.init(*grid, core.INIT_HASH if kind == "hash" else core.INIT_DEFAULT, seed=seed)
    want, prev = core.run_pair(U0, n) if n > 0 else (U0, None)
    W = np.ascontiguousarray(core.owned(want))
    tag = f"{G.n} ranks gpu_grid={outs[0][3]} {grid} odf={odf} {variant}/{launch}/graph={graph}/{exchange}" \
          f"/overlap={overlap} {kind} calls={calls}"
    bad = got.view(np.uint64) != W.view(np.uint64)
    if bad.any():
        idx = np.argwhere(bad)
        raise AssertionError(f"{tag}: {int(bad.sum())} cells differ; first (z,y,x)={idx[0].tolist()} "
                             f"got {got[tuple(idx[0])]!r} want {W[tuple(idx[0])]!r}")
    ck = core.checksum(want)
    assert all(o[1] == ck for o in outs), tag + " checksum"
    if n > 0:
        r = np.float64(core.residual(want, prev)).tobytes()
        assert all(np.float64(o[2]).tobytes() == r for o in outs), tag + " residual"
    return tag


def run_set_block_case(G, grid, odf, variant, exchange, launch="batched"):
    """Host upload on every rank (jacobi3d_set_block), collective refresh, run;
    iterate before the refresh must fail with J3D_ESTATE on a multi-rank context."""
    from inputs.generators import uniform_field

    U0 = uniform_field(*grid, seed=17, boundary=0.25)

    def body(rank):
        ctx = G.create(rank, grid, odf=odf, variant=variant, exchange=exchange, boundary=0.25, launch=launch)
        try:
            ctx.init("default")
            ctx.scatter_local(U0[1:-1, 1:-1, 1:-1])
            try:
                ctx.iterate(1)
                raise AssertionError("iterate with stale halos must fail on a multi-rank context")
            except jb.Jacobi3DError as e:
                assert e.code == jb.ESTATE, e
            ctx.refresh_halos()
            ctx.iterate(6)
            return ctx.gather_local()
        finally:
            ctx.close()

    got = _merge(G.run(body))
    want = np.ascontiguousarray(core.owned(core.run(U0, 6)))
    assert got.tobytes() == want.tobytes(), f"set_block case {variant}/{exchange}/{launch}"
    return f"set_block {variant}/{exchange}/{launch}"


def run_destroy_race(G, grid):
    """Persistent launch, ranks skewed by 1.5 s, destroy right after iterate (no
    collective in between): destroy's barrier must keep the faster rank's arena
    alive while the slower rank still polls its counters; then a fresh context
    gives the oracle's bits."""

    def body(rank):
        ctx = G.create(rank, grid, odf=2, variant="direct", launch="persistent", exchange="p2p")
        ctx.init("hash", seed=3)
        G.barrier()
        if rank == G.n - 1:
            time.sleep(1.5)
        ctx.iterate(40)
        ctx.close()

    G.run(body)
    run_case(G, grid, 2, "direct", "persistent", False, "p2p", 5, "hash", 4)
    return "destroy race"


def run_api_case(G, grid):
    """get_block of another rank's block -> J3D_ENOTLOCAL; a rank whose peer is
    late surfaces J3D_ETIMEOUT from synchronize (J3D_TIMEOUT_S) and completes
    once the peer catches up; results still equal the oracle."""
    late = G.n - 1

    def body(rank):
        ctx = G.create(rank, grid, odf=2, variant="direct", exchange="p2p")
        try:
            ctx.init("hash", seed=1)
            other = [b for b in range(ctx.n_blocks) if ctx.block_info(b)[2] != rank][0]
            try:
                ctx.get_block(other)
                raise AssertionError("get_block of a remote block must fail")
            except jb.Jacobi3DError as e:
                assert e.code == jb.ENOTLOCAL, e
            G.barrier()
            if rank == 0:
                os.environ["J3D_TIMEOUT_S"] = "3"
                ctx.iterate(2)
                try:
                    ctx.synchronize()
                    raise AssertionError("synchronize must time out while the peer is late")
                except jb.Jacobi3DError as e:
                    assert e.code == jb.ETIMEOUT, e
                finally:
                    os.environ["J3D_TIMEOUT_S"] = "120"
                ctx.synchronize()  # completes once the late rank has iterated too
            else:
                if rank == late:
                    time.sleep(8)
                ctx.iterate(2)
                ctx.synchronize()
            G.barrier()
            return ctx.gather_local()
        finally:
            ctx.close()

    got = _merge(G.run(body))
    want = np.ascontiguousarray(core.owned(core.run(core.init(*grid, core.INIT_HASH, seed=1), 2)))
    assert got.tobytes() == want.tobytes(), "api case"
    return "api / watchdog"


def run_graph_refused(G, grid):
    """CUDA graphs are refused (J3D_EUNSUPPORTED at connect) when ranks share a
    GPU: graph launches of one context share its internal streams, so a
    captured epoch wait could block the peer's work it waits for."""

    def body(rank):
        try:
            ctx = G.create(rank, grid, odf=2, variant="direct", graph=True, exchange="p2p")
        except jb.Jacobi3DError as e:
            assert e.code == jb.EUNSUPPORTED, e
            return "refused"
        ctx.close()
        return "created"

    out = G.run(body)
    assert out == ["refused"] * G.n, out
    return "graph refused on a shared GPU"


def run_fullsize(G):
    """bench.py's 2-GPU weak-scaling grid at full size (1536^3 per rank, 1536 x 1536
    x 3072, 116 GB on one B200): sampled cells on both sides of the inter-rank face
    and random ones, bitwise against the oracle on each cell's dependency cone, for
    the direct variant batched and persistent (P2P stores + epoch flags / cross-rank
    slab counters)."""
    from tests.helpers import cone_value

    grid, seed, n = (1536, 1536, 3072), 20220223, 3
    checked = []

    for launch in ("batched", "persistent"):
        def body(rank):
            rng = np.random.default_rng(100 + rank)
            ctx = G.create(rank, grid, odf=1, variant="direct", exchange="p2p", launch=launch)
            try:
                ctx.init("hash", seed=seed)
                ctx.iterate(n)
                ctx.synchronize()
                out = []
                for b in range(ctx.n_blocks):
                    (ox, oy, oz), (ex, ey, ez), owner = ctx.block_info(b)
                    if owner != rank:
                        continue
                    cells = [(int(rng.integers(ox, ox + ex)), int(rng.integers(oy, oy + ey)), z)
                             for z in (oz, oz + ez - 1) for _ in range(4)]  # both sides of the rank face
                    cells += [(int(rng.integers(ox, ox + ex)), int(rng.integers(oy, oy + ey)),
                               int(rng.integers(oz, oz + ez))) for _ in range(4)]
                    cells += [(0, 0, oz), (ex - 1, ey - 1, oz + ez - 1)]
                    for (i, j, k) in cells:
                        out.append(((i, j, k), ctx.get_region(b, (i - ox, j - oy, k - oz), (1, 1, 1))[0, 0, 0]))
                return out
            finally:
                ctx.close()

        for part in G.run(body):
            for cell, got in part:
                want = cone_value(grid, seed, n, cell)
                assert np.float64(got).tobytes() == np.float64(want).tobytes(), (launch, cell, got, want)
                checked.append(cell)
    return f"full size 1536^3 x 2 ranks: {len(checked)} sampled cells bitwise"


def cases_for(nr, which):
    """(grid, odf, variant, launch, graph, exchange, n, kind, seed[, overlap[, calls]])."""
    g = {2: (48, 40, 64), 4: (48, 64, 64), 8: (48, 48, 48)}[nr]
    gx = {2: (96, 40, 40), 4: (96, 48, 48), 8: (48, 48, 48)}[nr]
    cs = []
    if nr == 2:
        for exchange, variant, launch in itertools.product(["p2p", "host"], ["direct", "C", "unfused", "B"],
                                                           ["batched", "per_block"]):
            cs.append((g, 4, variant, launch, False, exchange, 9, "hash", 3))
        cs.append((g, 1, "direct", "batched", False, "p2p", 12, "default", 0))
        cs.append((g, 1, "unfused", "batched", False, "host", 12, "default", 0))
        # x split across ranks: peer x faces
        for exchange, variant in itertools.product(["p2p", "host"], ["direct", "C", "unfused"]):
            cs.append((gx, 2, variant, "batched", False, exchange, 6, "hash", 5))
        cs.append((gx, 2, "direct", "per_block", False, "p2p", 6, "hash", 5))
        cs.append((gx, 2, "direct", "batched", False, "p2p", 6, "hash", 5, True))
        # exterior-first overlap (Fig 1 manual overlap)
        for exchange, variant in itertools.product(["p2p", "host"], ["direct", "C", "unfused", "A"]):
            cs.append((g, 4, variant, "batched", False, exchange, 7, "hash", 2, True))
            cs.append((g, 1, variant, "batched", False, exchange, 5, "hash", 2, True))
        # persistent launches: cross-rank slab counters
        for grid_, odf_ in ((g, 4), (g, 1), (gx, 2), ((45, 34, 44), 2)):
            for n_ in (1, 6, 13):
                cs.append((grid_, odf_, "direct", "persistent", False, "p2p", n_, "hash", 7))
        cs.append((g, 8, "direct", "persistent", False, "auto", 0, "hash", 8, False, [2, 0, 1, 5, 3]))
        cs.append((g, 1, "direct", "persistent", False, "p2p", 30, "default", 0))
        cs.append(((45, 34, 44), 2, "direct", "batched", False, "p2p", 7, "hash", 1))
        cs.append(((45, 34, 44), 2, "C", "per_block", False, "host", 7, "hash", 1))
    else:
        # 4 ranks (1,2,2) / 8 ranks (2,2,2): every face kind (x, y, z) is a peer face at 8
        for variant, odf in itertools.product(["direct", "C", "unfused"], [1, 8]):
            cs.append((g, odf, variant, "batched", False, "p2p", 6, "hash", 11))
        cs.append((g, 1, "B", "per_block", False, "p2p", 5, "hash", 13))
        cs.append((g, 1, "direct", "per_block", False, "host", 5, "hash", 13))
        for variant in ("direct", "C", "unfused"):
            cs.append((g, 1, variant, "batched", False, "host", 5, "hash", 14))
        for variant, exchange in itertools.product(["direct", "unfused"], ["p2p", "host"]):
            cs.append((g, 8, variant, "batched", False, exchange, 5, "hash", 15, True))
        for odf, n_ in ((1, 7), (8, 7), (8, 1)):
            cs.append((g, odf, "direct", "persistent", False, "p2p", n_, "hash", 16))
        cs.append((g, 8, "direct", "persistent", False, "p2p", 0, "hash", 17, False, [3, 1, 4]))
        if nr == 4:
            cs.append((gx, 2, "direct", "batched", False, "p2p", 6, "hash", 5))
            cs.append((gx, 2, "direct", "persistent", False, "p2p", 6, "hash", 5))
    return cs


def main():
    which = sys.argv[1] if len(sys.argv) > 1 else "quick"
    ranks = [int(x) for x in sys.argv[2:]] or [2, 8]
    os.environ.setdefault("J3D_TIMEOUT_S", "120")
    only = os.environ.get("J3D_GROUP_ONLY")  # debugging: run only the cases whose arguments contain this text
    if os.environ.get("J3D_GROUP_DUMP_S"):  # debugging: dump every thread's stack if the run takes too long
        import faulthandler
        faulthandler.dump_traceback_later(float(os.environ["J3D_GROUP_DUMP_S"]), exit=True)
    n, failed = 0, []

    t_start = time.time()

    def attempt(fn, *a):
        nonlocal n
        if only and only not in repr(a[1:]) + fn.__name__:
            return
        n += 1
        t0 = time.time()
        try:
            tag = fn(*a)
            print(f"ok {time.time() - t0:6.2f}s {tag}", flush=True)
        except Exception as e:  # noqa: BLE001
            failed.append(f"{fn.__name__}{a[1:3]}: {e}")
            print("FAIL", fn.__name__, a[1:], e, flush=True)
            traceback.print_exc()
            if os.environ.get("J3D_GROUP_FAILFAST"):
                raise SystemExit(f"first failure after {n} cases")

    if which == "fullsize":
        attempt(run_fullsize, ThreadGroup(2))
        ranks = []
    for nr in ranks:
        G = ThreadGroup(nr)
        g = {2: (48, 40, 64), 4: (48, 64, 64), 8: (48, 48, 48)}[nr]
        if nr == 2:  # J3D_TIMEOUT_S is process-wide: only one rank may be waiting when it is lowered
            attempt(run_api_case, G, g)
            G = ThreadGroup(nr)
        if which == "api":
            continue
        attempt(run_graph_refused, G, g)
        G = ThreadGroup(nr)
        attempt(run_destroy_race, G, g)
        for v, x, la in (("direct", "p2p", "batched"), ("C", "host", "batched"), ("direct", "p2p", "persistent")):
            attempt(run_set_block_case, G, g, 2, v, x, la)
        for c in cases_for(nr, which) * int(os.environ.get("J3D_GROUP_REPEAT", "1")):
            attempt(run_case, G, *c)
    if failed:
        print("\n".join(failed))
        raise SystemExit(f"{len(failed)} of {n} cases failed")
    print(f"GROUP OK {n} cases on ranks {ranks} in {time.time() - t_start:.1f} s", flush=True)


if __name__ == "__main__":
    main()
