"""J3D_PERSISTENT (one launch per iterate(n) call, on-device slab dependency
tracking between iterations) vs the CPU oracle, bit for bit.

The launch mode changes only WHEN an item of iteration k+1 may start (as soon
as the z-chunk slabs it reads finished iteration k), never what it computes,
so every case must give the oracle's bits (reading R14).  Stress
cases use many short slabs (J3D_ZCHUNK) and many iterations so that a missing
dependency edge would show up as a race.
"""
import numpy as np
import pytest

from oracle import core
from tests.helpers import assert_bitwise, oracle_initial

pytestmark = pytest.mark.gpu

j3d = pytest.importorskip("paper_2202_11819_b200")


def _check(grid, odf, n, kind="hash", seed=3, block=(0, 0, 0), calls=None):
    calls = calls or [n]
    with j3d.Jacobi3D(grid, odf=odf, variant="direct", launch="persistent", block=block) as ctx:
        ctx.init(kind, seed=seed)
        ctx.reset_stats()
        for m in calls:
            ctx.iterate(m)
        ctx.synchronize()
        st = ctx.stats()
        got = ctx.gather_local()
        ck = ctx.checksum()
        res = ctx.residual() if sum(calls) > 0 else None
    total = sum(calls)
    U0 = oracle_initial(grid, kind, (0, 0, 0, 0), seed, 1.0)
    want, prev = core.run_pair(U0, total) if total > 0 else (U0, None)
    tag = f"persistent {grid} odf={odf} calls={calls}"
    assert_bitwise(got, core.owned(want), tag)
    assert ck == core.checksum(want), tag
    if res is not None:
        assert np.float64(res).tobytes() == np.float64(core.residual(want, prev)).tobytes(), tag
    # one stencil launch per non-empty iterate() call, whatever n is
    assert st["kernel_launches"] == sum(1 for m in calls if m > 0), (tag, st)
    return st


@pytest.mark.parametrize("grid,odf,block", [
    ((64, 64, 64), 8, (0, 0, 0)),      # BASELINE configs[0] shape
    ((200, 40, 30), 1, (0, 0, 0)),     # ragged tiles, one block
    ((45, 34, 22), 2, (0, 0, 0)),
    ((132, 72, 33), 4, (0, 0, 0)),
    ((16, 12, 4), 4, (16, 12, 1)),     # 1-cell-thick blocks: z neighbours in every slab
    ((9, 7, 5), 1, (0, 0, 0)),
    ((1, 1, 1), 1, (0, 0, 0)),
    ((48, 48, 48), 27, (0, 0, 0)),     # interior blocks with 6 neighbours
    ((64, 32, 96), 8, (0, 0, 0)),
])
@pytest.mark.parametrize("n", [1, 2, 7, 20])
def test_persistent_shapes(grid, odf, block, n):
    _check(grid, odf, n, block=block)


def test_persistent_default_init_config1():
    _check((64, 64, 64), 8, 20, kind="default")


def test_persistent_split_calls_and_zero():
    """Iterations spread over several calls (the completion counters carry on
    across launches) and n = 0 calls launch nothing."""
    _check((48, 40, 24), 4, 0, calls=[1, 0, 3, 2, 5, 0, 1])


@pytest.mark.parametrize("zchunk", [1, 2, 5])
def test_persistent_many_slabs_stress(zchunk, monkeypatch):
    """Many thin slabs and many iterations: tight dependency chains."""
    monkeypatch.setenv("J3D_ZCHUNK", str(zchunk))
    _check((64, 48, 40), 8, 60, seed=11)
    _check((32, 32, 32), 64, 40, seed=12)


def test_persistent_fine_grained_checksum():
    """96^3-like fine-grained regime (BASELINE configs[4] block shape, scaled):
    64 blocks of 48^3 on one GPU, 50 iterations, checksum and residual vs the
    oracle."""
    grid, n = (192, 192, 192), 50
    with j3d.Jacobi3D(grid, odf=64, variant="direct", launch="persistent") as ctx:
        ctx.init("hash", seed=7)
        ctx.iterate(n)
        ck = ctx.checksum()
        res = ctx.residual()
    want, prev = core.run_pair(core.init(*grid, core.INIT_HASH, seed=7), n)
    assert ck == core.checksum(want)
    assert np.float64(res).tobytes() == np.float64(core.residual(want, prev)).tobytes()


def test_persistent_matches_batched_long_run():
    """1000 iterations in one launch agree bit for bit with the batched mode
    (itself pinned to the oracle elsewhere) on a grid with 27 blocks."""
    grid = (72, 60, 48)
    out = {}
    for launch in ("persistent", "batched"):
        with j3d.Jacobi3D(grid, odf=27, variant="direct", launch=launch) as ctx:
            ctx.init("hash", seed=21)
            ctx.iterate(1000)
            out[launch] = (ctx.checksum(), ctx.residual())
    assert out["persistent"][0] == out["batched"][0]
    assert np.float64(out["persistent"][1]).tobytes() == np.float64(out["batched"][1]).tobytes()


def test_persistent_rejects_other_variants():
    for kw in ({"variant": "unfused"}, {"variant": "C"}, {"graph": True}):
        args = {"variant": "direct", "launch": "persistent"}
        args.update(kw)
        with pytest.raises(j3d.Jacobi3DError) as e:
            j3d.Jacobi3D((16, 16, 16), **args)
        assert e.value.code == -1
