"""Randomised CPU tests of jacobi3d_plan (no GPU) against the brute-force
decomposition oracle (oracle/decompose.py, SPEC.md
L358-384) and against face counts derived from the block grid by hand:
a GPU at position p of the GPU grid has one peer face per block on each of
its sides that touches another GPU; every block face inside a GPU's block
grid is a local face (counted once from each side)."""
import itertools

import pytest
from hypothesis import given, settings, strategies as st

from oracle.decompose import DecompositionError, plan as oracle_plan

j3d = pytest.importorskip("paper_2202_11819_b200")


def expected_faces(gpu, blk):
    peer_max = 0
    for pos in itertools.product(*(range(p) for p in gpu)):
        cnt = 0
        for a in range(3):
            side = blk[(a + 1) % 3] * blk[(a + 2) % 3]  # blocks on one face of the GPU's sub-grid
            cnt += side * ((pos[a] > 0) + (pos[a] < gpu[a] - 1))
        peer_max = max(peer_max, cnt)
    local = sum(2 * (blk[a] - 1) * blk[(a + 1) % 3] * blk[(a + 2) % 3] for a in range(3))
    return peer_max, local


# mostly composite extents so that most draws decompose; plain integers keep the error path covered
dims = st.one_of(st.integers(min_value=1, max_value=240), st.integers(min_value=1, max_value=40).map(lambda k: 6 * k),
                 st.integers(min_value=1, max_value=15).map(lambda k: 16 * k))


@settings(max_examples=400, deadline=None)
@given(gx=dims, gy=dims, gz=dims, n=st.sampled_from([1, 2, 3, 4, 6, 8, 12, 16]),
       odf=st.sampled_from([1, 2, 3, 4, 6, 8, 9, 12, 16, 27, 32, 64]))
def test_plan_random_grids(gx, gy, gz, n, odf):
    g = (gx, gy, gz)
    try:
        gpu, blk, ext = oracle_plan(g, n, odf)
    except DecompositionError:
        with pytest.raises(j3d.Jacobi3DError) as e:
            j3d.plan(g, odf=odf, n_gpus=n)
        assert e.value.code == -2
        return
    got = j3d.plan(g, odf=odf, n_gpus=n)
    assert (got["gpu_grid"], got["blk_grid"], got["blk_ext"]) == (gpu, blk, ext)
    assert got["n_blocks"] == odf * n
    peer_max, local = expected_faces(gpu, blk)
    assert got["peer_faces_max"] == peer_max
    assert got["local_faces"] == local
    for r in range(1, n):  # every rank plans the same grid; local faces are position-independent
        other = j3d.plan(g, odf=odf, n_gpus=n, rank=r)
        assert other["gpu_grid"] == got["gpu_grid"] and other["local_faces"] == local
