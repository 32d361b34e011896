"""Shared test helpers: run the oracle and the CUDA path on the same seeded
inputs and compare.  Test infrastructure (may import oracle/)."""
from __future__ import annotations

import numpy as np

from inputs.generators import owned
from oracle import core, twin

KINDS = {"default": core.INIT_DEFAULT, "const": core.INIT_CONST, "linear": core.INIT_LINEAR, "hash": core.INIT_HASH}


def oracle_initial(grid, kind="default", params=(0.0, 0.0, 0.0, 0.0), seed=0, boundary=1.0):
    gx, gy, gz = grid
    return core.init(gx, gy, gz, KINDS[kind], params, seed, boundary)


def gpu_run(ctx, n, kind="default", params=None, seed=0, field=None):
    """Init on the GPU (and optionally overwrite owned cells from a ghosted
    host field), iterate n times, return the assembled owned grid."""
    ctx.init(kind, params, seed)
    if field is not None:
        ctx.scatter_local(owned(field))
    ctx.iterate(n)
    ctx.synchronize()
    return ctx.gather_local()


def assert_bitwise(got: np.ndarray, want: np.ndarray, what=""):
    if got.tobytes() == np.ascontiguousarray(want).tobytes():
        return
    diff = np.argwhere(got.view(np.uint64) != np.ascontiguousarray(want).view(np.uint64))
    k, j, i = diff[0]
    raise AssertionError(f"{what}: {len(diff)} cells differ; first at (x={i},y={j},z={k}): "
                         f"got {got[k, j, i]!r} want {want[k, j, i]!r}")


def hash_value(gx, gy, gz, seed, i, j, k, boundary=1.0):
    """Initial value of global cell (i,j,k) under the HASH init (numpy twin)."""
    if not (0 <= i < gx and 0 <= j < gy and 0 <= k < gz):
        return boundary
    s = twin.splitmix64(np.array([seed], dtype=np.uint64))[0]
    g = np.uint64(i + gx * (j + gy * k))
    return float(twin.splitmix64(np.array([s ^ g], dtype=np.uint64))[0] >> np.uint64(11)) * 2.0 ** -53


def cone_value(grid, seed, n, cell, boundary=1.0):
    """Oracle value of one cell after n iterations of the HASH-initialised
    grid, computed from its dependency cone only: a box of radius n around the
    cell (plus a fixed shell) holds everything the cell can see in n steps
    (each step reaches one cell further), so the sub-box run is exact there."""
    gx, gy, gz = grid
    i, j, k = cell
    R = n
    lo = [max(c - R - 1, -1) for c in (i, j, k)]
    hi = [min(c + R + 1, g) for c, g in zip((i, j, k), grid)]
    xs = np.arange(lo[0], hi[0] + 1)
    ys = np.arange(lo[1], hi[1] + 1)
    zs = np.arange(lo[2], hi[2] + 1)
    Z, Y, X = np.meshgrid(zs, ys, xs, indexing="ij")
    inside = (X >= 0) & (X < gx) & (Y >= 0) & (Y < gy) & (Z >= 0) & (Z < gz)
    A = np.full(X.shape, boundary, dtype=np.float64)
    s = twin.splitmix64(np.array([seed], dtype=np.uint64))[0]
    g = (X[inside].astype(np.uint64) + np.uint64(gx) * (Y[inside].astype(np.uint64)
                                                         + np.uint64(gy) * Z[inside].astype(np.uint64)))
    A[inside] = (twin.splitmix64(s ^ g) >> np.uint64(11)).astype(np.float64) * 2.0 ** -53
    A = np.ascontiguousarray(A)
    R_ = core.run(A, n)
    return R_[k - lo[2], j - lo[1], i - lo[0]]
