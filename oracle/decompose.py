"""Brute-force surface-minimising 3D decomposition (the planner's oracle).

TEST INFRASTRUCTURE ONLY (see ``oracle/__init__.py``).

PAPER.md L562-565 (Sec. 4.1): "the global grid is divided into six
equal-sized blocks; the grid is decomposed in a way that minimizes the
aggregate surface area, which is tied to communication volume."  The paper
does not state a tie-break or what happens when a dimension does not divide;
SPEC.md L358-361/L376-384 fix both (reading R9): enumerate every
ordered factor triple (px,py,pz) with px*py*pz = n whose factors divide the
corresponding dimension, minimise the aggregate surface
n * 2*(bx*by + by*bz + bx*bz), ties -> lexicographically smallest triple;
no divisible triple -> error naming a failing dimension.

Hierarchical plan (reading R10): GPU grid first over n_gpus on the
global dims, then the per-GPU block grid over ODF on the per-GPU dims.
"""
from __future__ import annotations


class DecompositionError(ValueError):
    pass


def decompose(dims, n):
    gx, gy, gz = dims
    if n < 1 or min(dims) < 1:
        raise DecompositionError("extents and part count must be >= 1")
    best = None
    failing = set()
    for px in range(1, n + 1):
        if n % px:
            continue
        for py in range(1, n // px + 1):
            if (n // px) % py:
                continue
            pz = n // (px * py)
            bad = [name for name, g, p in (("x", gx, px), ("y", gy, py), ("z", gz, pz)) if g % p]
            if bad:
                failing.update(bad)
                continue
            bx, by, bz = gx // px, gy // py, gz // pz
            area = n * 2 * (bx * by + by * bz + bx * bz)
            key = (area, (px, py, pz))
            if best is None or key < best:
                best = key
    if best is None:
        raise DecompositionError(f"no divisible factorisation of {n} parts; failing dimension(s): {sorted(failing)}")
    return best[1]


def plan(gdims, n_gpus, odf):
    """Return (gpu_grid, blk_grid, blk_ext) for the hierarchical plan."""
    gpu = decompose(gdims, n_gpus)
    per_gpu = tuple(g // p for g, p in zip(gdims, gpu))
    blk = decompose(per_gpu, odf)
    ext = tuple(g // b for g, b in zip(per_gpu, blk))
    return gpu, blk, ext


def plan_with_blocks(gdims, n_gpus, odf, bdims):
    """Plan with user-given block extents: GPU grid as above, block grid =
    per-GPU dims / block dims, whose product must equal ODF."""
    gpu = decompose(gdims, n_gpus)
    per_gpu = tuple(g // p for g, p in zip(gdims, gpu))
    for name, g, b in zip("xyz", per_gpu, bdims):
        if b < 1 or g % b:
            raise DecompositionError(f"block extent does not divide per-GPU extent along {name}")
    blk = tuple(g // b for g, b in zip(per_gpu, bdims))
    if blk[0] * blk[1] * blk[2] != odf:
        raise DecompositionError("blocks per GPU != ODF")
    return gpu, blk, tuple(bdims)


def footprint_bytes(dims, parts):
    """SPEC.md L467-474 memory_footprint: 2 x block elements x 8 bytes."""
    px, py, pz = parts
    return 2 * (dims[0] // px) * (dims[1] // py) * (dims[2] // pz) * 8
