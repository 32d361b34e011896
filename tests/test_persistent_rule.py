"""The persistent launch's dependency rule, checked by brute force (CPU).

J3D_PERSISTENT lets an item of iteration k start once the *slabs* (one tile
row of one block over one z chunk) in its dependency list finished iteration
k-1 (setup.cu build_persist_deps).  The rule lists, for slab
(b, zc, ty): itself, (b, zc+-1, ty), (b, zc, ty+-1), the x neighbours'
(zc, ty), for an edge tile row the y neighbour's edge row, for an edge chunk
the z neighbour's edge chunk.

Here every slab's cell sets are enumerated on small decompositions -- the
cells it WRITES (its owned cells in the output buffer, plus the ghost cells
its direct-variant epilogue stores into the neighbours' output buffers) and
the cells it READS (the 7-point neighbourhoods of its owned cells in the input
buffer, ghosts included) -- and every hazard between consecutive iterations
(RAW: k reads what k-1 wrote; WAR: k overwrites what k-1 read, in the same
buffer because the two buffers alternate) must be covered by the rule, and
every listed dependency must be a real hazard.
"""
import itertools

import pytest


def slabs_of(nb, ext, ty_, nzc):
    nx, ny, nz = ext
    nty = -(-ny // ty_)
    zbounds = [(nz * c // nzc, nz * (c + 1) // nzc) for c in range(nzc)]
    return nty, zbounds


def neighbours(nb):
    """Block grid nb -> neighbour block (or None) per face f (0:-x 1:+x 2:-y 3:+y 4:-z 5:+z)."""
    out = {}
    for b in itertools.product(*(range(n) for n in nb)):
        nbr = []
        for f in range(6):
            a, d = f // 2, (1 if f % 2 else -1)
            c = list(b)
            c[a] += d
            nbr.append(tuple(c) if 0 <= c[a] < nb[a] else None)
        out[b] = nbr
    return out


def cell_sets(nb, ext, ty_, nzc):
    """Per slab (b, zc, ty): (reads, writes) as sets of (block, x, y, z) in
    ghosted local coordinates (-1 .. n), for the direct variant."""
    nx, ny, nz = ext
    nty, zb = slabs_of(nb, ext, ty_, nzc)
    nbrs = neighbours(nb)
    sets = {}
    for b in nbrs:
        for zc, (z0, z1) in enumerate(zb):
            for t in range(nty):
                y0, y1 = t * ty_, min(ny, (t + 1) * ty_)
                R, W = set(), set()
                for z in range(z0, z1):
                    for y in range(y0, y1):
                        for x in range(nx):
                            W.add((b, x, y, z))
                            for dx, dy, dz in ((0, 0, 0), (-1, 0, 0), (1, 0, 0), (0, -1, 0), (0, 1, 0),
                                               (0, 0, -1), (0, 0, 1)):
                                R.add((b, x + dx, y + dy, z + dz))
                            # epilogue: a boundary cell is stored into the neighbour's ghost layer
                            for f, (a, edge) in enumerate(((0, 0), (0, nx - 1), (1, 0), (1, ny - 1), (2, 0),
                                                           (2, nz - 1))):
                                n = nbrs[b][f]
                                if n is None or (x, y, z)[a] != edge:
                                    continue
                                g = [x, y, z]
                                g[a] = -1 if f % 2 else (nx, ny, nz)[a]  # lands on the other side
                                W.add((n, *g))
                sets[(b, zc, t)] = (R, W)
    return sets


def rule(nb, ext, ty_, nzc):
    """The dependency rule of setup.cu build_persist_deps."""
    nty, _ = slabs_of(nb, ext, ty_, nzc)
    nbrs = neighbours(nb)
    deps = {}
    for b in nbrs:
        for zc in range(nzc):
            for t in range(nty):
                d = {(b, zc, t)}
                if zc > 0:
                    d.add((b, zc - 1, t))
                if zc + 1 < nzc:
                    d.add((b, zc + 1, t))
                if t > 0:
                    d.add((b, zc, t - 1))
                if t + 1 < nty:
                    d.add((b, zc, t + 1))
                for f in (0, 1):
                    if nbrs[b][f] is not None:
                        d.add((nbrs[b][f], zc, t))
                if t == 0 and nbrs[b][2] is not None:
                    d.add((nbrs[b][2], zc, nty - 1))
                if t == nty - 1 and nbrs[b][3] is not None:
                    d.add((nbrs[b][3], zc, 0))
                if zc == 0 and nbrs[b][4] is not None:
                    d.add((nbrs[b][4], nzc - 1, t))
                if zc == nzc - 1 and nbrs[b][5] is not None:
                    d.add((nbrs[b][5], 0, t))
                deps[(b, zc, t)] = d
    return deps


def used(cells, ext):
    """Drop cells no 7-point stencil ever uses: edge / corner ghosts (two or
    more coordinates outside the owned range)."""
    nx, ny, nz = ext
    keep = set()
    for c in cells:
        x, y, z = c[1:]
        out = (x < 0 or x >= nx) + (y < 0 or y >= ny) + (z < 0 or z >= nz)
        if out <= 1:
            keep.add(c)
    return keep


@pytest.mark.parametrize("nb,ext,ty_,nzc", [
    ((2, 2, 2), (4, 6, 6), 2, 3),    # 8 blocks, 3 tile rows, 3 chunks
    ((1, 3, 2), (3, 5, 4), 2, 2),    # ragged last tile row
    ((2, 1, 1), (4, 4, 4), 4, 1),    # one tile row, one chunk per block
    ((1, 1, 3), (2, 3, 1), 1, 1),    # 1-plane blocks: edge chunk on both sides
    ((2, 2, 1), (3, 2, 5), 1, 5),    # 1-plane chunks, 1-row tiles
])
def test_rule_covers_exactly_the_hazards(nb, ext, ty_, nzc):
    sets = cell_sets(nb, ext, ty_, nzc)
    deps = rule(nb, ext, ty_, nzc)
    for s, (R, W) in sets.items():
        R = used(R, ext)
        need = set()
        for s2, (R2, W2) in sets.items():
            R2 = used(R2, ext)
            if R & W2 or W & R2:  # RAW (k reads what k-1 wrote) or WAR (k overwrites what k-1 read)
                need.add(s2)
        assert need <= deps[s], (s, sorted(need - deps[s]))
        assert deps[s] <= need, (s, sorted(deps[s] - need))
