"""The persistent launch's dependency tables, checked by brute force (CPU).

J3D_PERSISTENT lets an item of iteration k start once the *slabs* (one tile
row of one block over one z chunk) in its dependency list finished iteration
k-1.  The lists are taken from the library itself
(jacobi3d_debug_slab_deps: the same setup.cu slab_dep_refs that fills the
device tables, local and peer-tagged entries) for 1-, 2-, 4- and 8-rank
plans.

Here every slab's cell sets are enumerated on small decompositions -- the
cells it WRITES (its owned cells in the output buffer, plus the ghost cells
its direct-variant epilogue stores into the neighbours' output buffers) and
the cells it READS (the 7-point neighbourhoods of its owned cells in the input
buffer, ghosts included) -- and every hazard between consecutive iterations
(RAW: k reads what k-1 wrote; WAR: k overwrites what k-1 read, in the same
buffer because the two buffers alternate) must be in the library's list, and
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


def library_tables(grid, odf, n_gpus, ty_, nzc):
    """The library's lists for every rank (jacobi3d_debug_slab_deps, the code
    that fills the device tables), keyed by slab (block position, zc, ty),
    plus the block grid, block extent and the owner rank of every block."""
    from paper_2202_11819_b200 import jacobi3d as jb

    info = jb.plan(grid, odf=odf, n_gpus=n_gpus)
    nb = tuple(g * b for g, b in zip(info["gpu_grid"], info["blk_grid"]))
    ext = tuple(info["blk_ext"])

    def pos(i):  # block id: x-fastest on the global block grid (jacobi3d.h)
        return (int(i) % nb[0], int(i) // nb[0] % nb[1], int(i) // (nb[0] * nb[1]))

    deps, owner = {}, {}
    for r in range(n_gpus):
        rows = jb.debug_slab_deps(grid, odf=odf, n_gpus=n_gpus, rank=r, tile_ty=ty_, nzc=nzc)
        for b, zc, t, dr, db, dzc, dt in rows.tolist():
            key = (pos(b), zc, t)
            assert owner.setdefault(pos(b), r) == r, "a block listed by two ranks"
            deps.setdefault(key, set()).add((pos(db), dzc, dt, dr))
    return nb, ext, deps, owner


@pytest.mark.parametrize("grid,odf,n_gpus,ty_,nzc", [
    ((8, 12, 12), 8, 1, 2, 3),     # 1 rank: 8 blocks 4x6x6, 3 tile rows, 3 chunks
    ((3, 15, 8), 6, 1, 2, 2),      # ragged last tile row (5 rows, tiles of 2)
    ((8, 4, 4), 2, 1, 4, 1),       # one tile row, one chunk per block
    ((2, 3, 3), 3, 1, 1, 1),       # 1-plane blocks: an edge chunk on both sides
    ((6, 2, 5), 4, 1, 1, 5),       # 1-plane chunks, 1-row tiles
    ((8, 8, 8), 4, 2, 2, 2),       # 2 ranks: peer z faces
    ((16, 6, 6), 4, 2, 3, 3),      # 2 ranks split along x: peer x faces
    ((8, 8, 8), 1, 8, 2, 2),       # 8 ranks on the (2,2,2) grid: every face kind is a peer face
    ((8, 12, 8), 2, 8, 2, 2),      # 8 ranks, 2 blocks each
    ((12, 8, 8), 1, 4, 3, 2),      # 4 ranks (1,2,2)-like, ragged tile rows
])
def test_library_tables_equal_the_hazards(grid, odf, n_gpus, ty_, nzc):
    """Every slab's list in the library's tables (local and peer-tagged entries,
    from jacobi3d_debug_slab_deps) equals the set of slabs it has a hazard with
    across consecutive iterations -- RAW (k reads what k-1 wrote) or WAR (k
    overwrites what k-1 read) -- computed by brute force from the cell sets;
    and an entry's rank is the owner of the listed block."""
    nb, ext, deps, owner = library_tables(grid, odf, n_gpus, ty_, nzc)
    sets = cell_sets(nb, ext, ty_, nzc)
    assert set(deps) == set(sets), "the tables cover exactly the slabs of the decomposition"
    for s, (R, W) in sets.items():
        R = used(R, ext)
        need = set()
        for s2, (R2, W2) in sets.items():
            if R & W2 or W & used(R2, ext):
                need.add(s2)
        got = {d[:3] for d in deps[s]}
        assert len(got) == len(deps[s]), (s, "duplicate entries")
        assert got == need, (s, sorted(need - got), sorted(got - need))
        for d in deps[s]:
            assert d[3] == owner[d[0]], (s, d)
