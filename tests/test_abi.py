"""CPU tests of the boundary: the C-ABI library loads without a GPU, exports
every symbol include/*.h declares, and its planner (jacobi3d_plan, no GPU)
agrees with the brute-force decomposition oracle."""
import ctypes
import glob
import itertools
import os
import re

import pytest

from oracle.decompose import DecompositionError, plan as oracle_plan, plan_with_blocks

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
LIB = os.path.join(ROOT, "paper_2202_11819_b200", "libjacobi3d.so")


def declared_symbols():
    names = set()
    for h in glob.glob(os.path.join(ROOT, "include", "*.h")):
        src = open(h).read()
        names |= set(re.findall(r"^J3D_API\s+[\w\s\*]+?\b(jacobi3d_\w+)\s*\(", src, flags=re.M))
    return names


def test_library_exports_every_declared_symbol():
    assert os.path.exists(LIB), "build with python paper_2202_11819_b200/build.py"
    lib = ctypes.CDLL(LIB)
    names = declared_symbols()
    assert len(names) >= 20
    missing = [n for n in names if not hasattr(lib, n)]
    assert not missing, missing


def test_binding_names_match_header():
    import paper_2202_11819_b200.jacobi3d as b

    src = open(b.__file__).read()
    for n in declared_symbols():
        assert n in src, n


def test_plan_matches_oracle():
    import paper_2202_11819_b200 as j3d

    grids = [(64, 64, 64), (1536, 1536, 1536), (1536, 1536, 3072), (3072, 3072, 3072), (768, 768, 768),
             (48, 40, 24), (45, 34, 22), (132, 72, 33), (16, 12, 4), (192, 192, 192), (100, 60, 36)]
    for g, n, odf in itertools.product(grids, (1, 2, 4, 6, 8), (1, 2, 4, 8, 16, 27, 32, 64)):
        try:
            want = oracle_plan(g, n, odf)
        except DecompositionError:
            with pytest.raises(j3d.Jacobi3DError) as e:
                j3d.plan(g, odf=odf, n_gpus=n)
            assert e.value.code == -2
            continue
        got = j3d.plan(g, odf=odf, n_gpus=n)
        assert (got["gpu_grid"], got["blk_grid"], got["blk_ext"]) == want, (g, n, odf)
        assert got["n_blocks"] == odf * n


def test_plan_user_blocks_and_errors():
    import paper_2202_11819_b200 as j3d

    assert j3d.plan((16, 12, 4), odf=4, block=(16, 12, 1))["blk_grid"] == plan_with_blocks((16, 12, 4), 1, 4, (16, 12, 1))[1]
    with pytest.raises(j3d.Jacobi3DError) as e:
        j3d.plan((8, 8, 8), odf=2, block=(8, 8, 3))
    assert e.value.code == -2
    with pytest.raises(j3d.Jacobi3DError) as e:
        j3d.plan((0, 8, 8))
    assert e.value.code == -1
    with pytest.raises(j3d.Jacobi3DError) as e:
        j3d.plan((8, 8, 8), n_gpus=2, rank=2)
    assert e.value.code == -1


def test_plan_peer_faces():
    """(a).1/§8(e): peer faces per GPU 0/1/2/3 at 1/2/4/8 GPUs (ODF=1)."""
    import paper_2202_11819_b200 as j3d

    for n, g, want in ((1, (1536,) * 3, 0), (2, (1536, 1536, 3072), 1), (4, (1536, 3072, 3072), 2),
                       (8, (3072,) * 3, 3)):
        assert j3d.plan(g, n_gpus=n)["peer_faces_max"] == want


def test_persistent_launch_validation():
    """J3D_PERSISTENT is the direct variant without graphs, across GPUs over P2P
    only; anything else is rejected by the shared config check (jacobi3d_plan,
    no GPU)."""
    import paper_2202_11819_b200 as j3d
    from paper_2202_11819_b200 import jacobi3d as jb

    def rc(**kw):
        cfg = jb.make_config((16, 16, 16), **kw)
        return jb.lib.jacobi3d_plan(ctypes.byref(cfg), ctypes.byref(jb.PlanInfo()))

    assert jb.LAUNCHES["persistent"] == jb.PERSISTENT == 2
    assert rc(variant="direct", launch="persistent") == 0
    assert rc(variant="direct", launch="persistent", odf=8) == 0
    assert rc(variant="unfused", launch="persistent") == jb.EINVAL
    assert rc(variant="C", launch="persistent") == jb.EINVAL
    assert rc(variant="direct", launch="persistent", graph=True) == jb.EINVAL
    assert rc(variant="direct", launch="persistent", n_gpus=2) == 0             # P2P (auto) across GPUs
    assert rc(variant="direct", launch="persistent", n_gpus=2, exchange="p2p") == 0
    assert rc(variant="direct", launch="persistent", n_gpus=2, exchange="nccl") == jb.EINVAL
    assert rc(variant="direct", launch="persistent", n_gpus=2, exchange="host") == jb.EINVAL
    cfg = jb.make_config((16, 16, 16))
    cfg.launch = 3
    assert jb.lib.jacobi3d_plan(ctypes.byref(cfg), ctypes.byref(jb.PlanInfo())) == jb.EINVAL
    del j3d


def test_binding_constants_match_header():
    """Every J3D_* constant the ctypes binding mirrors has the header's value."""
    import paper_2202_11819_b200.jacobi3d as b

    hdr = {}
    for h in glob.glob(os.path.join(ROOT, "include", "*.h")):
        for name, val in re.findall(r"^#define\s+J3D_(\w+)\s+(-?\d+)\b", open(h).read(), flags=re.M):
            hdr[name] = int(val)
    pairs = {"OK": b.OK, "EINVAL": b.EINVAL, "EDECOMP": b.EDECOMP, "ENOMEM": b.ENOMEM, "ECUDA": b.ECUDA,
             "ENCCL": b.ENCCL, "ENOTLOCAL": b.ENOTLOCAL, "ESTATE": b.ESTATE, "ETIMEOUT": b.ETIMEOUT,
             "EUNSUPPORTED": b.EUNSUPPORTED, "UNFUSED": b.UNFUSED, "FUSE_A": b.FUSE_A, "FUSE_B": b.FUSE_B,
             "FUSE_C": b.FUSE_C, "FUSE_DIRECT": b.FUSE_DIRECT, "PER_BLOCK": b.PER_BLOCK, "BATCHED": b.BATCHED,
             "PERSISTENT": b.PERSISTENT, "XCHG_AUTO": b.XCHG_AUTO, "XCHG_NCCL": b.XCHG_NCCL,
             "XCHG_P2P": b.XCHG_P2P, "XCHG_HOST": b.XCHG_HOST, "INIT_DEFAULT": b.INIT_DEFAULT,
             "INIT_CONST": b.INIT_CONST, "INIT_LINEAR": b.INIT_LINEAR, "INIT_HASH": b.INIT_HASH}
    for k, v in pairs.items():
        assert hdr.get(k) == v, (k, hdr.get(k), v)
    assert ctypes.sizeof(b.Config) == 8 * 6 + 4 * 10 + 8  # jacobi3d_config: 6 int64, 10 int32, 1 double
    assert ctypes.sizeof(b.Stats) == 8 * 7  # jacobi3d_stats: 7 int64
