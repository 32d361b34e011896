"""Thin ctypes binding of libjacobi3d.so (include/jacobi3d.h).

Argument marshalling only: every step of the hot path runs in the library's
CUDA kernels.  There is no CPU fallback: if the library is missing this
module raises ImportError.
"""
from __future__ import annotations

import ctypes
import os

import numpy as np

_HERE = os.path.dirname(os.path.abspath(__file__))
LIB_PATH = os.path.join(_HERE, os.environ.get("J3D_LIB", "libjacobi3d.so"))  # J3D_LIB: experiment builds

# status codes
OK, EINVAL, EDECOMP, ENOMEM, ECUDA, ENCCL, ENOTLOCAL, ESTATE, ETIMEOUT, EUNSUPPORTED = 0, -1, -2, -3, -4, -5, -6, -7, -8, -9
# variants (PAPER.md L515-521 strategies A/B/C + the direct-ghost B200 variant)
UNFUSED, FUSE_A, FUSE_B, FUSE_C, FUSE_DIRECT = 0, 1, 2, 3, 4
VARIANTS = {"unfused": UNFUSED, "A": FUSE_A, "B": FUSE_B, "C": FUSE_C, "direct": FUSE_DIRECT}
PER_BLOCK, BATCHED, PERSISTENT = 0, 1, 2
LAUNCHES = {"per_block": PER_BLOCK, "batched": BATCHED, "persistent": PERSISTENT}
XCHG_AUTO, XCHG_NCCL, XCHG_P2P, XCHG_HOST = 0, 1, 2, 3
EXCHANGES = {"auto": XCHG_AUTO, "nccl": XCHG_NCCL, "p2p": XCHG_P2P, "host": XCHG_HOST}
INIT_DEFAULT, INIT_CONST, INIT_LINEAR, INIT_HASH = 0, 1, 2, 3
INITS = {"default": INIT_DEFAULT, "const": INIT_CONST, "linear": INIT_LINEAR, "hash": INIT_HASH}


class Config(ctypes.Structure):
    _fields_ = [("gx", ctypes.c_int64), ("gy", ctypes.c_int64), ("gz", ctypes.c_int64),
                ("bx", ctypes.c_int64), ("by", ctypes.c_int64), ("bz", ctypes.c_int64),
                ("odf", ctypes.c_int32), ("n_gpus", ctypes.c_int32), ("rank", ctypes.c_int32),
                ("device", ctypes.c_int32), ("variant", ctypes.c_int32), ("launch", ctypes.c_int32),
                ("use_graph", ctypes.c_int32), ("exchange", ctypes.c_int32), ("overlap", ctypes.c_int32),
                ("reserved", ctypes.c_int32), ("boundary", ctypes.c_double)]


class PlanInfo(ctypes.Structure):
    _fields_ = [("gpu_grid", ctypes.c_int32 * 3), ("blk_grid", ctypes.c_int32 * 3), ("blk_ext", ctypes.c_int64 * 3),
                ("n_blocks", ctypes.c_int64), ("bytes_per_gpu", ctypes.c_int64),
                ("peer_faces_max", ctypes.c_int32), ("local_faces", ctypes.c_int32)]


class Stats(ctypes.Structure):
    _fields_ = [("iterations", ctypes.c_int64), ("kernel_launches", ctypes.c_int64),
                ("graph_launches", ctypes.c_int64), ("last_graph_parity", ctypes.c_int64),
                ("launches_per_iter_block", ctypes.c_int64), ("tile_kind", ctypes.c_int64),
                ("work_items", ctypes.c_int64)]


class Jacobi3DError(RuntimeError):
    def __init__(self, code: int, msg: str):
        super().__init__(f"[{code}] {msg}")
        self.code = code


def _load():
    if not os.path.exists(LIB_PATH):
        raise ImportError(f"{LIB_PATH} is missing: build it with `python -m paper_2202_11819_b200.build` "
                          "(there is no CPU fallback)")
    L = ctypes.CDLL(LIB_PATH)
    P, I64, I32, D, U64 = ctypes.c_void_p, ctypes.c_int64, ctypes.c_int32, ctypes.c_double, ctypes.c_uint64
    sig = {
        "jacobi3d_plan": [ctypes.POINTER(Config), ctypes.POINTER(PlanInfo)],
        "jacobi3d_nccl_unique_id": [P],
        "jacobi3d_create": [ctypes.POINTER(Config), P, ctypes.POINTER(P)],
        "jacobi3d_ipc_export": [P, P, ctypes.c_size_t, ctypes.POINTER(ctypes.c_size_t)],
        "jacobi3d_ipc_connect": [P, P, ctypes.c_size_t],
        "jacobi3d_init": [P, ctypes.c_int, P, U64],
        "jacobi3d_set_block": [P, I64, P],
        "jacobi3d_refresh_halos": [P],
        "jacobi3d_iterate": [P, I64],
        "jacobi3d_synchronize": [P],
        "jacobi3d_get_block": [P, I64, P],
        "jacobi3d_block_info": [P, I64, P, P, P],
        "jacobi3d_get_region": [P, I64, P, P, P],
        "jacobi3d_residual": [P, ctypes.POINTER(D)],
        "jacobi3d_checksum": [P, ctypes.POINTER(U64)],
        "jacobi3d_time": [P, I64, I64, ctypes.POINTER(D)],
        "jacobi3d_get_stats": [P, ctypes.POINTER(Stats)],
        "jacobi3d_reset_stats": [P],
        "jacobi3d_profile_enable": [P, ctypes.c_int],
        "jacobi3d_profile_read": [P, ctypes.POINTER(D), ctypes.POINTER(I64), ctypes.POINTER(D)],
        "jacobi3d_set_skip_exchange": [P, ctypes.c_int],
        "jacobi3d_debug_slab_deps": [ctypes.POINTER(Config), I32, I32, P, I64, ctypes.POINTER(I64)],
        "jacobi3d_debug_control": [P, I32, I32, I64, P, P, P],
        "jacobi3d_destroy": [P],
        "jacobi3d_div7_selftest": [U64, U64, ctypes.POINTER(U64), P],
    }
    for name, args in sig.items():
        fn = getattr(L, name)
        fn.argtypes = args
        fn.restype = ctypes.c_int
    L.jacobi3d_last_error.argtypes = []
    L.jacobi3d_last_error.restype = ctypes.c_char_p
    return L


lib = _load()


def _ck(rc: int) -> None:
    if rc != OK:
        raise Jacobi3DError(rc, lib.jacobi3d_last_error().decode(errors="replace"))


def _enum(table, v):
    return table[v] if isinstance(v, str) else int(v)


def make_config(grid, odf=1, n_gpus=1, rank=0, device=0, block=(0, 0, 0), variant="direct", launch="batched",
                graph=False, exchange="auto", boundary=1.0, overlap=False) -> Config:
    gx, gy, gz = grid
    bx, by, bz = block
    return Config(gx, gy, gz, bx, by, bz, odf, n_gpus, rank, device, _enum(VARIANTS, variant),
                  _enum(LAUNCHES, launch), int(bool(graph)), _enum(EXCHANGES, exchange), int(bool(overlap)), 0,
                  boundary)


def plan(grid, odf=1, n_gpus=1, block=(0, 0, 0), rank=0, launch="batched") -> dict:
    """jacobi3d_plan: decomposition without a GPU."""
    cfg = make_config(grid, odf=odf, n_gpus=n_gpus, rank=rank, block=block, launch=launch)
    info = PlanInfo()
    _ck(lib.jacobi3d_plan(ctypes.byref(cfg), ctypes.byref(info)))
    return {"gpu_grid": tuple(info.gpu_grid), "blk_grid": tuple(info.blk_grid), "blk_ext": tuple(info.blk_ext),
            "n_blocks": info.n_blocks, "bytes_per_gpu": info.bytes_per_gpu,
            "peer_faces_max": info.peer_faces_max, "local_faces": info.local_faces}


def debug_slab_deps(grid, odf=1, n_gpus=1, rank=0, tile_ty=1, nzc=1, block=(0, 0, 0)) -> np.ndarray:
    """jacobi3d_debug_slab_deps (no GPU): the persistent launch's dependency
    lists of one rank, rows (block, zc, ty, dep_rank, dep_block, dep_zc, dep_ty)."""
    cfg = make_config(grid, odf=odf, n_gpus=n_gpus, rank=rank, block=block, launch="persistent")
    n = ctypes.c_int64()
    _ck(lib.jacobi3d_debug_slab_deps(ctypes.byref(cfg), tile_ty, nzc, None, 0, ctypes.byref(n)))
    out = np.zeros((n.value, 7), dtype=np.int64)
    _ck(lib.jacobi3d_debug_slab_deps(ctypes.byref(cfg), tile_ty, nzc, out.ctypes.data, n.value, ctypes.byref(n)))
    return out


def debug_control(key: bytes, rank: int, n_ranks: int, values) -> tuple[list[int], list[int]]:
    """jacobi3d_debug_control (no GPU): sum and max over ranks of values[r] for every
    round r through the shared-memory control plane; collective over n_ranks
    concurrent callers (threads or processes) with the same key."""
    vals = np.ascontiguousarray(np.asarray(values, dtype=np.uint64))
    n = len(vals)
    s_out = np.zeros(n, dtype=np.uint64)
    m_out = np.zeros(n, dtype=np.uint64)
    kb = (ctypes.c_uint8 * 128).from_buffer_copy(key)
    _ck(lib.jacobi3d_debug_control(kb, rank, n_ranks, n, vals.ctypes.data, s_out.ctypes.data, m_out.ctypes.data))
    return [int(x) for x in s_out], [int(x) for x in m_out]


def nccl_unique_id() -> bytes:
    buf = (ctypes.c_uint8 * 128)()
    _ck(lib.jacobi3d_nccl_unique_id(buf))
    return bytes(buf)


def div7_selftest(n: int, seed: int = 1):
    """Kernel division by 7 vs the IEEE routine on the current device."""
    bad = ctypes.c_uint64()
    ex = (ctypes.c_double * 3)()
    _ck(lib.jacobi3d_div7_selftest(n, seed, ctypes.byref(bad), ex))
    return bad.value, tuple(ex)


class Jacobi3D:
    """One rank's Jacobi3D context (jacobi3d_create ... jacobi3d_destroy)."""

    def __init__(self, grid, odf=1, n_gpus=1, rank=0, device=0, block=(0, 0, 0), variant="direct",
                 launch="batched", graph=False, exchange="auto", boundary=1.0, nccl_uid: bytes | None = None,
                 overlap=False):
        self.cfg = make_config(grid, odf, n_gpus, rank, device, block, variant, launch, graph, exchange, boundary,
                               overlap)
        self._h = ctypes.c_void_p()
        uid = None
        if nccl_uid is not None:
            uid = (ctypes.c_uint8 * 128).from_buffer_copy(nccl_uid)
        _ck(lib.jacobi3d_create(ctypes.byref(self.cfg), uid, ctypes.byref(self._h)))
        self.grid = tuple(grid)
        info = plan(grid, odf=odf, n_gpus=n_gpus, block=block, rank=rank)
        self.plan = info
        self.extent = info["blk_ext"]
        self.n_blocks = info["n_blocks"]

    # -- lifecycle
    def close(self):
        if self._h:
            _ck(lib.jacobi3d_destroy(self._h))
            self._h = ctypes.c_void_p()

    def __enter__(self):
        return self

    def __exit__(self, *a):
        self.close()

    def __del__(self):
        try:
            self.close()
        except Exception:
            pass

    # -- P2P bootstrap
    def ipc_export(self) -> bytes:
        buf = (ctypes.c_uint8 * 4096)()
        n = ctypes.c_size_t()
        _ck(lib.jacobi3d_ipc_export(self._h, buf, 4096, ctypes.byref(n)))
        return bytes(buf[: n.value])

    def ipc_connect(self, records: list[bytes]) -> None:
        ln = len(records[0])
        blob = b"".join(records)
        assert all(len(r) == ln for r in records)
        cbuf = (ctypes.c_uint8 * len(blob)).from_buffer_copy(blob)
        _ck(lib.jacobi3d_ipc_connect(self._h, cbuf, ln))

    # -- state
    def init(self, kind="default", params=None, seed=0):
        p = None
        if params is not None:
            arr = (ctypes.c_double * 4)(*(list(params) + [0.0] * (4 - len(params))))
            p = arr
        _ck(lib.jacobi3d_init(self._h, _enum(INITS, kind), p, seed))

    def set_block(self, block_id: int, data: np.ndarray):
        a = np.ascontiguousarray(data, dtype=np.float64)
        ex = self.extent
        assert a.shape == (ex[2], ex[1], ex[0]), (a.shape, ex)
        _ck(lib.jacobi3d_set_block(self._h, block_id, a.ctypes.data))

    def set_block_ptr(self, block_id: int, host_ptr: int):
        _ck(lib.jacobi3d_set_block(self._h, block_id, host_ptr))

    def get_block(self, block_id: int, out: np.ndarray | None = None) -> np.ndarray:
        ex = self.extent
        if out is None:
            out = np.empty((ex[2], ex[1], ex[0]), dtype=np.float64)
        assert out.flags["C_CONTIGUOUS"] and out.dtype == np.float64 and out.size == ex[0] * ex[1] * ex[2]
        _ck(lib.jacobi3d_get_block(self._h, block_id, out.ctypes.data))
        return out

    def get_region(self, block_id: int, lo, ext) -> np.ndarray:
        out = np.empty((ext[2], ext[1], ext[0]), dtype=np.float64)
        clo = (ctypes.c_int64 * 3)(*lo)
        cex = (ctypes.c_int64 * 3)(*ext)
        _ck(lib.jacobi3d_get_region(self._h, block_id, clo, cex, out.ctypes.data))
        return out

    def get_block_ptr(self, block_id: int, host_ptr: int):
        _ck(lib.jacobi3d_get_block(self._h, block_id, host_ptr))

    def block_info(self, block_id: int):
        o = (ctypes.c_int64 * 3)()
        e = (ctypes.c_int64 * 3)()
        r = ctypes.c_int32()
        _ck(lib.jacobi3d_block_info(self._h, block_id, o, e, ctypes.byref(r)))
        return tuple(o), tuple(e), r.value

    def refresh_halos(self):
        _ck(lib.jacobi3d_refresh_halos(self._h))

    def iterate(self, n: int):
        _ck(lib.jacobi3d_iterate(self._h, n))

    def synchronize(self):
        _ck(lib.jacobi3d_synchronize(self._h))

    def residual(self) -> float:
        d = ctypes.c_double()
        _ck(lib.jacobi3d_residual(self._h, ctypes.byref(d)))
        return d.value

    def checksum(self) -> int:
        u = ctypes.c_uint64()
        _ck(lib.jacobi3d_checksum(self._h, ctypes.byref(u)))
        return u.value

    def time(self, warmup: int, iters: int) -> float:
        d = ctypes.c_double()
        _ck(lib.jacobi3d_time(self._h, warmup, iters, ctypes.byref(d)))
        return d.value

    def stats(self) -> dict:
        s = Stats()
        _ck(lib.jacobi3d_get_stats(self._h, ctypes.byref(s)))
        return {k: getattr(s, k) for k, _ in Stats._fields_}

    def reset_stats(self):
        _ck(lib.jacobi3d_reset_stats(self._h))

    def profile_enable(self, on: bool = True):
        _ck(lib.jacobi3d_profile_enable(self._h, int(on)))

    def profile_read(self):
        ms, n, b = ctypes.c_double(), ctypes.c_int64(), ctypes.c_double()
        _ck(lib.jacobi3d_profile_read(self._h, ctypes.byref(ms), ctypes.byref(n), ctypes.byref(b)))
        return ms.value, n.value, b.value

    def set_skip_exchange(self, skip: bool):
        _ck(lib.jacobi3d_set_skip_exchange(self._h, int(skip)))

    # -- convenience: assemble this rank's blocks into a global array (owned cells only)
    def gather_local(self, out: np.ndarray | None = None) -> np.ndarray:
        gx, gy, gz = self.grid
        if out is None:
            out = np.full((gz, gy, gx), np.nan)
        for b in range(self.n_blocks):
            (ox, oy, oz), (ex, ey, ez), owner = self.block_info(b)
            if owner != self.cfg.rank:
                continue
            out[oz:oz + ez, oy:oy + ey, ox:ox + ex] = self.get_block(b)
        return out

    def scatter_local(self, field: np.ndarray):
        """Upload the owned cells of this rank's blocks from a global (gz,gy,gx) array."""
        for b in range(self.n_blocks):
            (ox, oy, oz), (ex, ey, ez), owner = self.block_info(b)
            if owner != self.cfg.rank:
                continue
            self.set_block(b, field[oz:oz + ez, oy:oy + ey, ox:ox + ex])
