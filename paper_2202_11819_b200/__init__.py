"""B200-native Jacobi3D hot path (arXiv 2202.11819, Choi/Richards/Kale).

The product is the C-ABI library ``libjacobi3d.so`` (include/jacobi3d.h):
hand-written sm_100a CUDA kernels plus the per-iteration orchestration
(streams, CUDA graphs, NCCL / NVLink P2P halo exchange).  This package holds
its sources (``csrc/``), the build script and a thin ctypes binding.
"""
from .jacobi3d import (  # noqa: F401
    Jacobi3D, Jacobi3DError, make_config, nccl_unique_id, plan,
    UNFUSED, FUSE_A, FUSE_B, FUSE_C, FUSE_DIRECT, PER_BLOCK, BATCHED,
    XCHG_AUTO, XCHG_NCCL, XCHG_P2P, INIT_DEFAULT, INIT_CONST, INIT_LINEAR, INIT_HASH,
)
