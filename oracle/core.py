"""ctypes wrapper of the plain-C Jacobi3D oracle (``oracle/jacobi3d_oracle.c``).

TEST INFRASTRUCTURE ONLY (see ``oracle/__init__.py``).

Every array handled here is the undecomposed grid *with* its ghost shell,
shape ``(gz+2, gy+2, gx+2)`` (x fastest), fp64.  ``owned(U)`` returns the
``(gz, gy, gx)`` view of the owned cells.

Definition followed: SURVEY.md §8(c) / DESIGN.md readings R1-R6, i.e. the
7-point average of SPEC.md L388 in the order self,-x,+x,-y,+y,-z,+z, IEEE
division by 7, Dirichlet ghost shell, two buffers (PAPER.md
L480-484).
"""
from __future__ import annotations

import ctypes
import os
import subprocess
import sys

import numpy as np

_HERE = os.path.dirname(os.path.abspath(__file__))
_SRC = os.path.join(_HERE, "jacobi3d_oracle.c")
_LIB = os.path.join(_HERE, "liboracle_jacobi3d.so")

INIT_DEFAULT, INIT_CONST, INIT_LINEAR, INIT_HASH = 0, 1, 2, 3

CFLAGS = ["-O2", "-fno-fast-math", "-ffp-contract=off", "-fopenmp", "-fPIC", "-shared", "-std=c11"]


def build(force: bool = False) -> str:
    """Compile the C oracle with gcc (no FMA contraction, no fast-math)."""
    if force or not os.path.exists(_LIB) or os.path.getmtime(_LIB) < os.path.getmtime(_SRC):
        tmp = _LIB + f".tmp{os.getpid()}"
        subprocess.check_call(["gcc", *CFLAGS, _SRC, "-o", tmp, "-lm"])
        os.replace(tmp, _LIB)
    return _LIB


_lib = None


def lib() -> ctypes.CDLL:
    global _lib
    if _lib is None:
        build()
        L = ctypes.CDLL(_LIB)
        i64, u64, dbl, ptr = ctypes.c_int64, ctypes.c_uint64, ctypes.c_double, ctypes.c_void_p
        L.oracle_init.argtypes = [i64, i64, i64, ctypes.c_int, ptr, u64, dbl, ptr]
        L.oracle_init.restype = None
        L.oracle_sweep.argtypes = [i64, i64, i64, ptr, ptr]
        L.oracle_sweep.restype = None
        L.oracle_sweep_owned.argtypes = [i64, i64, i64, ptr, ptr]
        L.oracle_sweep_owned.restype = None
        L.oracle_run.argtypes = [i64, i64, i64, ptr, ptr, i64]
        L.oracle_run.restype = ctypes.c_int
        L.oracle_checksum.argtypes = [i64, i64, i64, ptr]
        L.oracle_checksum.restype = u64
        L.oracle_residual.argtypes = [i64, i64, i64, ptr, ptr]
        L.oracle_residual.restype = dbl
        L.oracle_splitmix64_public.argtypes = [u64]
        L.oracle_splitmix64_public.restype = u64
        L.oracle_threads.argtypes = []
        L.oracle_threads.restype = ctypes.c_int
        L.oracle_set_threads.argtypes = [ctypes.c_int]
        L.oracle_set_threads.restype = None
        _lib = L
    return _lib


def _p(a: np.ndarray) -> int:
    assert a.dtype == np.float64 and a.flags["C_CONTIGUOUS"]
    return a.ctypes.data


def alloc(gx: int, gy: int, gz: int) -> np.ndarray:
    return np.empty((gz + 2, gy + 2, gx + 2), dtype=np.float64)


def owned(U: np.ndarray) -> np.ndarray:
    return U[1:-1, 1:-1, 1:-1]


def init(gx, gy, gz, kind=INIT_DEFAULT, params=(0.0, 0.0, 0.0, 0.0), seed=0, boundary=1.0) -> np.ndarray:
    U = alloc(gx, gy, gz)
    p = np.asarray(list(params) + [0.0] * (4 - len(params)), dtype=np.float64)
    lib().oracle_init(gx, gy, gz, kind, _p(p), seed, boundary, _p(U))
    return U


def sweep(U: np.ndarray) -> np.ndarray:
    gz, gy, gx = (s - 2 for s in U.shape)
    V = np.empty_like(U)
    lib().oracle_sweep(gx, gy, gz, _p(U), _p(V))
    return V


def run(U: np.ndarray, n: int) -> np.ndarray:
    """n Jacobi iterations; returns a new array (U is not modified)."""
    gz, gy, gx = (s - 2 for s in U.shape)
    A = U.copy()
    B = np.empty_like(U)
    which = lib().oracle_run(gx, gy, gz, _p(A), _p(B), n)
    return A if which == 0 else B


def run_pair(U: np.ndarray, n: int):
    """n >= 1 iterations; returns (u^n, u^(n-1)) for residual checks."""
    assert n >= 1
    prev = run(U, n - 1)
    return sweep(prev), prev


def checksum(U: np.ndarray) -> int:
    gz, gy, gx = (s - 2 for s in U.shape)
    return int(lib().oracle_checksum(gx, gy, gz, _p(np.ascontiguousarray(U))))


def residual(U: np.ndarray, Uprev: np.ndarray) -> float:
    gz, gy, gx = (s - 2 for s in U.shape)
    return float(lib().oracle_residual(gx, gy, gz, _p(U), _p(Uprev)))


def splitmix64(x: int) -> int:
    return int(lib().oracle_splitmix64_public(x & 0xFFFFFFFFFFFFFFFF))


def threads() -> int:
    return int(lib().oracle_threads())


def set_threads(n: int) -> None:
    lib().oracle_set_threads(int(n))


def sweep_owned_timing(U: np.ndarray, V: np.ndarray) -> None:
    """Owned-cell sweep U->V without the ghost copy (timing only; bit-identical
    to ``sweep`` when both buffers carry the same ghost shell)."""
    gz, gy, gx = (s - 2 for s in U.shape)
    lib().oracle_sweep_owned(gx, gy, gz, _p(U), _p(V))


if __name__ == "__main__":  # pragma: no cover
    print(build(force="--force" in sys.argv))
