"""numpy twin of the C oracle (same definition, array slicing).

TEST INFRASTRUCTURE ONLY (see ``oracle/__init__.py``).

Follows SURVEY.md §8(c): V = ((((((c + xm) + xp) + ym) + yp) + zm) + zp) / 7.0
on owned cells (SPEC.md L388 order), ghost shell copied (Dirichlet, SPEC.md
L430), two buffers.  Each numpy elementwise add/divide is
one IEEE round-to-nearest operation, so this is bitwise the C oracle.
Arrays are (gz+2, gy+2, gx+2), x fastest.
"""
from __future__ import annotations

import numpy as np

_MASK = np.uint64(0xFFFFFFFFFFFFFFFF)


def sweep(U: np.ndarray) -> np.ndarray:
    V = U.copy()
    c = U[1:-1, 1:-1, 1:-1]
    s = c + U[1:-1, 1:-1, :-2]      # -x
    s = s + U[1:-1, 1:-1, 2:]       # +x
    s = s + U[1:-1, :-2, 1:-1]      # -y
    s = s + U[1:-1, 2:, 1:-1]       # +y
    s = s + U[:-2, 1:-1, 1:-1]      # -z
    s = s + U[2:, 1:-1, 1:-1]       # +z
    V[1:-1, 1:-1, 1:-1] = s / 7.0
    return V


def run(U: np.ndarray, n: int) -> np.ndarray:
    for _ in range(n):
        U = sweep(U)
    return U


def splitmix64(x: np.ndarray) -> np.ndarray:
    """Vectorised splitmix64 (uint64 wrap-around)."""
    with np.errstate(over="ignore"):
        z = (x.astype(np.uint64) + np.uint64(0x9E3779B97F4A7C15)) & _MASK
        z = ((z ^ (z >> np.uint64(30))) * np.uint64(0xBF58476D1CE4E5B9)) & _MASK
        z = ((z ^ (z >> np.uint64(27))) * np.uint64(0x94D049BB133111EB)) & _MASK
        return z ^ (z >> np.uint64(31))


def gidx(gx: int, gy: int, gz: int) -> np.ndarray:
    k, j, i = np.meshgrid(np.arange(gz, dtype=np.uint64), np.arange(gy, dtype=np.uint64),
                          np.arange(gx, dtype=np.uint64), indexing="ij")
    return i + np.uint64(gx) * (j + np.uint64(gy) * k)


def init_hash(gx: int, gy: int, gz: int, seed: int, boundary: float = 1.0) -> np.ndarray:
    U = np.full((gz + 2, gy + 2, gx + 2), boundary, dtype=np.float64)
    s = splitmix64(np.array([seed], dtype=np.uint64))[0]
    bits = splitmix64(s ^ gidx(gx, gy, gz)) >> np.uint64(11)
    U[1:-1, 1:-1, 1:-1] = bits.astype(np.float64) * 2.0 ** -53
    return U


def checksum(U: np.ndarray) -> int:
    gz, gy, gx = (s - 2 for s in U.shape)
    bits = np.ascontiguousarray(U[1:-1, 1:-1, 1:-1]).view(np.uint64)
    h = splitmix64(bits ^ splitmix64(gidx(gx, gy, gz)))
    return int(np.sum(h, dtype=np.uint64))  # numpy uint64 sum wraps mod 2^64


def residual(U: np.ndarray, Uprev: np.ndarray) -> float:
    d = np.abs(U[1:-1, 1:-1, 1:-1] - Uprev[1:-1, 1:-1, 1:-1])
    return float(d.max()) if d.size else 0.0
