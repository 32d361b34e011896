"""Seeded input generators (no Jacobi arithmetic here).

Arrays are ghosted grids of shape (gz+2, gy+2, gx+2), x fastest, fp64,
matching the oracle's layout; ``owned(a)`` slices the owned cells for
``jacobi3d_set_block``-style uploads.
"""
from __future__ import annotations

import math

import numpy as np


def owned(a: np.ndarray) -> np.ndarray:
    return a[1:-1, 1:-1, 1:-1]


def sine_mode(gx: int, gy: int, gz: int, pqr=(1, 2, 3)) -> np.ndarray:
    """u0(i,j,k) = sin(p pi (i+1)/(gx+1)) sin(q pi (j+1)/(gy+1)) sin(r pi (k+1)/(gz+1))
    on owned cells, Dirichlet 0 ghost shell (the sine vanishes there)."""
    p, q, r = pqr
    a = np.zeros((gz + 2, gy + 2, gx + 2), dtype=np.float64)
    sx = np.sin(p * math.pi * np.arange(1, gx + 1) / (gx + 1))
    sy = np.sin(q * math.pi * np.arange(1, gy + 1) / (gy + 1))
    sz = np.sin(r * math.pi * np.arange(1, gz + 1) / (gz + 1))
    a[1:-1, 1:-1, 1:-1] = sz[:, None, None] * sy[None, :, None] * sx[None, None, :]
    return a


def uniform_field(gx: int, gy: int, gz: int, seed: int, boundary: float = 1.0,
                  lo: float = -1.0, hi: float = 1.0) -> np.ndarray:
    """Owned cells ~ U[lo, hi) from numpy's PCG64 with the given seed; ghost
    shell = boundary."""
    a = np.full((gz + 2, gy + 2, gx + 2), boundary, dtype=np.float64)
    rng = np.random.default_rng(seed)
    a[1:-1, 1:-1, 1:-1] = rng.uniform(lo, hi, size=(gz, gy, gx))
    return a


def sprinkle_nonfinite(a: np.ndarray, seed: int, count: int = 12) -> np.ndarray:
    """Copy of a ghosted field with ``count`` random owned cells set to +inf,
    -inf or NaN in turn (non-finite parity cases; R18)."""
    b = a.copy()
    gz, gy, gx = (s - 2 for s in a.shape)
    rng = np.random.default_rng(seed)
    vals = (math.inf, -math.inf, math.nan)
    for t in range(count):
        k, j, i = (int(rng.integers(0, n)) for n in (gz, gy, gx))
        b[k + 1, j + 1, i + 1] = vals[t % 3]
    return b
