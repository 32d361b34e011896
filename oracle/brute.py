"""Scalar brute force of the Jacobi3D definition, for tiny grids (<= 8^3).

TEST INFRASTRUCTURE ONLY (see ``oracle/__init__.py``).

``run_float``  : pure-Python loops with Python floats (IEEE binary64,
                 round-to-nearest): one add per term in the order
                 self,-x,+x,-y,+y,-z,+z then ``/ 7.0``.
``run_exact``  : the same recurrence in exact rational arithmetic
                 (``fractions.Fraction``): the value the fp64 method
                 approximates, used with an n*4*eps error bound.
Grids are nested lists indexed [k][j][i] over the ghosted extent
(g+2 per axis), boundary = Dirichlet ghost value.
"""
from __future__ import annotations

from fractions import Fraction


def make_grid(gx, gy, gz, interior, boundary):
    return [[[boundary if (i in (0, gx + 1) or j in (0, gy + 1) or k in (0, gz + 1)) else interior
              for i in range(gx + 2)] for j in range(gy + 2)] for k in range(gz + 2)]


def _step(U, gx, gy, gz, div):
    V = [[row[:] for row in plane] for plane in U]
    for k in range(1, gz + 1):
        for j in range(1, gy + 1):
            for i in range(1, gx + 1):
                s = U[k][j][i]
                s = s + U[k][j][i - 1]
                s = s + U[k][j][i + 1]
                s = s + U[k][j - 1][i]
                s = s + U[k][j + 1][i]
                s = s + U[k - 1][j][i]
                s = s + U[k + 1][j][i]
                V[k][j][i] = div(s)
    return V


def run_float(U, gx, gy, gz, n):
    for _ in range(n):
        U = _step(U, gx, gy, gz, lambda s: s / 7.0)
    return U


def run_exact(U, gx, gy, gz, n):
    U = [[[Fraction(v) for v in row] for row in plane] for plane in U]
    for _ in range(n):
        U = _step(U, gx, gy, gz, lambda s: s / 7)
    return U
