"""Pins of the CPU oracle against what the paper and the mathematics fix.

None of these compares the oracle with a retyping of its own formula: the
pins are hand-derived values (tests/golden, derivations written out there),
an independent symmetry-reduced recurrence in exact rationals, exact-rational
brute force with an error bound, fixed points that follow from exactness of
the arithmetic, a textbook eigenmode closed form, the discrete maximum
principle, an explicitly block-decomposed run with halo exchange (the
paper's method) and published splitmix64 reference vectors.
Each test cites the passage that fixes the expected behaviour.
"""
import math
import os
from fractions import Fraction

import numpy as np
import pytest

from oracle import brute, core, twin

EPS = 2.0 ** -52


def _load_golden(path):
    rows = []
    with open(path) as f:
        for line in f:
            line = line.split("#", 1)[0].strip()
            if line:
                rows.append(line.split())
    return rows


def _class_of(i, j, k, g=4):
    return sum(1 for c in (i, j, k) if c in (0, g - 1))


# ---------------------------------------------------------------- hand values

def test_hand_4cube_one_iteration_bitwise(golden_dir):
    """1 iteration, all-zero interior, unit boundary -> corner 3/7,
    face-adjacent 1/7.  After one iteration every sum is an exact integer, so the
    fp64 result must be RN(k/7) bit for bit (hex values worked by hand)."""
    want = {int(m): float.fromhex(h) for m, h in _load_golden(os.path.join(golden_dir, "hand_4cube_bits.txt"))}
    U = core.run(core.init(4, 4, 4), 1)
    O = core.owned(U)
    for k in range(4):
        for j in range(4):
            for i in range(4):
                got = O[k, j, i]
                assert got.tobytes() == np.float64(want[_class_of(i, j, k)]).tobytes(), (i, j, k, got)


@pytest.mark.parametrize("n", [1, 2, 3])
def test_hand_4cube_multi_iteration(golden_dir, n):
    """Hand-derived exact values (tests/golden/hand_4cube.txt) for n = 1..3:
    the fp64 oracle is within n*4*eps of the exact rational, and the exact
    brute force reproduces the hand value exactly."""
    rows = [r for r in _load_golden(os.path.join(golden_dir, "hand_4cube.txt")) if int(r[0]) == n]
    exact_by_class = {int(m): Fraction(int(a), int(b)) for _, m, a, b in rows}
    U = core.run(core.init(4, 4, 4), n)
    O = core.owned(U)
    E = brute.run_exact(brute.make_grid(4, 4, 4, 0.0, 1.0), 4, 4, 4, n)
    for k in range(4):
        for j in range(4):
            for i in range(4):
                want = exact_by_class[_class_of(i, j, k)]
                assert E[k + 1][j + 1][i + 1] == want
                assert abs(Fraction(float(O[k, j, i])) - want) <= n * 4 * EPS


def _class_recurrence(n):
    """Independent derivation: symmetry-reduced 4-state recurrence (see
    tests/golden/hand_4cube.txt header), exact rationals."""
    v = [Fraction(0)] * 4
    for _ in range(n):
        nv = []
        for m in range(4):
            s = v[m]
            s += m * (1 + (v[m - 1] if m > 0 else 0))
            s += (3 - m) * ((v[m + 1] if m < 3 else 0) + v[m])
            nv.append(s / 7)
        v = nv
    return v


@pytest.mark.parametrize("n", [4, 5, 8])
def test_4cube_matches_symmetry_recurrence(n):
    """Exact brute force == symmetry recurrence; fp64 oracle within n*4*eps;
    fp64 oracle bitwise == scalar-Python IEEE brute force."""
    v = _class_recurrence(n)
    G = brute.make_grid(4, 4, 4, 0.0, 1.0)
    E = brute.run_exact(G, 4, 4, 4, n)
    F = brute.run_float(G, 4, 4, 4, n)
    O = core.owned(core.run(core.init(4, 4, 4), n))
    for k in range(4):
        for j in range(4):
            for i in range(4):
                m = _class_of(i, j, k)
                assert E[k + 1][j + 1][i + 1] == v[m]
                assert abs(Fraction(float(O[k, j, i])) - v[m]) <= n * 4 * EPS
                assert np.float64(F[k + 1][j + 1][i + 1]).tobytes() == O[k, j, i].tobytes()


def test_3cube_spec_example():
    """1 iteration, 3x3x3 all-zero interior with unit boundary ->
    centre element 0, all others have >= 1 boundary neighbour (> 0)."""
    O = core.owned(core.run(core.init(3, 3, 3), 1))
    assert O[1, 1, 1] == 0.0
    mask = np.ones_like(O, dtype=bool)
    mask[1, 1, 1] = False
    assert (O[mask] > 0).all()


def test_zero_iterations_is_identity():
    """0 iterations -> initial grid."""
    U = core.init(5, 6, 7, core.INIT_HASH, seed=3)
    assert np.array_equal(core.run(U, 0), U)


# ---------------------------------------------------------------- fixed points

@pytest.mark.parametrize("c", [1.0, 0.75, -2.5, 3 * 2.0 ** -30])
def test_constant_fixed_point_bitwise(c):
    """SPEC.md L392/L457 and BASELINE.json north_star: a constant field with
    matching boundary is a fixed point.  For these c, 2c..7c are exact, so the
    sum is exactly 7c and the division returns c exactly, bit for bit."""
    U = core.init(9, 7, 6, core.INIT_CONST, (c,))
    R = core.run(U, 100)
    assert R.tobytes() == U.tobytes()


@pytest.mark.parametrize("coef", [(3.0, -5.0, 7.0, 1000.0), (0.5, 0.25, -0.125, 1.0), (1.0, 1.0, 1.0, 0.0)])
def test_linear_fixed_point_bitwise(coef):
    """BASELINE.json north_star: a discrete-harmonic (linear) field with
    matching Dirichlet boundaries is a fixed point.  u(i-1)+u(i+1) = 2u(i) for
    linear u, so the exact sum is 7u; with integer/dyadic coefficients every
    partial sum is exact, hence bitwise fixed."""
    U = core.init(11, 8, 9, core.INIT_LINEAR, coef)
    R = core.run(U, 100)
    assert R.tobytes() == U.tobytes()


def test_linear_init_values():
    """The LINEAR init evaluates a*i+b*j+c*k+d at ghost coordinates -1 and g
    (R7)."""
    U = core.init(4, 3, 2, core.INIT_LINEAR, (3.0, -5.0, 7.0, 1000.0))
    for k in range(-1, 3):
        for j in range(-1, 4):
            for i in range(-1, 5):
                assert U[k + 1, j + 1, i + 1] == 3 * i - 5 * j + 7 * k + 1000


# ---------------------------------------------------------------- closed form

@pytest.mark.parametrize("N,pqr", [(16, (1, 2, 3)), (24, (2, 1, 1))])
def test_sine_eigenmode_closed_form(N, pqr):
    """Textbook eigenmode of the 7-point average with Dirichlet-0 boundary:
    u0 = prod sin(p pi (i+1)/(N+1)) -> u^n = lambda^n u0,
    lambda = (1 + 2cos(p pi/(N+1)) + 2cos(q pi/(N+1)) + 2cos(r pi/(N+1)))/7.
    Tolerance 8*n*eps*max|u0| (rounding of 7 ops per step)."""
    from inputs.generators import sine_mode

    n = 100
    U0 = sine_mode(N, N, N, pqr)
    p, q, r = pqr
    lam = (1 + 2 * math.cos(p * math.pi / (N + 1)) + 2 * math.cos(q * math.pi / (N + 1))
           + 2 * math.cos(r * math.pi / (N + 1))) / 7
    R = core.run(U0, n)
    err = np.abs(core.owned(R) - lam ** n * core.owned(U0)).max()
    assert err <= 8 * n * EPS * np.abs(U0).max()


# ---------------------------------------------------------------- invariants

def test_max_principle_and_monotone():
    """Default init (0 interior, 1 boundary): the average of values in [0,1]
    stays in [0,1] and, since u^1 >= u^0 and the update is monotone,
    u^(n+1) >= u^n (discrete maximum principle)."""
    U = core.init(12, 10, 9)
    prev = U
    for _ in range(30):
        nxt = core.sweep(prev)
        o, p = core.owned(nxt), core.owned(prev)
        assert (o >= 0).all() and (o <= 1).all()
        assert (o >= p).all()
        prev = nxt


def test_numpy_twin_and_scalar_bruteforce_bitwise():
    """Three independently written fp64 versions agree bit for bit on 4^3 x 5
    and on a hash-random 7x5x6 grid."""
    for gx, gy, gz, kind in ((4, 4, 4, core.INIT_DEFAULT), (7, 5, 6, core.INIT_HASH)):
        U = core.init(gx, gy, gz, kind, seed=11)
        C = core.run(U, 5)
        T = twin.run(U, 5)
        assert C.tobytes() == T.tobytes()
        F = brute.run_float(U.tolist(), gx, gy, gz, 5)
        assert np.array(F).tobytes() == C.tobytes()


def test_hash_init_twin():
    """C and numpy implementations of the hash input generator agree."""
    for seed in (0, 1, 2, 3, 20220223):
        assert core.init(9, 8, 7, core.INIT_HASH, seed=seed).tobytes() == twin.init_hash(9, 8, 7, seed).tobytes()
    U = core.init(16, 16, 16, core.INIT_HASH, seed=1)
    o = core.owned(U)
    assert (o >= 0).all() and (o < 1).all() and len(np.unique(o)) == o.size


def _blocked_run(U, n, blocks):
    """The paper's method written out on the CPU: split the owned grid into
    bx*by*bz blocks each with its own ghost shell and two buffers; each
    iteration every block packs its faces, the faces are delivered to the
    neighbours' ghost layers (Dirichlet faces keep the boundary), then every
    block applies the stencil (Fig 1 L79-107: pack, exchange, unpack,
    update).  Uses the numpy twin's sweep per block."""
    gz, gy, gx = (s - 2 for s in U.shape)
    nbx, nby, nbz = blocks
    ex, ey, ez = gx // nbx, gy // nby, gz // nbz
    B = {}
    for bk in range(nbz):
        for bj in range(nby):
            for bi in range(nbx):
                B[bi, bj, bk] = U[bk * ez:bk * ez + ez + 2, bj * ey:bj * ey + ey + 2, bi * ex:bi * ex + ex + 2].copy()
    for _ in range(n):
        for key in B:
            B[key] = twin.sweep(B[key])
        # halo exchange of the new owned boundary layers into neighbours' ghosts
        for (bi, bj, bk), b in B.items():
            if bi + 1 < nbx:
                nb = B[bi + 1, bj, bk]
                nb[1:-1, 1:-1, 0] = b[1:-1, 1:-1, -2]
                b[1:-1, 1:-1, -1] = nb[1:-1, 1:-1, 1]
            if bj + 1 < nby:
                nb = B[bi, bj + 1, bk]
                nb[1:-1, 0, 1:-1] = b[1:-1, -2, 1:-1]
                b[1:-1, -1, 1:-1] = nb[1:-1, 1, 1:-1]
            if bk + 1 < nbz:
                nb = B[bi, bj, bk + 1]
                nb[0, 1:-1, 1:-1] = b[-2, 1:-1, 1:-1]
                b[-1, 1:-1, 1:-1] = nb[1, 1:-1, 1:-1]
    R = U.copy()
    for (bi, bj, bk), b in B.items():
        R[bk * ez + 1:bk * ez + ez + 1, bj * ey + 1:bj * ey + ey + 1, bi * ex + 1:bi * ex + ex + 1] = b[1:-1, 1:-1, 1:-1]
    return R


@pytest.mark.parametrize("blocks", [(2, 2, 2), (1, 2, 3), (4, 1, 1), (3, 2, 1)])
def test_decomposition_invariance_bitwise(blocks):
    """BASELINE.json north_star: a single-block run equals a many-block
    overdecomposed run bit for bit (halos of the same iteration only,
    PAPER.md L180-183 / L283-284)."""
    U = core.init(12, 12, 12, core.INIT_HASH, seed=2)
    assert _blocked_run(U, 7, blocks).tobytes() == core.run(U, 7).tobytes()


def test_interior_update_independent_of_halos():
    """PAPER.md L120-124 / Fig 1 (L89-91): "updating only the interior of the
    block does not depend on the neighbors' halo data".  With the ghost shell
    poisoned by NaN, every owned cell not adjacent to the shell is bitwise
    the full update; every cell adjacent to it is not (it reads a ghost)."""
    U = core.init(10, 9, 8, core.INIT_HASH, seed=5)
    full = core.owned(core.sweep(U))
    G = U.copy()
    G[0, :, :] = G[-1, :, :] = np.nan
    G[:, 0, :] = G[:, -1, :] = np.nan
    G[:, :, 0] = G[:, :, -1] = np.nan
    part = core.owned(core.sweep(G))
    assert part[1:-1, 1:-1, 1:-1].tobytes() == full[1:-1, 1:-1, 1:-1].tobytes()
    ext = np.ones(part.shape, dtype=bool)
    ext[1:-1, 1:-1, 1:-1] = False
    assert np.isnan(part[ext]).all()


# ---------------------------------------------------------------- checksum / residual

def test_splitmix64_reference_vectors():
    """S. Vigna's splitmix64.c reference output from state 0 (the generator
    used by the hash init and the checksum): 0xe220a8397b1dcdaf,
    0x6e789e6aa1b965f4, 0x06c45d188009454f, 0xf88bb8a8724c81ec."""
    g = 0x9E3779B97F4A7C15
    want = [0xE220A8397B1DCDAF, 0x6E789E6AA1B965F4, 0x06C45D188009454F, 0xF88BB8A8724C81EC]
    got = [core.splitmix64((i * g) & 0xFFFFFFFFFFFFFFFF) for i in range(4)]
    assert got == want
    tw = twin.splitmix64(np.array([(i * g) & 0xFFFFFFFFFFFFFFFF for i in range(4)], dtype=np.uint64))
    assert [int(x) for x in tw] == want


def test_checksum_properties():
    """Checksum (R15): order independent sum mod 2^64; equal for the
    C and numpy versions; additive over any partition of the owned cells;
    sensitive to one-ulp changes and to swapping two cells."""
    U = core.init(8, 7, 6, core.INIT_HASH, seed=9)
    c = core.checksum(U)
    assert c == twin.checksum(U)
    V = U.copy()
    V[3, 3, 3] = np.nextafter(V[3, 3, 3], 2.0)
    assert core.checksum(V) != c
    W = U.copy()
    W[1, 1, 1], W[2, 2, 2] = U[2, 2, 2], U[1, 1, 1]
    assert core.checksum(W) != c
    # additivity: zero-out halves contribute the same total (mod 2^64)
    A = U.copy(); A[1:4, 1:-1, 1:-1] = 0.0
    B = U.copy(); B[4:-1, 1:-1, 1:-1] = 0.0
    Z = U.copy(); Z[1:-1, 1:-1, 1:-1] = 0.0
    assert (core.checksum(A) + core.checksum(B) - core.checksum(Z)) % 2 ** 64 == c


def test_residual_pins():
    """Residual = max |u^n - u^(n-1)| over owned cells (R11).
    Constant field: 0.  4^3 default after 1 iteration: the corner moved from 0
    to RN(3/7), the largest change.  After 2: hand values 30/49-3/7 = 9/49
    (corner and edge) within 2 ulps."""
    U = core.init(6, 6, 6, core.INIT_CONST, (0.75,))
    a, b = core.run_pair(U, 3)
    assert core.residual(a, b) == 0.0
    a, b = core.run_pair(core.init(4, 4, 4), 1)
    assert core.residual(a, b) == float.fromhex("0x1.b6db6db6db6dbp-2")
    a, b = core.run_pair(core.init(4, 4, 4), 2)
    assert abs(core.residual(a, b) - 9 / 49) <= 4 * EPS
    assert core.residual(a, b) == twin.residual(a, b)


# ---------------------------------------------------------------- non-finite values (IEEE 754 semantics)

def _same_or_both_nan(a: np.ndarray, b: np.ndarray) -> bool:
    """NaN policy (R18): NaN-ness must agree, payloads are not part of
    the result; every other value bit for bit."""
    a = np.asarray(a, dtype=np.float64)
    b = np.asarray(b, dtype=np.float64)
    na, nb = np.isnan(a), np.isnan(b)
    return bool((na == nb).all() and (a[~na].view(np.uint64) == b[~nb].view(np.uint64)).all())


@pytest.mark.parametrize("inf", [math.inf, -math.inf])
def test_infinite_boundary_one_iteration(inf):
    """IEEE 754 (S:388's sum and /7 carried out in binary64): x + inf = inf for
    finite x and inf / 7 = inf.  4^3 grid, interior 0, Dirichlet boundary
    +-inf: after one iteration each of the 56 cells next to the boundary is
    +-inf and the inner 2x2x2 stays 0; the ghost shell is unchanged."""
    U = core.run(core.init(4, 4, 4, boundary=inf), 1)
    O = core.owned(U)
    for k in range(4):
        for j in range(4):
            for i in range(4):
                want = inf if _class_of(i, j, k) > 0 else 0.0
                assert O[k, j, i] == want, (i, j, k, O[k, j, i])
    assert (U[0] == inf).all() and (U[:, 0] == inf).all()
    # two more iterations: the scalar IEEE brute force agrees bit for bit
    B = brute.run_float(brute.make_grid(4, 4, 4, 0.0, inf), 4, 4, 4, 3)
    assert _same_or_both_nan(core.run(core.init(4, 4, 4, boundary=inf), 3), np.array(B))


@pytest.mark.parametrize("c", [1e308, -1e308, float.fromhex("0x1.fffffffffffffp+1023")])
def test_overflowing_sum_is_infinite(c):
    """IEEE 754 round-to-nearest overflow: a constant field c with |7c| > DBL_MAX
    (2c already overflows) sums to +-inf in S:388's order, and +-inf / 7 = +-inf:
    every owned cell is +-inf after one iteration (the CONST init fills the
    ghost shell with c as well)."""
    U = core.run(core.init(5, 4, 3, core.INIT_CONST, (c,)), 1)
    assert (core.owned(U) == math.copysign(math.inf, c)).all()
    assert (U[0] == c).all()


def test_mixed_infinities_give_nan_like_brute_force():
    """+inf boundary and one -inf interior cell: cells that see both get
    inf + (-inf) = NaN (IEEE 754 invalid operation), which then spreads.  The C
    oracle and the scalar brute force agree cell by cell (NaN-ness; R18)."""
    G = brute.make_grid(4, 4, 4, 0.0, math.inf)
    G[2][2][2] = -math.inf
    U = core.init(4, 4, 4, boundary=math.inf)
    U[2, 2, 2] = -math.inf
    for n in (1, 2, 3):
        want = np.array(brute.run_float([[row[:] for row in p] for p in G], 4, 4, 4, n))
        got = core.run(U, n)
        assert np.isnan(got).any() and _same_or_both_nan(got, want), n
        assert _same_or_both_nan(got, twin.run(U, n)), n


def test_residual_nan_policy():
    """Residual (R11) of a field whose change is NaN somewhere (inf - inf after
    the overflowed constant field, or a NaN cell) is NaN -- the numpy twin's
    np.max propagates NaN the same way -- and +inf for a finite -> inf change."""
    a, b = core.run_pair(core.init(3, 3, 3, core.INIT_CONST, (1e308,)), 2)  # inf - inf
    assert math.isnan(core.residual(a, b)) and math.isnan(twin.residual(a, b))
    a, b = core.run_pair(core.init(3, 3, 3, core.INIT_CONST, (1e308,)), 1)  # inf - 1e308
    assert core.residual(a, b) == math.inf == twin.residual(a, b)
    U = core.init(6, 5, 4, core.INIT_HASH, seed=3)
    V = U.copy()
    V[2, 3, 4] = math.nan
    assert math.isnan(core.residual(U, V)) and math.isnan(core.residual(V, U))
    assert math.isnan(twin.residual(U, V))


# ---------------------------------------------------------------- the timing sweep

@pytest.mark.parametrize("grid,kind,seed", [((9, 7, 5), core.INIT_HASH, 1), ((16, 12, 10), core.INIT_HASH, 2),
                                            ((8, 8, 8), core.INIT_DEFAULT, 0)])
def test_sweep_owned_equals_sweep(grid, kind, seed):
    """oracle_sweep_owned (the cpu_baseline / reference-arm sweep) skips the
    ghost-shell copy; with both buffers carrying the same Dirichlet shell it
    must give oracle_sweep's owned cells bit for bit, iteration after
    iteration, and leave the shell untouched."""
    U = core.init(*grid, kind, seed=seed)
    A, B = U.copy(), U.copy()
    ref = U
    for _ in range(4):
        core.sweep_owned_timing(A, B)
        A, B = B, A
        ref = core.sweep(ref)
        assert A.tobytes() == ref.tobytes()
