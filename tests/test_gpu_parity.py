"""CUDA path vs the CPU oracle, element by element, bit for bit.

BASELINE.json north_star: "In fp64 with fixed summation order and no FMA
contraction in the stencil the match must be bit-exact".  Every variant
(unfused, paper strategies A/B/C, direct), launch mode (per-block streams,
batched), graph on/off and ODF must give the oracle's bits (SPEC.md L423,
DESIGN.md reading R14).  All calls go through the C ABI (ctypes binding).
"""
import itertools

import numpy as np
import pytest

from inputs.generators import sine_mode, sprinkle_nonfinite, uniform_field
from oracle import core
from tests.helpers import assert_bitwise, gpu_run, oracle_initial

pytestmark = pytest.mark.gpu

j3d = pytest.importorskip("paper_2202_11819_b200")

VARIANTS = ["unfused", "A", "B", "C", "direct"]
LAUNCHES = ["per_block", "batched"]


def _case(grid, odf, variant, launch, graph, n, kind="default", params=None, seed=0, boundary=1.0, field=None,
          block=(0, 0, 0)):
    with j3d.Jacobi3D(grid, odf=odf, variant=variant, launch=launch, graph=graph, boundary=boundary,
                      block=block) as ctx:
        got = gpu_run(ctx, n, kind, params, seed, field)
        ck = ctx.checksum()
        res = ctx.residual() if n >= 1 else None
    U0 = field if field is not None else oracle_initial(grid, kind, params or (0, 0, 0, 0), seed, boundary)
    if n >= 1:
        want, prev = core.run_pair(U0, n)
    else:
        want, prev = U0, None
    tag = f"{grid} odf={odf} {variant}/{launch}/graph={graph} {kind} n={n}"
    assert_bitwise(got, core.owned(want), tag)
    assert ck == core.checksum(want), tag
    if res is not None:
        assert np.float64(res).tobytes() == np.float64(core.residual(want, prev)).tobytes(), tag


@pytest.mark.parametrize("variant,launch,graph", list(itertools.product(VARIANTS, LAUNCHES, [False, True])))
def test_config1_matrix(variant, launch, graph):
    """BASELINE.json configs[0]: 64^3, 2x2x2 blocks (ODF=8), 1 GPU, 20 iterations,
    Dirichlet boundaries -- default and hash inputs."""
    _case((64, 64, 64), 8, variant, launch, graph, 20)
    _case((64, 64, 64), 8, variant, launch, graph, 20, kind="hash", seed=1)


@pytest.mark.parametrize("seed", [1, 2, 3])
@pytest.mark.parametrize("variant", ["unfused", "direct", "C"])
def test_hash_seeds(seed, variant):
    _case((48, 40, 24), 4, variant, "batched", False, 20, kind="hash", seed=seed)


@pytest.mark.parametrize("grid,odf,block", [
    ((200, 40, 30), 1, (0, 0, 0)),     # several tiles + ragged tail in x (128+72) and y (16+16+8)
    ((45, 34, 22), 2, (0, 0, 0)),      # odd nx: scalar tail of the vector path
    ((132, 72, 33), 4, (0, 0, 0)),
    ((16, 12, 4), 4, (16, 12, 1)),     # 1-cell-thick blocks
    ((9, 7, 5), 1, (0, 0, 0)),         # tiny, everything ragged
    ((1, 1, 1), 1, (0, 0, 0)),         # a single cell
    ((48, 48, 48), 27, (0, 0, 0)),     # 3x3x3 blocks: interior blocks with 6 neighbours
    ((64, 32, 96), 8, (0, 0, 0)),
])
@pytest.mark.parametrize("variant", VARIANTS)
@pytest.mark.parametrize("launch", LAUNCHES)
def test_shapes(grid, odf, block, variant, launch):
    _case(grid, odf, variant, launch, False, 7, kind="hash", seed=5, block=block)


@pytest.mark.parametrize("variant", ["unfused", "C", "direct"])
def test_linear_fixed_point(variant):
    """North star: a linear (discrete-harmonic) field with matching Dirichlet
    boundaries is a fixed point -- bitwise after 100 iterations."""
    grid = (40, 24, 32)
    p = (3.0, -5.0, 7.0, 1000.0)
    with j3d.Jacobi3D(grid, odf=8, variant=variant) as ctx:
        got = gpu_run(ctx, 100, "linear", p)
    assert_bitwise(got, core.owned(oracle_initial(grid, "linear", p)), "linear fixed point")


@pytest.mark.parametrize("c", [1.0, -2.5])
def test_constant_fixed_point(c):
    grid = (33, 20, 17)
    with j3d.Jacobi3D(grid, odf=1, variant="direct") as ctx:
        got = gpu_run(ctx, 50, "const", (c,))
    assert (got == c).all()


def test_sine_mode_via_set_block():
    """Host-generated input uploaded with jacobi3d_set_block (Dirichlet 0)."""
    U0 = sine_mode(40, 40, 40, (1, 2, 3))
    _case((40, 40, 40), 8, "direct", "batched", False, 30, boundary=0.0, field=U0)
    _case((40, 40, 40), 8, "unfused", "per_block", False, 30, boundary=0.0, field=U0)


def test_uniform_field_via_set_block():
    U0 = uniform_field(36, 28, 20, seed=7, boundary=0.5)
    for v in VARIANTS:
        _case((36, 28, 20), 4, v, "batched", True, 11, boundary=0.5, field=U0)


def test_zero_iterations_and_repeat_calls():
    """iterate(0) is a no-op; several iterate() calls == one call."""
    grid = (40, 40, 40)
    U0 = oracle_initial(grid, "hash", seed=3)
    for v, l in itertools.product(["unfused", "direct", "C"], LAUNCHES):
        with j3d.Jacobi3D(grid, odf=8, variant=v, launch=l) as ctx:
            ctx.init("hash", seed=3)
            ctx.iterate(0)
            assert_bitwise(ctx.gather_local(), core.owned(U0), "n=0")
            for n in (1, 2, 3, 4):
                ctx.iterate(n)
            assert_bitwise(ctx.gather_local(), core.owned(core.run(U0, 10)), f"split calls {v}/{l}")


def test_launch_count_law():
    """kernel launches per interior block per iteration are
    13 / 8 / 3 / 1 for no fusion / A / B / C (and 1 for direct); graph mode
    does one graph launch per iteration alternating the two parities
    (PAPER.md L529-530)."""
    want = {"unfused": 13, "A": 8, "B": 3, "C": 1, "direct": 1}
    for v, n in want.items():
        with j3d.Jacobi3D((48, 48, 48), odf=27, variant=v, launch="per_block") as ctx:
            ctx.init("default")
            ctx.reset_stats()
            ctx.iterate(6)
            ctx.synchronize()
            assert ctx.stats()["launches_per_iter_block"] == n, v
        with j3d.Jacobi3D((48, 48, 48), odf=27, variant=v, launch="per_block", graph=True) as ctx:
            ctx.init("default")
            ctx.reset_stats()
            parities = []
            for _ in range(5):
                ctx.iterate(1)
                parities.append(ctx.stats()["last_graph_parity"])
            st = ctx.stats()
            assert st["graph_launches"] == 5 and parities == [0, 1, 0, 1, 0]
            assert st["launches_per_iter_block"] == n, v


def test_errors():
    with pytest.raises(j3d.Jacobi3DError) as e:
        j3d.Jacobi3D((7, 8, 8), odf=3)
    assert e.value.code == -2
    with pytest.raises(j3d.Jacobi3DError) as e:
        j3d.Jacobi3D((8, 8, 8), odf=2, block=(8, 8, 3))
    assert e.value.code == -2
    with j3d.Jacobi3D((16, 16, 16), odf=2) as ctx:
        ctx.init("default")
        with pytest.raises(j3d.Jacobi3DError) as e:
            ctx.residual()
        assert e.value.code == -7
        with pytest.raises(j3d.Jacobi3DError) as e:
            ctx.get_block(5)
        assert e.value.code == -1


def test_get_region_matches_get_block():
    with j3d.Jacobi3D((70, 40, 30), odf=2, variant="direct") as ctx:
        ctx.init("hash", seed=9)
        ctx.iterate(3)
        full = ctx.get_block(1)
        reg = ctx.get_region(1, (5, 3, 2), (11, 7, 4))
        assert_bitwise(reg, full[2:6, 3:10, 5:16], "region")


def test_div7_matches_ieee_division():
    """The stencil's s/7 (Markstein-corrected reciprocal, kept unless the
    quotient is zero, subnormal or NaN; then the exact routine: integer path
    for subnormal quotients, s*y for +-inf) is the IEEE
    round-to-nearest division on 2^27 inputs per seed: random bit patterns
    (every double, +-inf and NaNs included), subnormals, exact/tie-prone
    dyadic values, +-0, +-DBL_MAX and the top binades (sums near overflow).
    NaN results compare by NaN-ness (R18)."""
    from paper_2202_11819_b200.jacobi3d import div7_selftest

    for seed in (1, 2):
        bad, ex = div7_selftest(1 << 27, seed)
        assert bad == 0, ex


@pytest.mark.parametrize("scale_exp", [-1060, -1030, -1074 + 60])
def test_subnormal_values(scale_exp):
    """Sums whose quotient is subnormal take the stencil's exact rare path
    (DESIGN.md "Division"); mixed signs and -0.0 included, Dirichlet 0."""
    U0 = uniform_field(40, 24, 16, seed=11, boundary=0.0) * 2.0 ** scale_exp
    U0[5:9, 5:9, 5:9] = -0.0
    for v in ("direct", "unfused", "C"):
        _case((40, 24, 16), 4, v, "batched", False, 9, boundary=0.0, field=U0)


@pytest.mark.parametrize("seed", [1, 2, 3])
def test_schedule_perturbation_does_not_change_bits(seed, monkeypatch):
    """SPEC.md L425 analogue: a perturbed launch order of the per-block
    streams (J3D_ORDER_SEED shuffles the block order) changes timings, never
    the bits."""
    monkeypatch.setenv("J3D_ORDER_SEED", str(seed))
    for v in ("unfused", "A", "C", "direct"):
        _case((48, 48, 48), 27, v, "per_block", False, 9, kind="hash", seed=seed)


def test_medium_grid_checksums_and_determinism():
    """T7: 256x192x160, ODF 8, 30 iterations: every variant / launch / graph
    combination reproduces the oracle's checksum; three repeated runs of the
    same context give identical checksums (S:571 analogue)."""
    grid = (256, 192, 160)
    U0 = oracle_initial(grid, "hash", seed=20220223)
    want = core.checksum(core.run(U0, 30))
    for v, l, g in itertools.product(VARIANTS, LAUNCHES, [False, True]):
        with j3d.Jacobi3D(grid, odf=8, variant=v, launch=l, graph=g) as ctx:
            sums = []
            for _ in range(3):
                ctx.init("hash", seed=20220223)
                ctx.iterate(30)
                sums.append(ctx.checksum())
            assert sums == [want] * 3, (v, l, g)


@pytest.mark.parametrize("kind", list(range(28)))
def test_every_tile_kind(kind, monkeypatch):
    """Every row of the kernel's tile table (J3D_TILE, kernels.cu J3D_TILES:
    both lane maps, 1-3 CTAs/SM, 4-8 stages) on ragged multi-block grids, direct
    and C variants (x ghost vectors, fused prologue/epilogue)."""
    monkeypatch.setenv("J3D_TILE", str(kind))
    _case((200, 45, 30), 2, "direct", "batched", False, 6, kind="hash", seed=kind + 1)
    _case((96, 40, 24), 8, "C", "batched", False, 5, kind="hash", seed=kind + 2)
    _case((45, 34, 22), 2, "unfused", "batched", False, 5, kind="hash", seed=kind + 3)


@pytest.mark.parametrize("grid,odf,launch", [((64, 64, 64), 8, "batched"), ((45, 34, 22), 2, "batched"),
                                             ((96, 96, 96), 8, "persistent"), ((200, 40, 30), 1, "persistent")])
def test_plan_bytes_match_allocation(grid, odf, launch):
    """jacobi3d_plan's bytes_per_gpu (no GPU) equals the arena the context
    allocates (x ghost arrays, persistent counters and face buffers included)."""
    import struct

    want = j3d.plan(grid, odf=odf, launch=launch)["bytes_per_gpu"]
    with j3d.Jacobi3D(grid, odf=odf, variant="direct", launch=launch) as ctx:
        rec = ctx.ipc_export()
    assert struct.unpack_from("<Q", rec, 16)[0] == want


def _same_or_both_nan(got, want):
    got = np.asarray(got, dtype=np.float64)
    want = np.ascontiguousarray(want, dtype=np.float64)
    ng, nw = np.isnan(got), np.isnan(want)
    if not (ng == nw).all():
        bad = np.argwhere(ng != nw)
        raise AssertionError(f"NaN-ness differs in {len(bad)} cells, first {bad[0].tolist()}")
    assert_bitwise(np.where(ng, 0.0, got), np.where(nw, 0.0, want), "non-NaN cells")


def _case_nonfinite(grid, odf, variant, launch, n, kind="default", params=None, boundary=1.0, field=None):
    """NaN policy (R18): NaN-ness equal and every other cell bit for
    bit; the checksum (bits of every cell) only where no cell is NaN; the
    residual NaN-ness or bits."""
    with j3d.Jacobi3D(grid, odf=odf, variant=variant, launch=launch, boundary=boundary) as ctx:
        got = gpu_run(ctx, n, kind, params, 0, field)
        ck = ctx.checksum()
        res = ctx.residual()
    U0 = field if field is not None else oracle_initial(grid, kind, params or (0, 0, 0, 0), 0, boundary)
    want, prev = core.run_pair(U0, n)
    W = core.owned(want)
    _same_or_both_nan(got, W)
    if not np.isnan(W).any():
        assert ck == core.checksum(want)
    r = core.residual(want, prev)
    assert (np.isnan(res) and np.isnan(r)) or np.float64(res).tobytes() == np.float64(r).tobytes(), (res, r)


@pytest.mark.parametrize("variant,launch", [("direct", "batched"), ("direct", "persistent"), ("C", "batched"),
                                            ("unfused", "per_block")])
def test_nonfinite_values(variant, launch):
    """IEEE semantics of S:388's sum and /7 for non-finite values (the oracle's
    pins: test_oracle_pins non-finite section): a +-inf Dirichlet boundary,
    a constant field whose sum overflows (1e308, -DBL_MAX), and a field with
    +-inf / NaN cells (inf - inf = NaN spreads) -- the stencil's rare path
    must give +-inf where the fast division would give NaN."""
    grid = (70, 34, 20)
    _case_nonfinite(grid, 4, variant, launch, 6, boundary=float("inf"))
    _case_nonfinite(grid, 4, variant, launch, 6, boundary=float("-inf"))
    _case_nonfinite(grid, 4, variant, launch, 3, kind="const", params=(1e308,))
    _case_nonfinite(grid, 4, variant, launch, 3, kind="const", params=(-float.fromhex("0x1.fffffffffffffp+1023"),))
    U0 = sprinkle_nonfinite(uniform_field(*grid, seed=13, boundary=0.5), seed=5)
    _case_nonfinite(grid, 4, variant, launch, 5, boundary=0.5, field=U0)
