"""The dependency-cone helper used by the full-size GPU parity test is exact
(checked against a full oracle run on a small grid)."""
from oracle import core
from tests.helpers import cone_value


def test_cone_value_matches_full_run():
    grid = (19, 17, 13)
    n = 3
    full = core.run(core.init(*grid, core.INIT_HASH, seed=20220223), n)
    for c in [(0, 0, 0), (18, 16, 12), (9, 8, 6), (1, 15, 3), (5, 0, 12), (4, 5, 6)]:
        i, j, k = c
        assert cone_value(grid, 20220223, n, c) == full[k + 1, j + 1, i + 1]
