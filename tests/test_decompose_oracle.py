"""Pins of the decomposition oracle (oracle/decompose.py) against the paper's
and SPEC's worked examples (tests/golden/planner.txt) and its arithmetic."""
import os

import pytest

from oracle.decompose import DecompositionError, decompose, footprint_bytes, plan


def _rows(golden_dir):
    out = []
    with open(os.path.join(golden_dir, "planner.txt")) as f:
        for line in f:
            line = line.split("#", 1)[0].strip()
            if line:
                t = line.split()
                out.append(tuple(int(x) for x in t[:7]))
    return out


def test_golden_decompositions(golden_dir):
    for gx, gy, gz, n, px, py, pz in _rows(golden_dir):
        assert decompose((gx, gy, gz), n) == (px, py, pz)


def test_spec_max_face_9mib():
    """1536^3 over 6 -> block 1536x768x512, max face 1536x768
    elements = 9437184 B = 9 MiB (PAPER.md L621 'up to 9 MB')."""
    px, py, pz = decompose((1536, 1536, 1536), 6)
    b = (1536 // px, 1536 // py, 1536 // pz)
    assert b == (1536, 768, 512)
    assert max(b[0] * b[1], b[1] * b[2], b[0] * b[2]) * 8 == 9437184


def test_spec_footprints():
    """SPEC.md L473-474 (PAPER.md L620 'roughly 9 GB' / '18 MB')."""
    assert footprint_bytes((1536,) * 3, decompose((1536,) * 3, 6)) == 9663676416
    assert footprint_bytes((192,) * 3, decompose((192,) * 3, 6)) == 18874368


def test_errors():
    """no divisible factorisation -> error naming the dimension;
    SPEC.md L127: zero extent -> configuration error."""
    with pytest.raises(DecompositionError, match="x"):
        decompose((7, 1, 1), 2)
    with pytest.raises(DecompositionError):
        decompose((0, 4, 4), 1)


def test_tie_break_lexicographic():
    """ties -> lexicographically smallest triple.  A cube over 2
    parts has three equal-surface splits; (1,1,2) is the smallest."""
    assert decompose((64, 64, 64), 2) == (1, 1, 2)
    assert decompose((64, 64, 64), 4) == (1, 2, 2)


def test_survey_config_plans():
    """weak 1536^3/GPU and ODF block grids."""
    assert plan((1536, 1536, 1536), 1, 1) == ((1, 1, 1), (1, 1, 1), (1536, 1536, 1536))
    assert plan((1536, 1536, 3072), 2, 1)[0] == (1, 1, 2)
    assert plan((1536, 3072, 3072), 4, 1)[0] == (1, 2, 2)
    assert plan((3072, 3072, 3072), 8, 8) == ((2, 2, 2), (2, 2, 2), (768, 768, 768))
    assert plan((1536,) * 3, 1, 4)[1:] == ((1, 2, 2), (1536, 768, 768))
    assert plan((1536,) * 3, 1, 16)[1:] == ((2, 2, 4), (768, 768, 384))
    assert plan((1536,) * 3, 1, 32)[1:] == ((2, 4, 4), (768, 384, 384))
    assert plan((768,) * 3, 8, 64) == ((2, 2, 2), (4, 4, 4), (96, 96, 96))
    assert plan((64,) * 3, 1, 8) == ((1, 1, 1), (2, 2, 2), (32, 32, 32))
