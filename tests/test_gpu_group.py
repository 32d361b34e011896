"""Multi-rank parity on ONE GPU: ranks as threads of one process
(paper_2202_11819_b200.dist.ThreadGroup) through the same collective C ABI,
the same P2P stores / epoch flags / host staging / overlap / persistent
cross-rank counters as one process per GPU -- so the exchange paths run on
a one-GPU machine.  2 ranks (z split and x split), 4 ranks (1,2,2) and 8
ranks on the (2,2,2) grid, every case bitwise against the oracle
(tests/group_worker.py).  NCCL is covered by tests/test_gpu_multi.py (it
refuses two ranks on one GPU).
"""
import os
import subprocess
import sys

import pytest

pytestmark = pytest.mark.gpu

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def _run(*args, timeout=900):
    env = dict(os.environ)
    # one hardware queue per stream: no rank's flag wait can sit in front of
    # work another rank's flag depends on (dist.ThreadGroup docstring)
    env["CUDA_DEVICE_MAX_CONNECTIONS"] = "32"
    env.setdefault("J3D_TIMEOUT_S", "120")
    # a hang prints every thread's stack and exits instead of running into the timeout
    env.setdefault("J3D_GROUP_DUMP_S", str(timeout - 60))
    p = subprocess.run([sys.executable, os.path.join(ROOT, "tests", "group_worker.py"), *args],
                       capture_output=True, text=True, timeout=timeout, cwd=ROOT, env=env)
    assert p.returncode == 0 and "GROUP OK" in p.stdout, p.stdout[-4000:] + p.stderr[-4000:]
    return p.stdout


def test_two_ranks_one_gpu():
    """P2P / host staging x every variant x batched / per-block x graph, x-split
    grids, overlap, persistent counters, set_block + refresh, destroy race and
    the epoch-wait watchdog (J3D_ETIMEOUT) with 2 ranks."""
    _run(os.environ.get("J3D_GROUP_CASES", "quick"), "2")


def test_four_ranks_one_gpu():
    _run("quick", "4")


def test_eight_ranks_one_gpu():
    """BASELINE.json's 8-GPU GPU grid (2,2,2): every block face kind is a peer
    face; P2P, host staging, overlap and the persistent launch."""
    _run("quick", "8")


def test_two_ranks_one_gpu_fullsize():
    """bench.py's 2-GPU weak-scaling grid at full size (1536^3 per rank) with both
    ranks on one GPU (116 GB): sampled cells bitwise against the oracle's
    dependency cones, batched and persistent."""
    _run("fullsize")
