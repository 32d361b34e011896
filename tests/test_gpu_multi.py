"""Multi-GPU parity through torchrun (NCCL and NVLink P2P backends).

Runs tests/mp_worker.py on every visible GPU (2 or 4), one process per GPU,
rendezvous on 127.0.0.1.  Skipped when fewer than 2 GPUs are visible.
"""
import os
import socket
import subprocess
import sys

import pytest

from tests.conftest import gpu_count

pytestmark = [pytest.mark.gpu, pytest.mark.multigpu]

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    p = s.getsockname()[1]
    s.close()
    return p


def _torchrun(n, args, timeout):
    """torchrun on 127.0.0.1 with a free port; a port taken between the probe and
    the rendezvous (EADDRINUSE: the ephemeral range is shared with the previous
    run's closing connections) is retried with another one."""
    for _ in range(4):
        cmd = [sys.executable, "-m", "torch.distributed.run", "--nnodes=1", f"--nproc-per-node={n}",
               "--master-addr", "127.0.0.1", "--master-port", str(_free_port()),
               os.path.join(ROOT, "tests", "mp_worker.py"), *args]
        p = subprocess.run(cmd, capture_output=True, text=True, timeout=timeout, cwd=ROOT)
        if p.returncode == 0 or "EADDRINUSE" not in p.stderr:
            return p
    return p


@pytest.mark.skipif(gpu_count() < 2, reason="needs >= 2 GPUs")
def test_multi_gpu_parity():
    n = 4 if gpu_count() >= 4 else 2
    p = _torchrun(n, [os.environ.get("J3D_MP_CASES", "quick")], 1800)
    assert p.returncode == 0 and "MP OK" in p.stdout, p.stdout[-3000:] + p.stderr[-5000:]


@pytest.mark.skipif(gpu_count() < 2, reason="needs >= 2 GPUs")
def test_multi_gpu_fullsize_sampled():
    """Weak scaling at bench.py's full size (1536^3 per GPU), sampled parity."""
    n = 4 if gpu_count() >= 4 else 2
    p = _torchrun(n, ["fullsize"], 1200)
    assert p.returncode == 0 and "MP OK fullsize" in p.stdout, p.stdout[-3000:] + p.stderr[-5000:]
