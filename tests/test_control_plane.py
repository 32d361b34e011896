"""The shared-memory control plane of multi-rank contexts, on CPU (no GPU).

The P2P and host-staging backends create no NCCL communicator: barriers, the
residual's max and the checksum's sum go through one POSIX shared-memory
segment per rank (csrc/control.cu: a collective sequence number, two value
slots).  jacobi3d_debug_control runs that code on its own; here ranks are
threads of this process (as dist.ThreadGroup runs them) and separate
processes (as torchrun runs them), over hundreds of consecutive collectives
(the two-slot reuse argument of DESIGN.md §7), and a missing rank must end in
J3D_ETIMEOUT rather than a hang.
"""
import multiprocessing as mp
import os
import random
import threading

import pytest

from paper_2202_11819_b200 import jacobi3d as jb

M64 = (1 << 64) - 1


def _values(n_ranks, rounds, seed):
    rng = random.Random(seed)
    return [[rng.getrandbits(64) if rng.random() < 0.9 else rng.choice([0, M64, 1 << 63]) for _ in range(rounds)]
            for _ in range(n_ranks)]


def _check(vals, outs):
    n_ranks, rounds = len(vals), len(vals[0])
    for r in range(rounds):
        want_sum = sum(v[r] for v in vals) & M64
        want_max = max(v[r] for v in vals)
        for rank in range(n_ranks):
            s, m = outs[rank]
            assert s[r] == want_sum, (rank, r)
            assert m[r] == want_max, (rank, r)


@pytest.mark.parametrize("n_ranks,rounds", [(2, 300), (3, 200), (8, 150)])
def test_thread_ranks(n_ranks, rounds):
    key = os.urandom(128)
    vals = _values(n_ranks, rounds, seed=n_ranks)
    outs, errs = [None] * n_ranks, []

    def body(rank):
        try:
            outs[rank] = jb.debug_control(key, rank, n_ranks, vals[rank])
        except Exception as e:  # noqa: BLE001
            errs.append(e)

    ts = [threading.Thread(target=body, args=(r,)) for r in range(n_ranks)]
    for t in ts:
        t.start()
    for t in ts:
        t.join(timeout=120)
    assert not errs, errs
    _check(vals, outs)


def _proc(key, rank, n_ranks, values, q):
    from paper_2202_11819_b200 import jacobi3d as jb_

    q.put((rank, jb_.debug_control(key, rank, n_ranks, values)))


def test_process_ranks():
    n_ranks, rounds = 2, 200
    key = os.urandom(128)
    vals = _values(n_ranks, rounds, seed=7)
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    ps = [ctx.Process(target=_proc, args=(key, r, n_ranks, vals[r], q)) for r in range(n_ranks)]
    for p in ps:
        p.start()
    outs = [None] * n_ranks
    for _ in range(n_ranks):
        rank, out = q.get(timeout=120)
        outs[rank] = out
    for p in ps:
        p.join(timeout=60)
        assert p.exitcode == 0
    _check(vals, outs)


def test_missing_rank_times_out(monkeypatch):
    monkeypatch.setenv("J3D_TIMEOUT_S", "1")
    with pytest.raises(jb.Jacobi3DError) as e:
        jb.debug_control(os.urandom(128), 0, 2, [1, 2, 3])
    assert e.value.code == jb.ETIMEOUT
