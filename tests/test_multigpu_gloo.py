"""CPU, world_size 2 (gloo): the sharded multisection driver of multigpu.py.

The device engine is replaced by an exact local evaluator (eigenvalue counts
of a dense symmetric matrix), so the test exercises exactly the host logic
that runs across GPUs: the deterministic shift list, the contiguous shard
rule, the counts all-gather, and the replay that must give estimates
identical on every rank and identical to single-process multisection.
"""

import os
import socket

import numpy as np
import pytest
import torch.multiprocessing as mp

from paper_2311_08618_b200 import bisection
from paper_2311_08618_b200.multigpu import split_even


class _Dummy:
    def __init__(self, n):
        self.n = n


def _spectrum():
    rng = np.random.default_rng(3)
    A = rng.standard_normal((120, 120))
    return np.sort(np.linalg.eigvalsh(A + A.T))


def _counts(w, mus):
    return [int(np.searchsorted(w, mu, side="left")) for mu in mus]


def _free_port():
    with socket.socket() as s:
        s.bind(("127.0.0.1", 0))
        return s.getsockname()[1]


def _worker(rank, world, port, out):
    import torch.distributed as dist

    from paper_2311_08618_b200.multigpu import multisection_distributed

    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    w = _spectrum()
    seen = []

    def local_eval(mus):
        seen.extend(mus)
        return _counts(w, mus)

    ests, ev = multisection_distributed(_Dummy(120), [1, 7, 60, 61, 120], (-40.0, 40.0), 1e-9,
                                        per_rank=15, local_eval=local_eval)
    out[rank] = ([e.value for e in ests], [e.iterations for e in ests], len(seen), ev.rounds)
    dist.destroy_process_group()


def test_split_even_contiguous():
    for n in range(0, 40):
        for world in (1, 2, 3, 8):
            sl = split_even(n, world)
            assert sl[0][0] == 0 and sl[-1][1] == n
            assert all(a[1] == b[0] for a, b in zip(sl, sl[1:]))
            sizes = [h - l for l, h in sl]
            assert max(sizes) - min(sizes) <= 1


def test_two_rank_multisection_identical_to_serial():
    w = _spectrum()
    serial = bisection.multisection(_Dummy(120), [1, 7, 60, 61, 120], (-40.0, 40.0), 1e-9,
                                    batch=30, evaluate=lambda mus: _counts(w, mus))
    world = 2
    mgr = mp.Manager()
    out = mgr.dict()
    port = _free_port()
    ctx = mp.get_context("spawn")
    procs = [ctx.Process(target=_worker, args=(r, world, port, out)) for r in range(world)]
    for p in procs:
        p.start()
    for p in procs:
        p.join(timeout=240)
        assert p.exitcode == 0
    v0, it0, n0, r0 = out[0]
    v1, it1, n1, r1 = out[1]
    assert v0 == v1 == [e.value for e in serial]
    assert it0 == it1 == [e.iterations for e in serial]
    assert r0 == r1
    # each rank factorized only its contiguous half of every round's shifts
    assert abs(n0 - n1) <= r0
    for e, k in zip(serial, [1, 7, 60, 61, 120]):
        assert abs(e.value - w[k - 1]) <= 1e-9


def test_sequential_and_multisection_agree_on_exact_counts():
    w = _spectrum()
    ev = lambda mus: _counts(w, mus)  # noqa: E731
    for batch in (1, 3, 7, 64):
        ests = bisection.multisection(_Dummy(120), [2, 50, 119], (-40.0, 40.0), 1e-8, batch=batch,
                                      evaluate=ev)
        for e in ests:
            # replay the plain sequential loop of spectrum.py:153-166
            a, b, it = -40.0, 40.0, 0
            while b - a >= 1e-8:
                it += 1
                mu = 0.5 * (a + b)
                if ev([mu])[0] >= e.k:
                    b = mu
                else:
                    a = mu
            assert e.value == 0.5 * (a + b) and e.iterations == it, (batch, e.k)


def _failing_worker(rank, world, port, out):
    import torch.distributed as dist

    from paper_2311_08618_b200.multigpu import ShardError, multisection_distributed

    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    w = _spectrum()
    calls = [0]

    def local_eval(mus):
        calls[0] += 1
        if rank == 1 and calls[0] == 2:
            raise ValueError("injected device failure")
        return _counts(w, mus)

    try:
        multisection_distributed(_Dummy(120), [60], (-40.0, 40.0), 1e-9, per_rank=7,
                                 local_eval=local_eval)
        out[rank] = "no error"
    except ShardError:
        out[rank] = "ShardError"
    except ValueError as exc:
        out[rank] = f"ValueError: {exc}"
    dist.destroy_process_group()


def test_failing_rank_raises_everywhere_without_hanging():
    """a rank whose evaluation raises still joins the round's all-gather
    (sentinel rows), so the other ranks raise ShardError instead of blocking."""
    world = 2
    mgr = mp.Manager()
    out = mgr.dict()
    port = _free_port()
    ctx = mp.get_context("spawn")
    procs = [ctx.Process(target=_failing_worker, args=(r, world, port, out)) for r in range(world)]
    for p in procs:
        p.start()
    for p in procs:
        p.join(timeout=240)
        assert p.exitcode == 0
    assert out[0] == "ShardError"
    assert out[1] == "ValueError: injected device failure"


def _static_worker(rank, world, port, out):
    import torch.distributed as dist

    from paper_2311_08618_b200.multigpu import static_partition_distributed

    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    w = _spectrum()
    seen = []

    def ev(mus):
        seen.extend(mus)
        return _counts(w, mus)

    ests = static_partition_distributed(_Dummy(120), 55, 70, (-40.0, 40.0), 1e-9, per_sweep=15,
                                        evaluate=ev)
    out[rank] = ([(e.k, e.value, e.iterations) for e in ests], len(seen))
    dist.destroy_process_group()


def test_k_sharded_static_partition_identical_to_serial():
    """cfg4-style index range: contiguous k chunks per rank (parallel.py:85-96),
    private caches, one all-gather of the estimates; identical to serial."""
    w = _spectrum()
    serial = bisection.multisection(_Dummy(120), list(range(55, 71)), (-40.0, 40.0), 1e-9,
                                    batch=15, evaluate=lambda mus: _counts(w, mus))
    world = 2
    mgr = mp.Manager()
    out = mgr.dict()
    port = _free_port()
    ctx = mp.get_context("spawn")
    procs = [ctx.Process(target=_static_worker, args=(r, world, port, out)) for r in range(world)]
    for p in procs:
        p.start()
    for p in procs:
        p.join(timeout=240)
        assert p.exitcode == 0
    want = [(e.k, e.value, e.iterations) for e in serial]
    assert out[0][0] == out[1][0] == want
    assert out[0][1] > 0 and out[1][1] > 0
