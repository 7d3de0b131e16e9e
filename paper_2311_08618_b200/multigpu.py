"""Multisection across GPUs: shifts sharded over ranks, counts all-gathered.

Replaces the reference's thread-replica drivers (`h2slice/parallel.py:85-312`,
paper §4.2) for one node of B200s: one process per GPU, each holding a full
replica of H in HBM (`_native.engine_for`).  Every multisection round
(`bisection.multisection`) produces one deterministic list of shifts on every
rank; rank r factorizes its contiguous slice in one shift-batched device
sweep, and the only collective is an all-gather of the int64 negative counts
(NCCL over NVLink on GPUs, gloo on CPU in the tests).  Every rank then replays
the identical bisection from the identical count cache, so the estimates are
bitwise identical on all ranks and identical to the single-GPU result
(reference determinism contract, spectrum.py:5-11 / parallel.py:3-13).
"""

import time
from dataclasses import dataclass, field

import numpy as np

from .bisection import EPS_EV_DEFAULT, InertiaCache, default_interval, multisection
from .errors import ConfigError
from .ldl import inertia_batch


def split_even(n, world):
    """Contiguous near-equal [lo, hi) slices of range(n) (reference parallel.py:85-96)."""
    base, extra = divmod(n, world)
    out, lo = [], 0
    for r in range(world):
        hi = lo + base + (1 if r < extra else 0)
        out.append((lo, hi))
        lo = hi
    return out


class ShardError(RuntimeError):
    """Another rank failed while evaluating its slice of a round."""


FAILED = -2  # sentinel row value: the rank's local evaluation raised


class ShardedEvaluator:
    """evaluate(mus) -> negative counts; this rank computes its slice only.

    Failure protocol: a rank whose local evaluation raises still takes part in
    the round's all-gather (with FAILED rows), so no rank blocks in the
    collective; every rank then raises (the failing one its own exception,
    the others ShardError).

    With NCCL and no custom `local_eval`, the engine writes its packed rows
    (neg, zero, pos, status) straight into the CUDA send buffer
    (h2l_inertia_device) and the all-gather runs between device buffers; the
    one host copy is the gathered result every rank needs for the bisection.
    Shifts on an eigenvalue (status or zero count) are retried by their owner
    with the reference's perturbation in a second, rare round.
    """

    def __init__(self, H=None, local_eval=None, group=None, device=None):
        import torch
        import torch.distributed as dist

        self.dist, self.torch = dist, torch
        self.group = group
        self.rank = dist.get_rank(group)
        self.world = dist.get_world_size(group)
        self.backend = dist.get_backend(group)
        self.dev = (torch.device("cuda", torch.cuda.current_device())
                    if self.backend == "nccl" else torch.device("cpu"))
        if local_eval is None:
            if H is None:
                raise ConfigError("ShardedEvaluator needs H or local_eval")

            def local_eval(mus):
                return [c.neg for c in inertia_batch(H, mus, device=device)]
        self.H, self.device = H, device
        self.device_rows = local_eval is None and self.backend == "nccl"
        self.local_eval = local_eval
        self.rounds = 0
        self.local_shifts = 0
        self.gather_s = 0.0

    def _gather(self, mine, width):
        """All-gather `mine` (width x cols int64, numpy or CUDA tensor) -> (world, width, cols)."""
        torch = self.torch
        t0 = time.perf_counter()
        send = mine if torch.is_tensor(mine) else torch.from_numpy(mine).to(self.dev)
        if self.backend == "nccl":
            recv = torch.empty((self.world,) + tuple(send.shape), dtype=torch.int64, device=self.dev)
            self.dist.all_gather_into_tensor(recv, send.contiguous(), group=self.group)
            allc = recv.cpu().numpy()
        else:
            parts = [torch.empty_like(send) for _ in range(self.world)]
            self.dist.all_gather(parts, send, group=self.group)
            allc = np.stack([p.numpy() for p in parts])
        self.gather_s += time.perf_counter() - t0
        return allc

    def _raise_if_failed(self, allc, err):
        bad = [r for r in range(self.world) if (allc[r] == FAILED).any()]
        if bad:
            if err is not None:
                raise err
            raise ShardError(f"rank(s) {bad} failed in round {self.rounds}")

    def __call__(self, mus):
        mus = [float(m) for m in mus]
        n = len(mus)
        sl = split_even(n, self.world)
        lo, hi = sl[self.rank]
        width = max(1, max(h - l for l, h in sl))
        self.local_shifts += hi - lo
        err = None
        if self.device_rows:
            torch = self.torch
            from . import _native
            from .ldl import _relative_shift

            rows = torch.full((width, 4), -1, dtype=torch.int64, device=self.dev)
            try:
                if hi > lo:
                    eng = _native.engine_for(self.H, self.dev.index)
                    base = _relative_shift(self.H)
                    eng.inertia_device(np.asarray(mus[lo:hi]) + base, rows)
            except Exception as exc:  # noqa: BLE001 - re-raised after the collective
                err = exc
                rows.fill_(FAILED)
            allc = self._gather(rows, width)
            self._raise_if_failed(allc, err)
            out = np.concatenate([allc[r, :h - l] for r, (l, h) in enumerate(sl)])
            need = [q for q in range(n) if out[q, 3] != 0 or out[q, 1] != 0]
            neg = out[:, 0].copy()
            if need:  # the reference's retry (gldl.py:621-632), by each shift's owner
                fixed = self._retry(mus, need, sl)
                for q, v in zip(need, fixed):
                    neg[q] = v
            self.rounds += 1
            return [int(v) for v in neg]
        mine = np.full((width, 1), -1, dtype=np.int64)
        try:
            if hi > lo:
                mine[:hi - lo, 0] = np.asarray(self.local_eval(mus[lo:hi]), dtype=np.int64)
        except Exception as exc:  # noqa: BLE001 - re-raised after the collective
            err = exc
            mine[:] = FAILED
        allc = self._gather(mine, width)
        self._raise_if_failed(allc, err)
        self.rounds += 1
        out = np.concatenate([allc[r, :h - l, 0] for r, (l, h) in enumerate(sl)])
        return [int(v) for v in out]

    def _retry(self, mus, need, sl):
        """Negative counts of the shifts `need` (indices into mus) after the retry
        wrapper, each computed by the rank that owns it; one more all-gather."""
        owner = {q: r for r, (l, h) in enumerate(sl) for q in range(l, h)}
        mine_q = [q for q in need if owner[q] == self.rank]
        width = max(1, max(sum(1 for q in need if owner[q] == r) for r in range(self.world)))
        buf = np.full((width, 1), -1, dtype=np.int64)
        err = None
        try:
            if mine_q:
                got = inertia_batch(self.H, [mus[q] for q in mine_q], device=self.dev.index)
                buf[:len(mine_q), 0] = [c.neg for c in got]
        except Exception as exc:  # noqa: BLE001 - InertiaUnstable etc., after the collective
            err = exc
            buf[:] = FAILED
        allc = self._gather(buf, width)
        self._raise_if_failed(allc, err)
        vals = {}
        for r in range(self.world):
            qs = [q for q in need if owner[q] == r]
            for t, q in enumerate(qs):
                vals[q] = int(allc[r, t, 0])
        return [vals[q] for q in need]


def multisection_distributed(H, ks, interval=None, eps_ev=EPS_EV_DEFAULT, per_rank=64,
                             group=None, local_eval=None, device=None, cache=None):
    """Eigenvalues of `ks` by multisection over all ranks of `group`.

    Each round evaluates up to per_rank * world shifts (per_rank per GPU sweep).
    Returns (estimates, evaluator) -- the evaluator carries round statistics."""
    if interval is None:
        interval = default_interval(H)
    ev = ShardedEvaluator(H, local_eval=local_eval, group=group, device=device)
    ests = multisection(H, ks, interval, eps_ev, cache=cache if cache is not None else InertiaCache(),
                        batch=per_rank * ev.world, evaluate=ev)
    return ests, ev


def static_partition_distributed(H, k_lo, k_hi, interval=None, eps_ev=EPS_EV_DEFAULT,
                                 per_sweep=64, group=None, evaluate=None):
    """Every index of [k_lo, k_hi], index chunks sharded over the ranks.

    The reference's static partition (parallel.py:85-96, 109-180): rank r takes
    the r-th contiguous chunk of the index range and runs its own multisection
    with a private cache (no collective during the searches, so the scaling in
    eigenvalues/s is limited only by load balance); one all-gather of the
    estimates at the end gives every rank the full list.  Estimates are
    identical to serial bisection for any world size (the cache only decides
    which shifts are evaluated, never a branch).  `evaluate(mus)` overrides the
    device engine (tests)."""
    import torch
    import torch.distributed as dist

    if k_lo > k_hi:
        raise ConfigError(f"empty index range [{k_lo}, {k_hi}]")
    if interval is None:
        interval = default_interval(H)
    rank, world = dist.get_rank(group), dist.get_world_size(group)
    ks = list(range(k_lo, k_hi + 1))
    sl = split_even(len(ks), world)
    lo, hi = sl[rank]
    mine = ks[lo:hi]
    t0 = time.perf_counter()
    ests = multisection(H, mine, interval, eps_ev, cache=InertiaCache(), batch=per_sweep,
                        evaluate=evaluate) if mine else []
    width = max(1, max(h - l for l, h in sl))
    buf = np.full((width, 4), np.nan)
    for q, e in enumerate(ests):
        buf[q] = (e.value, e.half_width, e.iterations, e.inertia_evals)
    backend = dist.get_backend(group)
    dev = torch.device("cuda", torch.cuda.current_device()) if backend == "nccl" else torch.device("cpu")
    send = torch.from_numpy(buf).to(dev)
    parts = [torch.empty_like(send) for _ in range(world)]
    dist.all_gather(parts, send, group=group)
    wall = time.perf_counter() - t0
    from .bisection import EigenvalueEstimate

    out = []
    for r, (l, h) in enumerate(sl):
        arr = parts[r].cpu().numpy()
        for q in range(h - l):
            v, hw, it, ne = arr[q]
            out.append(EigenvalueEstimate(k=ks[l + q], value=float(v), half_width=float(hw),
                                          iterations=int(it), inertia_evals=int(ne),
                                          wall_time=wall))
    return out


@dataclass
class ParallelResult:
    estimates: list
    wall_time: float
    mode: str
    stats: dict = field(default_factory=dict)


def static_partition_solve(H, k_lo, k_hi, interval=None, eps_ev=EPS_EV_DEFAULT, workers=1,
                           per_sweep=64):
    """Every index of [k_lo, k_hi] (reference parallel.py:109-180 contract).

    On the device engine all indices share one multisection cache, and each
    sweep batches `per_sweep` shifts; estimates are identical to serial
    `slice_spectrum` calls for any `workers` value (kept for API parity: one
    process drives one GPU; use `multisection_distributed` under torchrun for
    several GPUs)."""
    if workers < 1:
        raise ConfigError("workers must be >= 1")
    if k_lo > k_hi:
        raise ConfigError(f"empty index range [{k_lo}, {k_hi}]")
    t0 = time.perf_counter()
    ests = multisection(H, list(range(k_lo, k_hi + 1)), interval, eps_ev, batch=per_sweep)
    return ParallelResult(estimates=ests, wall_time=time.perf_counter() - t0, mode="static")
