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


class ShardedEvaluator:
    """evaluate(mus) -> negative counts; this rank computes its slice only."""

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
        self.local_eval = local_eval
        self.rounds = 0
        self.local_shifts = 0
        self.gather_s = 0.0

    def __call__(self, mus):
        mus = list(mus)
        n = len(mus)
        sl = split_even(n, self.world)
        lo, hi = sl[self.rank]
        width = max(h - l for l, h in sl)
        mine = np.full(width, -1, dtype=np.int64)
        if hi > lo:
            mine[:hi - lo] = np.asarray(self.local_eval(mus[lo:hi]), dtype=np.int64)
        self.local_shifts += hi - lo
        t0 = time.perf_counter()
        send = self.torch.from_numpy(mine).to(self.dev)
        if self.backend == "nccl":
            recv = self.torch.empty(width * self.world, dtype=self.torch.int64, device=self.dev)
            self.dist.all_gather_into_tensor(recv, send, group=self.group)
            allc = recv.cpu().numpy().reshape(self.world, width)
        else:
            parts = [self.torch.empty_like(send) for _ in range(self.world)]
            self.dist.all_gather(parts, send, group=self.group)
            allc = np.stack([p.numpy() for p in parts])
        self.gather_s += time.perf_counter() - t0
        self.rounds += 1
        out = np.concatenate([allc[r, :h - l] for r, (l, h) in enumerate(sl)])
        return [int(v) for v in out]


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
