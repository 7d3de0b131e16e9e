"""Eigenvalue location by inertia bisection (the caller of the hot path).

Semantics follow the reference's spectrum slicing (`h2slice/spectrum.py`):
midpoints are always mu = 0.5 (a + b) of the current bracket of the ORIGINAL
interval, the loop runs `while b - a >= eps_ev`, nu(mu) >= k moves b, cached
counts at other shifts resolve a branch only through monotonicity
(`spectrum.py:97-110`), endpoints are verified lazily (`spectrum.py:167-170`)
and `default_interval` is the Gershgorin interval of the dense realisation
with the upper end padded by 1e-10 max(1, |lo|, |hi|) (`spectrum.py:113-124`).

On top of the sequential `slice_spectrum` (one shift per device sweep) this
module adds the shift-batched multisection driver `multisection`: each round
evaluates, in ONE batched device call, every midpoint of the next q
bisection levels of every unresolved index that the cache cannot resolve,
then replays the exact sequential bisection from the cache.  Because every
decision is still taken on the same recursive midpoints with the same counts,
the estimates are bitwise identical to sequential bisection; only the number
of evaluated shifts grows (2^q - 1 per q levels) while the number of device
sweeps drops by q.  The evaluator is pluggable so that the multi-GPU driver
(`multigpu.py`) can shard the shift list across ranks.
"""

import bisect as _bisect
import json
import threading
import time
from dataclasses import asdict, dataclass

import numpy as np

from .errors import ConfigError, H2SliceError, NotInInterval, OracleTooLarge
from .h2matrix import gershgorin_interval, reconstruct_dense
from .ldl import inertia, inertia_batch

EPS_EV_DEFAULT = 1e-5
MAX_BISECT_ITERATIONS = 200


@dataclass
class EigenvalueEstimate:
    """value = bracket midpoint; the eigenvalue lies within half_width of it."""

    k: int
    value: float
    half_width: float
    iterations: int
    inertia_evals: int
    wall_time: float

    def to_json(self):
        return json.dumps(asdict(self), sort_keys=True)

    @staticmethod
    def from_json(text):
        return EigenvalueEstimate(**json.loads(text))


class InertiaCache:
    """Sorted store of (shift -> negative count); lookups use monotonicity."""

    def __init__(self):
        self._keys = []
        self._vals = {}
        self._lock = threading.Lock()
        self.fresh_evals = 0
        self.hits = 0

    def __len__(self):
        return len(self._keys)

    def exact(self, mu):
        with self._lock:
            return self._vals.get(mu)

    def le(self, mu):
        """Count at the largest cached shift <= mu (or None)."""
        with self._lock:
            i = _bisect.bisect_right(self._keys, mu)
            return self._vals[self._keys[i - 1]] if i else None

    def ge(self, mu):
        """Count at the smallest cached shift >= mu (or None)."""
        with self._lock:
            i = _bisect.bisect_left(self._keys, mu)
            return self._vals[self._keys[i]] if i < len(self._keys) else None

    def insert(self, mu, nu):
        with self._lock:
            if mu not in self._vals:
                _bisect.insort(self._keys, mu)
                self._vals[mu] = nu

    def resolve(self, mu, k):
        """True / False when the cache decides nu(mu) >= k, else None."""
        lv = self.le(mu)
        if lv is not None and lv >= k:
            return True
        gv = self.ge(mu)
        if gv is not None and gv < k:
            return False
        return None


def _branch(H, mu, k, cache):
    got = cache.resolve(mu, k)
    if got is not None:
        cache.hits += 1
        return got
    v = inertia(H, mu).neg
    cache.insert(mu, v)
    cache.fresh_evals += 1
    return v >= k


def default_interval(H, cap=None):
    """Gershgorin interval of the dense realisation, upper end padded."""
    try:
        A = reconstruct_dense(H, cap)
    except OracleTooLarge as exc:
        raise OracleTooLarge(exc.n, exc.cap,
                             message=f"{exc}; supply an explicit search interval") from None
    lo, hi = gershgorin_interval(A)
    return lo, hi + 1e-10 * max(1.0, abs(lo), abs(hi))


def _check_args(H, k, interval, eps_ev):
    if not 1 <= k <= H.n:
        raise ConfigError(f"k={k} outside 1..{H.n}")
    if eps_ev <= 0:
        raise ConfigError("eps_ev must be positive")
    a0, b0 = float(interval[0]), float(interval[1])
    if not a0 < b0:
        raise ConfigError(f"empty search interval ({a0}, {b0})")
    return a0, b0


def slice_spectrum(H, k, interval=None, eps_ev=EPS_EV_DEFAULT, cache=None):
    """k-th smallest eigenvalue (1-based) by bisection, one shift per sweep."""
    t0 = time.perf_counter()
    if interval is None:
        interval = default_interval(H)
    a0, b0 = _check_args(H, k, interval, eps_ev)
    cache = InertiaCache() if cache is None else cache
    fresh0 = cache.fresh_evals
    a, b = a0, b0
    moved_a = moved_b = False
    it = 0
    while b - a >= eps_ev:
        it += 1
        if it > MAX_BISECT_ITERATIONS:
            raise H2SliceError(f"bisection exceeded {MAX_BISECT_ITERATIONS} iterations; "
                               f"interval ({a0}, {b0}) with eps_ev={eps_ev} is unreasonable")
        mu = 0.5 * (a + b)
        if _branch(H, mu, k, cache):
            b, moved_b = mu, True
        else:
            a, moved_a = mu, True
    if not moved_a and _branch(H, a0, k, cache):
        raise NotInInterval(k, a0, b0)
    if not moved_b and not _branch(H, b0, k, cache):
        raise NotInInterval(k, a0, b0)
    return EigenvalueEstimate(k=k, value=0.5 * (a + b), half_width=0.5 * (b - a), iterations=it,
                              inertia_evals=cache.fresh_evals - fresh0,
                              wall_time=time.perf_counter() - t0)


def slice_range(H, k_lo, k_hi, interval=None, eps_ev=EPS_EV_DEFAULT, cache=None):
    """Every index of [k_lo, k_hi] with one shared cache (extremes first)."""
    if k_lo > k_hi:
        raise ConfigError(f"empty index range [{k_lo}, {k_hi}]")
    if interval is None:
        interval = default_interval(H)
    cache = InertiaCache() if cache is None else cache
    order = [k_lo] if k_lo == k_hi else [k_lo, k_hi]
    order += list(range(k_lo + 1, k_hi))
    got = {k: slice_spectrum(H, k, interval, eps_ev, cache) for k in order}
    return [got[k] for k in range(k_lo, k_hi + 1)]


# ------------------------------------------------------------ multisection
class _Walk:
    __slots__ = ("k", "a", "b", "a0", "b0", "moved_a", "moved_b", "it", "evals")

    def __init__(self, k, a0, b0):
        self.k, self.a, self.b, self.a0, self.b0 = k, a0, b0, a0, b0
        self.moved_a = self.moved_b = False
        self.it = 0
        self.evals = 0

    def done(self, eps_ev):
        return not (self.b - self.a >= eps_ev)


def _frontier(w, q, eps_ev, cache):
    """Midpoints of the next q bisection levels of w the cache cannot resolve."""
    out = []
    nodes = [(w.a, w.b)]
    for _ in range(q):
        nxt = []
        for a, b in nodes:
            if not (b - a >= eps_ev):
                continue
            mu = 0.5 * (a + b)
            if cache.resolve(mu, w.k) is None and cache.exact(mu) is None:
                out.append(mu)
            nxt += [(a, mu), (mu, b)]
        nodes = nxt
    return out


def _advance(w, q, eps_ev, cache):
    """Replay up to q sequential bisection steps from the cache."""
    for _ in range(q):
        if w.done(eps_ev):
            return
        w.it += 1
        if w.it > MAX_BISECT_ITERATIONS:
            raise H2SliceError(f"bisection exceeded {MAX_BISECT_ITERATIONS} iterations")
        mu = 0.5 * (w.a + w.b)
        got = cache.resolve(mu, w.k)
        if got is None:  # cannot happen: every unresolved midpoint was evaluated
            raise H2SliceError(f"multisection walk found no count at {mu!r}")
        if got:
            w.b, w.moved_b = mu, True
        else:
            w.a, w.moved_a = mu, True


def device_evaluator(H, device=None, stats=None):
    """evaluate(mus) -> negative counts, through the batched device engine."""

    def evaluate(mus):
        return [c.neg for c in inertia_batch(H, mus, device=device, stats_out=stats)]

    return evaluate


def multisection(H, ks, interval=None, eps_ev=EPS_EV_DEFAULT, cache=None, batch=64,
                 evaluate=None):
    """Eigenvalues of every k in `ks` by batched multisection (see module doc).

    Estimates are identical to `slice_spectrum` with the same interval and
    eps_ev.  `batch` bounds the shifts per device sweep; `evaluate(mus)`
    returns negative counts (defaults to the device engine of H)."""
    t0 = time.perf_counter()
    if interval is None:
        interval = default_interval(H)
    ks = [int(k) for k in ks]
    if not ks:
        return []
    a0 = b0 = None
    for k in ks:
        a0, b0 = _check_args(H, k, interval, eps_ev)
    cache = InertiaCache() if cache is None else cache
    evaluate = device_evaluator(H) if evaluate is None else evaluate
    walks = {k: _Walk(k, a0, b0) for k in ks}
    rounds = 0
    while True:
        live = [w for w in walks.values() if not w.done(eps_ev)]
        if not live:
            break
        # depth q so that the union of frontiers fits the batch
        per = max(1, batch // len(live))
        q = max(1, int(np.floor(np.log2(per + 1))))
        want = []
        seen = set()
        for w in live:
            for mu in _frontier(w, q, eps_ev, cache):
                if mu not in seen:
                    seen.add(mu)
                    want.append(mu)
        if want:
            negs = evaluate(want)
            for mu, v in zip(want, negs):
                cache.insert(mu, int(v))
            cache.fresh_evals += len(want)
            share = len(want) / len(live)
            for w in live:
                w.evals += share
        for w in live:
            _advance(w, q, eps_ev, cache)
        rounds += 1
    # lazy endpoint checks, batched (spectrum.py:167-170)
    ends = sorted({a0 for w in walks.values() if not w.moved_a}
                  | {b0 for w in walks.values() if not w.moved_b})
    ends = [mu for mu in ends if cache.exact(mu) is None]
    if ends:
        for mu, v in zip(ends, evaluate(ends)):
            cache.insert(mu, int(v))
        cache.fresh_evals += len(ends)
    for w in walks.values():
        if not w.moved_a and cache.resolve(a0, w.k):
            raise NotInInterval(w.k, a0, b0)
        if not w.moved_b and not cache.resolve(b0, w.k):
            raise NotInInterval(w.k, a0, b0)
    wall = time.perf_counter() - t0
    return [EigenvalueEstimate(k=w.k, value=0.5 * (w.a + w.b), half_width=0.5 * (w.b - w.a),
                               iterations=w.it, inertia_evals=int(round(w.evals)),
                               wall_time=wall) for w in (walks[k] for k in ks)]


@dataclass
class ShiftAccuracyReport:
    mu: float
    residual_norm: float
    min_eig_gap: float
    matrix_norm: float
    satisfied: bool
