"""Inertia of shifted rank-structured matrices: public API over the CUDA engine.

Drop-in for the reference's `h2slice.gldl` entry points
(`/root/reference/pkg/src/h2slice/gldl.py:605-633`):

  generalized_ldl(H, keep_factors=False) -> GldlFactorization
  inertia(H, mu=0.0, max_retries=3)      -> InertiaCount

with the same exceptions (`ShiftHitEigenvalue` on a singular pivot block,
`InertiaUnstable` after the perturbed retries) and the same retry rule
mu <- mu (1 + d) + d, d = 1e-11 max(1, |mu|) (gldl.py:621-632).  Every
factorization runs in libh2ldl.so on the GPU; `inertia_batch` exposes the
shift-batched mode (many shifts per factorization sweep).
"""

from dataclasses import dataclass, field

import numpy as np

from . import _native
from .errors import InertiaUnstable, ShiftHitEigenvalue

RETRY_DELTA = 1e-11
MAX_SHIFT_RETRIES = 3


@dataclass
class InertiaCount:
    """(neg, zero, pos) eigenvalue sign counts (gldl.py:33-46)."""

    neg: int
    zero: int
    pos: int

    @property
    def n(self):
        return self.neg + self.zero + self.pos

    def as_tuple(self):
        return (self.neg, self.zero, self.pos)


@dataclass
class GldlFactorization:
    """Result of one device factorization: inertia plus structural statistics."""

    n: int
    shift: float
    inertia_counts: InertiaCount
    stats: dict = field(default_factory=dict)

    @property
    def kept(self):
        return False

    def reconstruct(self):
        raise ValueError("factors were not kept; the device engine keeps no explicit factors")


def _relative_shift(H):
    return float(H.shift - H.origin().shift)


def _stats_view(st):
    return {
        "fill_blocks": int(st["fill_blocks"]),
        "recompressions": int(st["recompressions"]),
        "rank_added": int(st["rank_added"]),
        "dropped_fro": float(st["dropped_fro"]),
        "max_front": int(st["max_front"]),
        "device": st,
    }


def generalized_ldl(H, keep_factors=False, device=None):
    """Inertia-revealing generalized LDL^T of H (including its shift) on the GPU."""
    if keep_factors:
        raise NotImplementedError(
            "keep_factors=True (validation-only factor reconstruction) is not provided by the "
            "device engine")
    eng = _native.engine_for(H, device)
    counts, status, st = eng.inertia([_relative_shift(H)])
    if status[0] == _native.H2L_SHIFT_SINGULAR:
        raise ShiftHitEigenvalue(H.shift)
    c = InertiaCount(*(int(v) for v in counts[0]))
    return GldlFactorization(n=H.n, shift=H.shift, inertia_counts=c, stats=_stats_view(st))


def inertia_batch(H, mus, max_retries=MAX_SHIFT_RETRIES, device=None, stats_out=None):
    """Inertia of H - mu I for every mu in `mus`, all shifts in batched sweeps.

    Shifts that hit an eigenvalue (singular pivot or a zero count) are
    retried in a further batched sweep with the reference's perturbation; a
    shift still failing after `max_retries` raises InertiaUnstable.
    """
    mus = [float(m) for m in mus]
    eng = _native.engine_for(H, device)
    base = _relative_shift(H)
    out = [None] * len(mus)
    cur = list(mus)
    todo = list(range(len(mus)))
    last = {}
    for attempt in range(max_retries + 1):
        if not todo:
            break
        counts, status, st = eng.inertia([base + cur[q] for q in todo])
        if stats_out is not None:
            stats_out.append(st)
        again = []
        for row, q in enumerate(todo):
            if status[row] == _native.H2L_SHIFT_OK and counts[row, 1] == 0:
                out[q] = InertiaCount(*(int(v) for v in counts[row]))
            else:
                last[q] = ShiftHitEigenvalue(cur[q])
                d = RETRY_DELTA * max(1.0, abs(mus[q]))
                cur[q] = cur[q] * (1.0 + d) + d
                again.append(q)
        todo = again
    if todo:
        q = todo[0]
        raise InertiaUnstable(mus[q], max_retries + 1) from last[q]
    return out


def inertia(H, mu=0.0, max_retries=MAX_SHIFT_RETRIES, device=None):
    """Eigenvalue sign counts of H - mu I (retry wrapper of gldl.py:615-633)."""
    return inertia_batch(H, [mu], max_retries, device)[0]


def ldl_counts_array(H, mus, device=None):
    """Raw engine call: (counts[s,3], status[s], stats) without retries (bench/tests)."""
    eng = _native.engine_for(H, device)
    base = _relative_shift(H)
    return eng.inertia(np.asarray(mus, dtype=np.float64) + base)
