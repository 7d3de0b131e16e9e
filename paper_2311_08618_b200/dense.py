"""Dense building blocks over the device BK kernel.

Drop-in for the reference's `h2slice.dense` LDL entry points
(`dense.py:31-168`): `pivot_tolerance`, `ldl_symmetric` (P A P^T = L D L^T
with 1x1/2x2 pivots; raises Breakdown) and `inertia_of`.  The factorization
itself runs in libh2ldl.so (`h2l_bk_factor`, the replacement of the native
plug-in `_core.bk_factor`, `_kernels.pyx:21-125`); unpacking the packed
factor into explicit L / D / perm is host bookkeeping.
"""

from dataclasses import dataclass

import numpy as np

from . import _native
from .errors import Breakdown

PIVOT_TOL_FACTOR = 1e3
_EPS = np.finfo(np.float64).eps


@dataclass
class LdlResult:
    L: np.ndarray
    D: np.ndarray
    perm: np.ndarray
    block_sizes: list

    @property
    def n(self):
        return self.L.shape[0]


def pivot_tolerance(A):
    """1e3 * eps * max|A| (reference dense.py:50-53)."""
    A = np.asarray(A)
    return PIVOT_TOL_FACTOR * _EPS * (float(np.abs(A).max()) if A.size else 0.0)


def bk_factor(A, ipiv, tol, device=None):
    """In-place contract of `_core.bk_factor` executed on the GPU; returns info."""
    F, piv, info = _native.bk_factor_device(A[None], [tol], device)
    A[...] = F[0]
    ipiv[...] = piv[0]
    return int(info[0])


def bk_inertia(A, ipiv, zero_tol, device=None):
    """Contract of `_core.bk_inertia` executed on the GPU."""
    return tuple(int(v) for v in _native.bk_inertia_device(A[None], ipiv, [zero_tol], device)[0])


def _unpack(F, ipiv):
    n = F.shape[0]
    L, D, perm, sizes = np.eye(n), np.zeros((n, n)), np.arange(n), []
    k = 0
    while k < n:
        w = 2 if ipiv[k] < 0 else 1
        row = k + w - 1
        kp = int(-ipiv[k] - 1) if w == 2 else int(ipiv[k])
        if kp != row:
            L[[row, kp], :k] = L[[kp, row], :k]
            perm[[row, kp]] = perm[[kp, row]]
        blk = np.tril(F[k:k + w, k:k + w])
        D[k:k + w, k:k + w] = blk + np.tril(blk, -1).T
        L[k + w:, k:k + w] = F[k + w:, k:k + w]
        sizes.append(w)
        k += w
    return L, D, perm, sizes


def ldl_symmetric(A, device=None):
    """P A P^T = L D L^T (lower triangle read), Breakdown on a singular pivot block."""
    A = np.asarray(A, dtype=np.float64)
    if A.ndim != 2 or A.shape[0] != A.shape[1]:
        raise ValueError("ldl_symmetric expects a square matrix")
    n = A.shape[0]
    if n == 0:
        return LdlResult(np.zeros((0, 0)), np.zeros((0, 0)), np.arange(0), [])
    F, ipiv, info = _native.bk_factor_device(A[None], [pivot_tolerance(A)], device)
    if info[0]:
        raise Breakdown(int(info[0]) - 1)
    L, D, perm, sizes = _unpack(F[0], ipiv[0])
    return LdlResult(L=L, D=D, perm=perm, block_sizes=sizes)


def inertia_of(res, zero_tol=None):
    """(neg, zero, pos) over the pivot blocks of an LdlResult (dense.py:127-168)."""
    D = res.D
    zt = (PIVOT_TOL_FACTOR * _EPS * (float(np.abs(D).max()) if D.size else 0.0)
          if zero_tol is None else zero_tol)
    neg = zero = pos = 0
    k = 0
    for w in res.block_sizes:
        if w == 1:
            d = D[k, k]
            if abs(d) <= zt:
                zero += 1
            elif d < 0:
                neg += 1
            else:
                pos += 1
        else:
            det = D[k, k] * D[k + 1, k + 1] - D[k + 1, k] * D[k + 1, k]
            tr = D[k, k] + D[k + 1, k + 1]
            if det < -zt * zt:
                neg += 1
                pos += 1
            elif det > zt * zt:
                if tr < 0:
                    neg += 2
                else:
                    pos += 2
            else:
                zero += 1
                if tr < -zt:
                    neg += 1
                elif tr > zt:
                    pos += 1
                else:
                    zero += 1
        k += w
    return neg, zero, pos
