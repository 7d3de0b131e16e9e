"""ORACLE — test infrastructure only (tests/, smoke(), bench cpu_baseline).

Dense building blocks of the reference restated on the CPU:
  * `bk_factor` / `bk_inertia`: ctypes bindings of oracle/bk_ref.c, the C
    restatement of `_core/_kernels.pyx:21-168` (bit-identical, see bk_ref.c);
  * `ldl_symmetric` / `inertia_of` / `pivot_tolerance`: `dense.py:50-168`.
The product path never imports this module.
"""

import ctypes
import os
import subprocess
from dataclasses import dataclass

import numpy as np

HERE = os.path.dirname(os.path.abspath(__file__))
LIB = os.path.join(HERE, "lib", "libbkref.so")
PIVOT_TOL_FACTOR = 1e3
EPS = np.finfo(np.float64).eps


class Breakdown(Exception):
    def __init__(self, column):
        self.column = column
        super().__init__(f"singular pivot at column {column}")


def build(force=False):
    """gcc -O2 -ffp-contract=off: products/sums round like the Cython build."""
    src = os.path.join(HERE, "bk_ref.c")
    if not force and os.path.exists(LIB) and os.path.getmtime(LIB) >= os.path.getmtime(src):
        return LIB
    os.makedirs(os.path.dirname(LIB), exist_ok=True)
    subprocess.check_call(["gcc", "-O2", "-ffp-contract=off", "-fPIC", "-shared", src,
                           "-o", LIB, "-lm"])
    return LIB


_lib = None


def _load():
    global _lib
    if _lib is None:
        _lib = ctypes.CDLL(build())
        dp = ctypes.POINTER(ctypes.c_double)
        ip = ctypes.POINTER(ctypes.c_int64)
        _lib.oracle_bk_factor.argtypes = [dp, ctypes.c_int64, ip, ctypes.c_double]
        _lib.oracle_bk_factor.restype = ctypes.c_int
        _lib.oracle_bk_inertia.argtypes = [dp, ctypes.c_int64, ip, ctypes.c_double, ip]
        _lib.oracle_bk_inertia.restype = None
    return _lib


def _dp(a):
    return a.ctypes.data_as(ctypes.POINTER(ctypes.c_double))


def _ip(a):
    return a.ctypes.data_as(ctypes.POINTER(ctypes.c_int64))


def bk_factor(A, ipiv, tol):
    """In-place BK on C-contiguous float64 A (lower triangle); returns 0 or k+1."""
    assert A.flags.c_contiguous and A.dtype == np.float64
    assert ipiv.flags.c_contiguous and ipiv.dtype == np.int64
    return int(_load().oracle_bk_factor(_dp(A), A.shape[0], _ip(ipiv), float(tol)))


def bk_inertia(A, ipiv, zero_tol):
    out = np.zeros(3, dtype=np.int64)
    _load().oracle_bk_inertia(_dp(np.ascontiguousarray(A)), A.shape[0], _ip(ipiv),
                              float(zero_tol), _ip(out))
    return tuple(int(v) for v in out)


def pivot_tolerance(A):
    """1e3 * eps * max|A| (`dense.py:50-53`)."""
    return PIVOT_TOL_FACTOR * EPS * (float(np.abs(A).max()) if A.size else 0.0)


@dataclass
class Ldl:
    L: np.ndarray
    D: np.ndarray
    perm: np.ndarray
    sizes: list


def ldl_symmetric(A):
    """P A P^T = L D L^T via the BK kernel, unpacked (`dense.py:56-124`)."""
    n = A.shape[0]
    if n == 0:
        return Ldl(np.zeros((0, 0)), np.zeros((0, 0)), np.arange(0), [])
    F = np.array(A, dtype=np.float64, order="C", copy=True)
    ipiv = np.zeros(n, dtype=np.int64)
    info = bk_factor(F, ipiv, pivot_tolerance(F))
    if info:
        raise Breakdown(info - 1)
    L = np.eye(n)
    D = np.zeros((n, n))
    perm = np.arange(n)
    sizes = []
    k = 0
    while k < n:
        two = ipiv[k] < 0
        r = k + 1 if two else k          # row exchanged at this step
        kp = int(-ipiv[k] - 1) if two else int(ipiv[k])
        if kp != r:
            L[[r, kp], :k] = L[[kp, r], :k]
            perm[[r, kp]] = perm[[kp, r]]
        w = 2 if two else 1
        D[k:k + w, k:k + w] = np.tril(F[k:k + w, k:k + w]) + np.tril(F[k:k + w, k:k + w], -1).T
        L[k + w:, k:k + w] = F[k + w:, k:k + w]
        sizes.append(w)
        k += w
    return Ldl(L, D, perm, sizes)


def inertia_of(res, zero_tol=None):
    """Sign counts over the pivot blocks (`dense.py:127-168`)."""
    D = res.D
    if zero_tol is None:
        zero_tol = PIVOT_TOL_FACTOR * EPS * (float(np.abs(D).max()) if D.size else 0.0)
    zt = zero_tol
    neg = zero = pos = 0
    k = 0
    for w in res.sizes:
        if w == 1:
            d = D[k, k]
            if abs(d) <= zt:
                zero += 1
            elif d < 0:
                neg += 1
            else:
                pos += 1
        else:
            det = D[k, k] * D[k + 1, k + 1] - D[k + 1, k] ** 2
            tr = D[k, k] + D[k + 1, k + 1]
            if det < -zt * zt:
                neg, pos = neg + 1, pos + 1
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
