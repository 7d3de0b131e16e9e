"""Stress: batched device BK vs the oracle C kernel (bit-exact) on many matrices."""
import os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np
from oracle import dense_ref
from paper_2311_08618_b200 import _native

for n, count in ((128, 3000), (64, 3000), (200, 600)):
    rng = np.random.default_rng(n)
    A = rng.standard_normal((count, n, n))
    A = A + A.transpose(0, 2, 1)
    # make some strongly indefinite with small diagonal -> lots of 2x2 pivots
    A[::2] -= np.eye(n) * 0.0
    A[1::2, np.arange(n), np.arange(n)] *= 1e-3
    tol = np.array([dense_ref.pivot_tolerance(a) for a in A])
    F, ipiv, info = _native.bk_factor_device(A, tol)
    bad = 0
    for q in range(count):
        Fo = np.ascontiguousarray(A[q]).copy()
        po = np.zeros(n, dtype=np.int64)
        io = dense_ref.bk_factor(Fo, po, tol[q])
        if io != info[q] or not np.array_equal(po, ipiv[q]) or not np.array_equal(Fo, F[q]):
            bad += 1
    print(f"n={n} count={count} mismatches={bad}", flush=True)
