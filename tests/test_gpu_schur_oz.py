"""GPU: the INT8-tensor-core (Ozaki) Schur update C -= X Bg^T (k_schur_oz.cu).

The kernel slices every row of X and Bg into 8 exact 7-bit integer slices under the
row's power-of-two scale and sums the 36 slice-pair products of weight >= 2^-63 in
int32 tensor memory.  The test target is one diagonal segment (C itself), so the
production epilogue writes C[r, c] -= (X Bg^T)[r, c] for c >= r and the mirrored
C[c, r].  Bar: the error is within 2^-52 * K * max|X_r| * max|Bg_c| of the exact
product (computed here in extended precision), i.e. fp64 accuracy.  Shapes cover
ragged R and K, K below one 64-byte block, rows with widely different scales, zero
rows, and several shifts.
"""

import ctypes

import numpy as np
import pytest

from paper_2311_08618_b200 import _native

pytestmark = pytest.mark.gpu

_f64p = ctypes.POINTER(ctypes.c_double)


def _oz(X, B, reps=0):
    lib = _native.load_testing_library()
    f = lib.h2l_internal_schur_oz
    f.argtypes = [ctypes.c_int, ctypes.c_int, ctypes.c_int, ctypes.c_int, _f64p, _f64p, _f64p,
                  ctypes.c_int, _f64p, ctypes.c_int]
    s, R, K = X.shape
    X = np.ascontiguousarray(X)
    B = np.ascontiguousarray(B)
    C = np.zeros((s, R, R))
    ms = ctypes.c_double(0.0)
    rc = f(0, R, K, s, X.ctypes.data_as(_f64p), B.ctypes.data_as(_f64p), C.ctypes.data_as(_f64p),
           reps, ctypes.byref(ms), 0)
    assert rc == 0, lib.h2l_testing_last_error().decode()
    return C, ms.value


def _exact(X, B):
    return np.einsum("srk,sck->src", X.astype(np.longdouble), B.astype(np.longdouble))


@pytest.mark.parametrize("s,R,K", [(1, 128, 64), (2, 300, 200), (1, 37, 5), (3, 257, 129),
                                   (1, 64, 448), (2, 513, 70)])
def test_schur_oz_matches_exact_product(s, R, K):
    rng = np.random.default_rng(R * 1000 + K)
    X = rng.standard_normal((s, R, K)) * np.exp2(rng.integers(-30, 30, (s, R, 1)))
    B = rng.standard_normal((s, R, K)) * np.exp2(rng.integers(-30, 30, (s, R, 1)))
    X[:, R // 3, :] = 0.0                     # a zero row
    B[:, :, K // 2] *= 1e-12                  # a column far below the row scale
    C, _ = _oz(X, B)
    ex = _exact(X, B)
    mx = np.abs(X).max(axis=2)
    mb = np.abs(B).max(axis=2)
    for z in range(s):
        U = np.triu(ex[z])
        want = -(U + U.T - np.diag(np.diag(ex[z])))   # upper written, mirrored below
        scale = K * np.outer(mx[z], mb[z])
        scale = np.maximum(np.triu(scale), np.triu(scale).T)
        err = np.abs(C[z].astype(np.longdouble) - want)
        ratio = err / np.where(scale > 0, scale, 1.0)
        assert float(ratio.max()) <= 2.0 ** -52, float(ratio.max())


def test_schur_oz_at_least_as_accurate_as_fp64_gemm():
    rng = np.random.default_rng(5)
    s, R, K = 1, 384, 320
    X = rng.standard_normal((s, R, K))
    B = rng.standard_normal((s, R, K))
    C, _ = _oz(X, B)
    ex = _exact(X, B)[0]
    iu = np.triu_indices(R)
    e_oz = float(np.abs(-C[0].astype(np.longdouble) - ex)[iu].max())
    e_64 = float(np.abs((X[0] @ B[0].T).astype(np.longdouble) - ex)[iu].max())
    assert e_oz <= 4 * e_64, (e_oz, e_64)


@pytest.mark.parametrize("name", ["mini_cfg1_1024", "mini_cfg3_1024", "grid3d6_hss_e8",
                                  "grid3d6_h2_e6", "circle256_h2_e8", "grid2d10_h2_e7"])
def test_engine_counts_with_dmma_schur(name):
    """The engine with the Schur update on the fp64 DMMA pipe (schur_arith 0; the default
    is the INT8 path, exercised by every other engine test) returns the reference's
    counts on every golden shift."""
    from conftest import golden
    from paper_2311_08618_b200 import h2matrix

    H = h2matrix.load_payload(f"tests/golden/h_{name}.npz")
    z = golden(f"counts_{name}.npz")
    eng = _native.engine_for(H)
    mus = np.asarray(z["mus"], dtype=np.float64)
    try:
        eng.set_option("schur_arith", 0)
        counts, status, st = eng.inertia(mus)
    finally:
        eng.set_option("schur_arith", 1)
    assert not status.any()
    assert np.array_equal(counts, z["counts"]), (name, counts.tolist(), z["counts"].tolist())
