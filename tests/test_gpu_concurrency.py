"""GPU: results must not depend on what else runs on the device.

Regression tests for a pivot-decision race in the BK kernel (a thread read
A(imax, imax) after the row-max barrier while thread 0 could already be
interchanging it) that only showed when other kernels perturbed warp
scheduling: BK bit-exactness and engine counts are checked while a
background stream keeps the SMs busy, and with several concurrent waves.
"""

import ctypes
import threading
import time

import numpy as np
import pytest

from conftest import golden
from oracle import dense_ref
from paper_2311_08618_b200 import _native, configs, construct

pytestmark = pytest.mark.gpu


class Noise:
    """Background fp64 matmuls on a separate torch stream."""

    def __enter__(self):
        import torch

        self.stop = False

        def run():
            s = torch.cuda.Stream()
            with torch.cuda.stream(s):
                a = torch.randn(2048, 2048, dtype=torch.float64, device="cuda")
                while not self.stop:
                    a @ a
                    s.synchronize()

        self.th = threading.Thread(target=run)
        self.th.start()
        time.sleep(0.5)
        return self

    def __exit__(self, *exc):
        self.stop = True
        self.th.join()


@pytest.mark.parametrize("n,count", [(16, 2000), (64, 600), (128, 300)])
def test_bk_bit_exact_under_load(n, count):
    rng = np.random.default_rng(n)
    A = rng.standard_normal((count, n, n))
    A = A + A.transpose(0, 2, 1)
    tol = np.array([dense_ref.pivot_tolerance(a) for a in A])
    with Noise():
        F, ipiv, info = _native.bk_factor_device(A, tol)
    for q in range(count):
        Fo = np.ascontiguousarray(A[q]).copy()
        po = np.zeros(n, dtype=np.int64)
        assert dense_ref.bk_factor(Fo, po, tol[q]) == info[q], q
        assert np.array_equal(po, ipiv[q]) and np.array_equal(Fo, F[q]), q


def test_gemm_matches_naive_under_load():
    lib = _native.load_testing_library()
    f = lib.h2l_internal_gemm_check
    f.argtypes = [ctypes.c_int] * 7 + [ctypes.POINTER(ctypes.c_double)]
    md = ctypes.c_double()
    with Noise():
        for shape in ((128, 128, 128, 16, 8), (64, 64, 64, 100, 8), (100, 70, 50, 20, 4)):
            assert f(0, *shape, 5, ctypes.byref(md)) == 0
            assert md.value == 0.0, shape


def test_engine_counts_concurrent_waves_and_load():
    cloud, kern, tree, st = configs.config_problem("cfg1", seed=0)
    H = construct(kern, tree, st, 1e-8)
    eigs = golden("cfg1.npz")["eigs"]
    eng = _native.DeviceEngine(0)
    eng.upload(H)
    eng.set_option("max_batch", 16)
    eng.set_option("concurrency", 4)
    rng = np.random.default_rng(11)
    with Noise():
        for _ in range(3):
            # shifts inside the dense part of the spectrum: every count is sensitive
            mus = np.sort(rng.uniform(-20.0, 20.0, 96))
            gap = np.min(np.abs(eigs[:, None] - mus[None, :]), axis=0)
            mus = mus[gap > 1e-6]
            counts, status, _ = eng.inertia(mus)
            assert not status.any()
            assert np.array_equal(counts[:, 0], np.searchsorted(eigs, mus))
