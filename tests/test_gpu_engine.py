"""GPU parity: libh2ldl.so against the reference's golden outputs and the oracle.

Every call goes through the C ABI (ctypes) into the sm_100a kernels.  The bar:
  * BK kernel: packed factor and ipiv bit-identical to the reference kernel;
  * engine: inertia counts identical to the reference engine's on the same
    exported H payloads, every golden shift (all are >= 10 eps ||A|| away from
    the spectrum), single-shift and shift-batched;
  * cfg1: bisection estimate of lambda_1024 identical to the reference's
    (eps_ev = 1e-8) and within eps_ev of LAPACK eigvalsh.
"""

import hashlib

import numpy as np
import pytest

from conftest import golden, instance_names
from paper_2311_08618_b200 import (
    InertiaUnstable,
    ShiftHitEigenvalue,
    build_tree,
    configs,
    construct,
    flat_structure,
    generalized_ldl,
    inertia,
    inertia_batch,
    matrix_kernel,
    multisection,
    slice_spectrum,
)
from paper_2311_08618_b200 import _native, dense, h2matrix
from paper_2311_08618_b200.geometry import PointCloud

pytestmark = pytest.mark.gpu


def test_native_library_is_the_cuda_build():
    lib = _native.load_library()
    assert b"sm_100a" in lib.h2l_version()


def test_bk_kernel_bit_identical_to_reference():
    z = golden("bk_random.npz")
    for t in range(int(z["count"])):
        A = np.ascontiguousarray(z[f"A_{t}"])
        F, ipiv, info = _native.bk_factor_device(A[None], [float(z[f"tol_{t}"])])
        ref = z[f"info_{t}"]
        assert info[0] == ref[0], t
        if info[0] == 0:
            assert np.array_equal(ipiv[0], z[f"ipiv_{t}"]), t
            cnt = _native.bk_inertia_device(F, ipiv, [0.0])[0]
            assert tuple(cnt) == tuple(ref[1:]), t
        assert hashlib.sha256(F[0].tobytes()).hexdigest() == str(z[f"Fsha_{t}"]), (t, A.shape)


def test_bk_kernel_batched_random():
    rng = np.random.default_rng(7)
    A = rng.standard_normal((12, 40, 40))
    A = A + A.transpose(0, 2, 1)
    tol = [dense.pivot_tolerance(a) for a in A]
    F, ipiv, info = _native.bk_factor_device(A, tol)
    assert not info.any()
    for q in range(12):
        w = np.linalg.eigvalsh(A[q])
        res = dense.ldl_symmetric(A[q])
        assert dense.inertia_of(res) == (int((w < 0).sum()), 0, int((w > 0).sum()))
        P = np.eye(40)[res.perm]
        assert np.abs(P.T @ res.L @ res.D @ res.L.T @ P - A[q]).max() < 1e-9 * np.abs(A[q]).max()


def test_dense_kats_on_device():
    res = dense.ldl_symmetric(np.array([[0.0, 2.0], [2.0, 0.0]]))
    assert res.block_sizes == [2] and dense.inertia_of(res) == (1, 0, 1)
    from paper_2311_08618_b200 import Breakdown

    with pytest.raises(Breakdown):
        dense.ldl_symmetric(np.diag([1.0, 0.0, -1.0]))


@pytest.mark.parametrize("name", instance_names())
def test_engine_counts_equal_reference(name):
    H = h2matrix.load_payload(f"tests/golden/h_{name}.npz")
    z = golden(f"counts_{name}.npz")
    mus = [float(m) for m in z["mus"]]
    want = [tuple(int(v) for v in c) for c in z["counts"]]
    # shift-batched: all shifts in one sweep
    got = [c.as_tuple() for c in inertia_batch(H, mus)]
    assert got == want, name
    # one shift per sweep (reference call pattern)
    for q in range(0, len(mus), 5):
        assert inertia(H, mus[q]).as_tuple() == want[q], (name, q)


@pytest.mark.parametrize("name", ["grid1d256_h2_e8", "mini_cfg3_1024", "circle256_hss_e8"])
def test_engine_structure_stats_match_reference(name):
    H = h2matrix.load_payload(f"tests/golden/h_{name}.npz")
    z = golden(f"counts_{name}.npz")
    for q in range(0, len(z["mus"]), 6):
        f = generalized_ldl(h2matrix.shift_diagonal(H, float(z["mus"][q])))
        fb, rc, ra, mf = (int(v) for v in z["stats"][q])
        assert f.stats["fill_blocks"] == fb, (name, q)
        assert f.stats["max_front"] == mf, (name, q)
        assert f.stats["recompressions"] == rc, (name, q)


def _diag_H(values):
    A = np.diag(np.asarray(values, dtype=float))
    cloud = PointCloud(np.arange(len(values), dtype=float).reshape(-1, 1))
    tree = build_tree(cloud, 32)
    return construct(matrix_kernel(A), tree, flat_structure(tree), 1e-9)


def test_root_only_and_retry_semantics():
    # reference test_gldl.py:20-28 and :104-124
    H = _diag_H(np.arange(1.0, 9.0))
    assert inertia(H, 3.5).as_tuple() == (3, 0, 5)
    assert inertia(H, 0.0).as_tuple() == (0, 0, 8)
    assert inertia(H, 100.0).as_tuple() == (8, 0, 0)
    assert inertia(H, 4.0).as_tuple() == (4, 0, 4)
    with pytest.raises(InertiaUnstable) as ei:
        inertia(H, 4.0, max_retries=0)
    assert isinstance(ei.value.__cause__, ShiftHitEigenvalue)


def test_flat_tree_with_levels():
    # BLR2 over a leveled tree: leaf elimination then flat merge to the root
    vals = np.linspace(-3.0, 5.0, 40)
    A = np.diag(vals)
    cloud = PointCloud(np.arange(40.0).reshape(-1, 1))
    tree = build_tree(cloud, 8)
    H = construct(matrix_kernel(A), tree, flat_structure(tree), 1e-9)
    for mu in (-3.5, -1.1, 0.05, 2.2, 5.5):
        assert inertia(H, mu).neg == int((vals < mu).sum())


@pytest.fixture(scope="module")
def cfg1():
    cloud, kern, tree, st = configs.config_problem("cfg1", seed=0)
    return construct(kern, tree, st, 1e-8), golden("cfg1.npz")


def test_cfg1_counts_along_reference_trace(cfg1):
    H, z = cfg1
    trace = z["trace"]
    got = inertia_batch(H, [float(r[0]) for r in trace])
    for row, c in zip(trace, got):
        assert c.as_tuple() == tuple(int(v) for v in row[1:]), row[0]


def test_cfg1_eigenvalue_bitwise_equals_reference(cfg1):
    H, z = cfg1
    iv = tuple(float(v) for v in z["interval"])
    val, hw, iters, evals = z["estimate"]
    est = slice_spectrum(H, 1024, iv, 1e-8)
    assert est.value == val and est.iterations == int(iters) and est.inertia_evals == int(evals)
    assert abs(est.value - z["eigs"][1023]) <= 1e-8
    (ms,) = multisection(H, [1024], iv, 1e-8, batch=63)
    assert ms.value == val and ms.iterations == int(iters)


def test_cfg1_multisection_many_eigenvalues(cfg1):
    H, z = cfg1
    iv = tuple(float(v) for v in z["interval"])
    ks = [1, 2, 512, 1023, 1024, 1025, 2047, 2048]
    ests = multisection(H, ks, iv, 1e-8, batch=128)
    w = z["eigs"]
    for e in ests:
        assert abs(e.value - w[e.k - 1]) <= 1e-8 + 1e-12 * abs(w[e.k - 1]), e.k


def test_cfg1_multisection_over_nccl_world1(cfg1):
    # the multi-GPU driver (NCCL all-gather of counts) on the one GPU of the box
    import os

    import torch
    import torch.distributed as dist

    from paper_2311_08618_b200.multigpu import multisection_distributed

    H, z = cfg1
    iv = tuple(float(v) for v in z["interval"])
    os.environ.setdefault("MASTER_ADDR", "127.0.0.1")
    os.environ.setdefault("MASTER_PORT", "29517")
    torch.cuda.set_device(0)
    dist.init_process_group("nccl", rank=0, world_size=1)
    try:
        ests, ev = multisection_distributed(H, [1024, 1], iv, 1e-8, per_rank=63)
    finally:
        dist.destroy_process_group()
    assert ests[0].value == float(z["estimate"][0])
    assert abs(ests[1].value - z["eigs"][0]) <= 1e-8
    assert ev.rounds > 0 and ev.world == 1


@pytest.mark.parametrize("name", instance_names()[:6])
def test_engine_elimination_flops_match_oracle(name):
    """The survey §8d flop count the bench's roofline and CPU-sample scaling use is
    the same number on the device engine and in the oracle (same H, same shift)."""
    from oracle import engine_ref
    from paper_2311_08618_b200.ldl import ldl_counts_array

    H = h2matrix.load_payload(f"tests/golden/h_{name}.npz")
    mu = float(golden(f"counts_{name}.npz")["mus"][0])
    _, _, st = ldl_counts_array(H, [mu])
    want = engine_ref.OracleEngine(H, mu, {}).run().elim_flops
    assert st["elim_flops"] == pytest.approx(want, rel=1e-12)


@pytest.mark.parametrize("n", [232, 300, 417, 520])
def test_cluster_bk_bit_identical_to_single_cta(n):
    """The cluster BK (fronts above one CTA's shared memory) replays the single-CTA
    kernel's arithmetic: factor, permutation, pivot blocks and counts bit-identical."""
    import ctypes

    lib = _native.load_testing_library()
    f = lib.h2l_internal_bk_engine
    f.restype = ctypes.c_int
    rng = np.random.default_rng(n)
    count = 3
    A = rng.standard_normal((count, n, n))
    A = A + A.transpose(0, 2, 1)
    A[1] += np.diag(np.linspace(-3, 3, n))
    A[2, :, : n // 3] *= 1e-3  # scale spread: more row-max tests and 2x2 pivots
    A[2, : n // 3, :] *= 1e-3
    outs = []
    for mode in (0, 1):
        a = np.ascontiguousarray(A.copy())
        perm = np.zeros((count, n), np.int32)
        dinfo = np.zeros((count, 3 * n))
        counts = np.zeros((count, 3), np.int64)
        status = np.zeros(count, np.int32)
        rc = f(0, mode, n, count, a.ctypes.data_as(ctypes.c_void_p), perm.ctypes.data_as(ctypes.c_void_p),
               dinfo.ctypes.data_as(ctypes.c_void_p), counts.ctypes.data_as(ctypes.c_void_p),
               status.ctypes.data_as(ctypes.c_void_p))
        assert rc == 0
        outs.append((np.tril(a), perm, dinfo, counts, status))
    for x, y in zip(*outs):
        assert np.array_equal(x, y)
    w = [np.linalg.eigvalsh(A[q]) for q in range(count)]
    assert [int(c[0]) for c in outs[1][3]] == [int(np.sum(v < 0)) for v in w]
    assert (outs[0][2][:, 2::3] == 2.0).any()  # 2x2 pivots were exercised


@pytest.mark.parametrize("n", [40, 186, 350, 500])
def test_gram_ordering_cluster_qr(n):
    """Recompression ordering (k_qr.cu): the cluster pivoted QR of a Gram matrix
    returns an orthogonal Q^T with Q^T M P upper triangular, the pivots of a
    column-pivoted QR (scipy/LAPACK dgeqp3 on the same M), and agrees with the
    single-CTA fallback kernel."""
    import ctypes

    import scipy.linalg

    lib = _native.load_testing_library()
    f = lib.h2l_internal_gram_order
    f.restype = ctypes.c_int
    rng = np.random.default_rng(n)
    count = 2
    G = rng.standard_normal((count, n, 3 * n)) * np.logspace(0, -6, n)[None, :, None]
    M = np.ascontiguousarray(G @ G.transpose(0, 2, 1))
    res = []
    for mode in (0, 1):
        qt = np.zeros((count, n, n))
        tau = np.zeros((count, n))
        piv = np.zeros((count, n), np.int32)
        rc = f(0, mode, n, count, M.ctypes.data_as(ctypes.c_void_p), qt.ctypes.data_as(ctypes.c_void_p),
               tau.ctypes.data_as(ctypes.c_void_p), piv.ctypes.data_as(ctypes.c_void_p))
        assert rc == 0
        res.append((qt, piv))
    for q in range(count):
        qt, piv = res[0][0][q], res[0][1][q]
        assert np.abs(qt @ qt.T - np.eye(n)).max() < 1e-12
        R = qt @ M[q][:, piv]
        assert np.abs(np.tril(R, -1)).max() <= 1e-10 * np.abs(R).max()
        _, _, P = scipy.linalg.qr(M[q], pivoting=True)
        k = min(n, 20)  # leading pivots: well separated norms
        assert np.array_equal(piv[:k], P[:k])
        assert np.array_equal(piv, res[1][1][q])
        assert np.abs(qt - res[1][0][q]).max() < 1e-10


@pytest.mark.parametrize("name", instance_names()[:8])
def test_low_degree_first_order_keeps_counts(name):
    """The optional low-degree-first elimination order (engine option elim_order=1,
    for fronts that do not fit in ascending order) changes fills and ranks but
    not the inertia: counts equal the reference's on every golden shift."""
    H = h2matrix.load_payload(f"tests/golden/h_{name}.npz")
    z = golden(f"counts_{name}.npz")
    eng = _native.engine_for(H)
    try:
        eng.set_option("elim_order", 1)
        counts, status, _ = eng.inertia(np.asarray(z["mus"], dtype=np.float64))
    finally:
        eng.set_option("elim_order", 0)
    assert not status.any()
    assert np.array_equal(counts, z["counts"])


@pytest.mark.parametrize("option", ["qr_budget", "block_cache", "block_classes", "schedule"])
def test_engine_options_keep_counts(option):
    """Performance options (budgeted Gram ordering, block free list, elimination
    schedule) never change the inertia: counts equal the reference's with the
    option off and on, on instances with recompression and merges."""
    names = [n for n in instance_names() if n.startswith("mini")] + ["circle256_h2_e8"]
    values = {"qr_budget": (0, 1), "block_cache": (0, 1, 2), "block_classes": (0, 1),
              "schedule": (0, 2, 1)}[option]
    for name in names:
        H = h2matrix.load_payload(f"tests/golden/h_{name}.npz")
        z = golden(f"counts_{name}.npz")
        eng = _native.engine_for(H)
        try:
            for v in values:
                eng.set_option(option, v)
                counts, status, st = eng.inertia(np.asarray(z["mus"], dtype=np.float64))
                assert not status.any(), (name, option, v)
                assert np.array_equal(counts, z["counts"]), (name, option, v)
        finally:
            eng.set_option(option, {"qr_budget": 1, "block_cache": 2, "block_classes": 1,
                                    "schedule": 1}[option])
