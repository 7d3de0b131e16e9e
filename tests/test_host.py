"""CPU: host logic, the C-ABI library surface and the plan exporter (no GPU calls)."""

import ctypes
import os
import re

import numpy as np
import pytest

from conftest import ROOT
from paper_2311_08618_b200 import (
    ConfigError,
    EigenvalueEstimate,
    InertiaCache,
    NativeError,
    build_tree,
    classify,
    construct,
    flat_structure,
    generate_grid,
    laplace_kernel,
    sfc_order,
    strong,
)
from paper_2311_08618_b200 import _native, bisection, h2matrix
from paper_2311_08618_b200.geometry import PointCloud


def _header_functions():
    text = open(os.path.join(ROOT, "include", "h2ldl.h")).read()
    return sorted(set(re.findall(r"^\s*(?:int|const char \*)\s*(h2l_\w+)\s*\(", text, re.M)))


def test_library_exports_every_header_symbol():
    lib = _native.load_library()
    names = _header_functions()
    assert {"h2l_create", "h2l_inertia", "h2l_upload", "h2l_bk_factor"} <= set(names)
    for name in names:
        assert hasattr(lib, name), name
    assert set(names) == set(_native.SYMBOLS)
    assert b"sm_100a" in lib.h2l_version()


def test_library_is_sm100a_cubin():
    # the shared object must carry sm_100a SASS (no PTX-JIT fallback path)
    import subprocess

    out = subprocess.run(["cuobjdump", "--list-elf", _native.LIB_PATH], capture_output=True,
                         text=True)
    assert out.returncode == 0 and "sm_100a" in out.stdout


def _c_layout(struct, fields, tmpdir):
    import subprocess

    src = os.path.join(tmpdir, "lay.c")
    body = "".join(f'printf("{f} %zu\\n", offsetof({struct}, {f}));' for f in fields)
    with open(src, "w") as fh:
        fh.write('#include <stdio.h>\n#include <stddef.h>\n#include "h2ldl.h"\n'
                 f'int main(void){{printf("sizeof %zu\\n", sizeof({struct}));{body}return 0;}}\n')
    exe = os.path.join(tmpdir, "lay")
    subprocess.check_call(["gcc", "-I", os.path.join(ROOT, "include"), src, "-o", exe])
    out = subprocess.run([exe], capture_output=True, text=True, check=True).stdout.split()
    return {out[i]: int(out[i + 1]) for i in range(0, len(out), 2)}


@pytest.mark.parametrize("struct,cls", [("h2l_plan", _native.Plan), ("h2l_stats", _native.Stats)])
def test_ctypes_structs_match_c_header(struct, cls, tmp_path):
    names = [f for f, _ in cls._fields_]
    lay = _c_layout(struct, names, str(tmp_path))
    assert lay["sizeof"] == ctypes.sizeof(cls)
    for f in names:
        assert lay[f] == getattr(cls, f).offset, f


def test_build_plan_offsets_cover_arena():
    H = h2matrix.load_payload(os.path.join(ROOT, "tests", "golden", "h_grid1d256_h2_e8.npz"))
    plan, keep = _native.build_plan(H)
    ranges, dense, lowrank, deferred, brank, bdim, boff, diag_off, dense_off, low_off, arena = keep
    assert plan.n == 256 and plan.depth == H.tree.depth
    assert plan.arena_len == arena.size
    L = H.tree.depth
    for i, off in enumerate(diag_off):
        m = H.tree.size(L, i)
        assert np.array_equal(arena[off:off + m * m].reshape(m, m), H.leaf_diag[i])
    for (l, i, j), off in zip(lowrank, low_off):
        C = H.couplings[(l, i, j)]
        assert np.array_equal(arena[off:off + C.size].reshape(C.shape), C)
    for (l, i), bs in H.bases.items():
        nd = (1 << l) - 1 + i
        assert brank[nd] == bs.rank and bdim[nd] == bs.m
        if bs.m:
            Q = arena[boff[nd]:boff[nd] + bs.m * bs.m].reshape(bs.m, bs.m)
            assert np.array_equal(Q, bs.square())


def test_payload_roundtrip():
    H = h2matrix.load_payload(os.path.join(ROOT, "tests", "golden", "h_circle256_hss_e8.npz"))
    tmp = os.path.join(ROOT, "tests", "_tmp_payload.npz")
    try:
        h2matrix.save_payload(tmp, H)
        H2 = h2matrix.load_payload(tmp)
    finally:
        if os.path.exists(tmp):
            os.remove(tmp)
    A1, A2 = h2matrix.reconstruct_dense(H), h2matrix.reconstruct_dense(H2)
    assert np.array_equal(A1, A2)


def test_no_gpu_entry_points_fail_loudly():
    # without a usable device every compute entry point raises (no CPU fallback)
    import torch

    if torch.cuda.is_available():
        pytest.skip("a GPU is present")
    with pytest.raises(NativeError):
        _native.DeviceEngine(0)
    with pytest.raises(NativeError):
        _native.bk_factor_device(np.eye(4)[None], [1e-12])


def test_construct_matches_reference_accuracy_bar():
    # reference test_compress.py:20-27: reconstruction error < 50 eps
    cloud = generate_grid(160, 1)
    cloud = cloud.permuted(sfc_order(cloud))
    tree = build_tree(cloud, 16)
    A = laplace_kernel(cloud).block(np.arange(160), np.arange(160))
    for st in (flat_structure(tree), classify(tree, strong(1.0))):
        H = construct(laplace_kernel(cloud), tree, st, 1e-7)
        err = np.linalg.norm(h2matrix.reconstruct_dense(H) - A, 2) / np.linalg.norm(A, 2)
        assert err < 50 * 1e-7


def test_shift_diagonal_shares_payload():
    H = h2matrix.load_payload(os.path.join(ROOT, "tests", "golden", "h_circle256_hss_e8.npz"))
    S = h2matrix.shift_diagonal(H, 3.0)
    T = h2matrix.shift_diagonal(S, -1.0)
    assert S.origin() is H and T.origin() is H
    assert T.shift == 2.0 and T.leaf_diag is H.leaf_diag
    A = h2matrix.reconstruct_dense(H)
    assert np.array_equal(h2matrix.reconstruct_dense(T), A - 2.0 * np.eye(H.n))


def test_inertia_cache_semantics():
    # reference test_spectrum.py:124-140
    c = InertiaCache()
    c.insert(5.0, 10)
    c.insert(2.0, 3)
    assert c.le(1.5) is None and c.le(3.0) == 3 and c.le(2.0) == 3
    assert c.ge(3.0) == 10 and c.ge(5.0) == 10 and c.ge(6.0) is None
    assert c.exact(5.0) == 10 and c.exact(3.3) is None and len(c) == 2
    c.insert(5.0, 99)
    assert c.exact(5.0) == 10
    assert c.resolve(6.0, 10) is True and c.resolve(1.0, 4) is False and c.resolve(2.5, 4) is None
    assert c.resolve(1.0, 3) is None and c.resolve(4.0, 11) is False


def test_estimate_json_roundtrip():
    est = EigenvalueEstimate(k=7, value=1.25, half_width=5e-6, iterations=21, inertia_evals=17,
                             wall_time=0.125)
    assert EigenvalueEstimate.from_json(est.to_json()) == est


def test_multisection_argument_validation():
    class H:
        n = 8

    with pytest.raises(ConfigError):
        bisection.multisection(H, [0], (0.0, 1.0), 1e-3, evaluate=lambda m: [0] * len(m))
    with pytest.raises(ConfigError):
        bisection.multisection(H, [1], (1.0, 1.0), 1e-3, evaluate=lambda m: [0] * len(m))
    with pytest.raises(ConfigError):
        bisection.multisection(H, [1], (0.0, 1.0), 0.0, evaluate=lambda m: [0] * len(m))


def test_multisection_not_in_interval():
    from paper_2311_08618_b200 import NotInInterval

    vals = np.linspace(1.0, 16.0, 16)

    class H:
        n = 16

    # a shift exactly on an eigenvalue is retried slightly above it (gldl.py:621-632)
    ev = lambda mus: [int(np.sum(vals <= m)) for m in mus]  # noqa: E731
    with pytest.raises(NotInInterval):
        bisection.multisection(H, [1], (2.5, 20.0), 1e-6, evaluate=ev)
    with pytest.raises(NotInInterval):
        bisection.multisection(H, [16], (0.0, 10.0), 1e-6, evaluate=ev)
    (e,) = bisection.multisection(H, [16], (0.0, 16.0), 1e-6, evaluate=ev)
    assert abs(e.value - 16.0) < 5e-7


def test_multisection_matches_oracle_bisection():
    # host driver over the oracle evaluator == the oracle's sequential bisection
    from oracle import engine_ref

    H = h2matrix.load_payload(os.path.join(ROOT, "tests", "golden", "h_grid1d256_h2_e8.npz"))
    z = np.load(os.path.join(ROOT, "tests", "golden", "counts_grid1d256_h2_e8.npz"))
    w = z["eigs"]
    iv = (float(w[0] - 1.0), float(w[-1] + 1.0))
    cache = {}
    ev = lambda mus: [engine_ref.inertia(H, m, skel_cache=cache)[0] for m in mus]  # noqa: E731
    ests = bisection.multisection(H, [5, 128], iv, 1e-6, batch=15, evaluate=ev)
    for e in ests:
        val, hw, it, _, _ = engine_ref.slice_spectrum(H, e.k, iv, 1e-6, skel_cache=cache)
        assert e.value == val and e.iterations == it
        assert abs(e.value - w[e.k - 1]) < 1e-6
