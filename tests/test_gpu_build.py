"""GPU: device-side H2 construction.

Bar (reference test_compress.py:20-27): reconstruction error <= 50 eps ||A||;
and parity on the identical H: the CUDA engine's counts on the device-built
matrix equal the oracle's counts on its host export and LAPACK's counts.
"""

import numpy as np
import pytest

from oracle import engine_ref
from paper_2311_08618_b200 import (
    WEAK,
    build_tree,
    classify,
    flat_structure,
    generate_circle,
    generate_grid,
    inertia_batch,
    laplace_kernel,
    sfc_order,
    strong,
)
from paper_2311_08618_b200 import configs, gpu_build, h2matrix

pytestmark = pytest.mark.gpu


def _cloud(kind, n):
    c = generate_circle(n) if kind == "circle" else generate_grid(n, int(kind[-2]))
    return c.permuted(sfc_order(c))


CASES = [("circle", 256, 32, "hss"), ("circle", 256, 32, "h2"), ("grid1d", 256, 32, "h2"),
         ("grid3d", 6, 16, "h2"), ("grid2d", 12, 16, "blr2")]


@pytest.mark.parametrize("kind,n,leaf,fmt", CASES)
def test_device_construction_accuracy_and_parity(kind, n, leaf, fmt):
    eps = 1e-8
    cloud = _cloud(kind, n)
    tree = build_tree(cloud, leaf)
    st = {"hss": lambda: classify(tree, WEAK), "h2": lambda: classify(tree, strong(1.0)),
          "blr2": lambda: flat_structure(tree)}[fmt]()
    kern = laplace_kernel(cloud)
    Hd = gpu_build.construct_device(kern, tree, st, eps)
    Hh = gpu_build.to_host(Hd)
    N = cloud.n
    A = kern.block(np.arange(N), np.arange(N))
    R = h2matrix.reconstruct_dense(Hh)
    assert np.linalg.norm(R - A, 2) <= 50 * eps * np.linalg.norm(A, 2)
    for bs in Hh.bases.values():
        Q = bs.square()
        if Q.size:
            assert np.abs(Q.T @ Q - np.eye(Q.shape[0])).max() < 1e-12
    w = np.linalg.eigvalsh(R)
    rng = np.random.default_rng(3)
    mus = []
    while len(mus) < 12:
        i = int(rng.integers(0, N - 1))
        mu = float(w[i] + (w[i + 1] - w[i]) * rng.uniform(0.25, 0.75))
        if np.min(np.abs(w - mu)) > 10 * eps * np.abs(w).max():
            mus.append(mu)
    got = [c.as_tuple() for c in inertia_batch(Hd, mus)]
    cache = {}
    want = [engine_ref.inertia(Hh, mu, skel_cache=cache) for mu in mus]
    assert got == want
    assert [g[0] for g in got] == [int(np.sum(w < mu)) for mu in mus]


def test_mini_config3_device_build():
    Hd, cloud = gpu_build.config_device("cfg3", n=2048, leaf=64)
    Hh = gpu_build.to_host(Hd)
    R = h2matrix.reconstruct_dense(Hh)
    kern = configs.config_kernel("cfg3", cloud)
    A = kern.block(np.arange(2048), np.arange(2048))
    assert np.linalg.norm(R - A, 2) <= 50 * 1e-8 * np.linalg.norm(A, 2)
    w = np.linalg.eigvalsh(R)
    mus = [float(0.5 * (w[k] + w[k + 1])) for k in (10, 700, 1023, 1500, 2040)]
    got = [c.neg for c in inertia_batch(Hd, mus)]
    assert got == [11, 701, 1024, 1501, 2041]


def test_gershgorin_device_and_arena_export():
    Hd, cloud = gpu_build.config_device("cfg1", n=1024, leaf=64)
    kern = Hd._kernel
    A = kern.block(np.arange(cloud.n), np.arange(cloud.n))
    lo, hi = h2matrix.gershgorin_interval(A)
    glo, ghi = gpu_build.gershgorin_device(kern, rows=300, pad=0.0)
    assert glo == pytest.approx(lo, rel=1e-12) and ghi == pytest.approx(hi, rel=1e-12)
    plo, phi = gpu_build.gershgorin_device(kern)
    assert plo < lo and phi > hi
    Hh = gpu_build.to_host(Hd)
    for k, v in Hd.leaf_offdiag.items():
        assert np.array_equal(Hh.leaf_offdiag[k], v.cpu().numpy())
    for k, b in Hd.bases.items():
        assert np.array_equal(Hh.bases[k].square(), b.square().cpu().numpy())
