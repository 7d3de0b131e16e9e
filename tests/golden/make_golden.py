"""Generate the golden fixtures in tests/golden/ from the REFERENCE itself.

Run here (the build container) only: it copies /root/reference/pkg to a temp
dir, compiles its Cython kernel with the reference's own setup.py, imports the
reference package `h2slice` and records its outputs.  The GPU box never runs
this (it has no /root/reference); it only reads the committed .npz files.

    python tests/golden/make_golden.py            # all fixtures
    python tests/golden/make_golden.py bk cfg1    # a subset

Fixtures
  bk_random.npz    reference `_core._kernels.bk_factor` on random symmetric
                   matrices (test_backend.py:67-89 style) + test_dense KATs:
                   packed factor, ipiv, info, bk_inertia.
  sfc.npz          reference `sfc_order` permutations and `classify` output.
  h_<name>.npz     reference-constructed H payloads (save_payload format)
  counts_<name>.npz reference `gldl.inertia` counts + `generalized_ldl` stats
                   at seeded shifts, and LAPACK eigvalsh of reconstruct_dense.
  cfg1.npz         config 1: ordered points, block checksums of the reference
                   H, default_interval, slice_spectrum(k=1024, 1e-8) trace and
                   estimate, and eigvalsh of the dense matrix.
"""

import hashlib
import os
import shutil
import subprocess
import sys
import tempfile

import pin_host_fp  # noqa: F401  (before numpy: host-independent rounding, see its docstring)
import numpy as np  # noqa: E402

HERE = os.path.dirname(os.path.abspath(__file__))
REPO = os.path.dirname(os.path.dirname(HERE))
sys.path.insert(0, REPO)


def reference_path():
    """Build a private copy of the reference and return its src dir."""
    cache = os.path.join(tempfile.gettempdir(), "h2slice_ref_build")
    src = os.path.join(cache, "src")
    if not os.path.exists(os.path.join(cache, ".built")):
        shutil.rmtree(cache, ignore_errors=True)
        shutil.copytree("/root/reference/pkg", cache)
        subprocess.check_call([sys.executable, "setup.py", "build_ext", "--inplace"], cwd=cache,
                              stdout=subprocess.DEVNULL)
        open(os.path.join(cache, ".built"), "w").close()
    return src


sys.path.insert(0, reference_path())
import h2slice  # noqa: E402  (the reference)
from h2slice import _core  # noqa: E402
from h2slice.compress import construct, reconstruct_dense, shift_diagonal  # noqa: E402
from h2slice.geometry import generate_circle, generate_grid, laplace_kernel, sfc_order  # noqa: E402
from h2slice.gldl import generalized_ldl, inertia  # noqa: E402
from h2slice.partition import WEAK, build_tree, classify, flat_structure, strong  # noqa: E402
from h2slice.spectrum import InertiaCache, default_interval, slice_spectrum  # noqa: E402

assert _core.BACKEND == "compiled"

from paper_2311_08618_b200 import configs  # noqa: E402
from paper_2311_08618_b200.h2matrix import save_payload  # noqa: E402


def gen_bk():
    rng = np.random.default_rng(81)
    mats = []
    for _ in range(24):
        n = int(rng.integers(2, 48))
        A = rng.standard_normal((n, n))
        mats.append((A + A.T) / 2)
    rng = np.random.default_rng(101)
    for n in (64, 96, 128, 160, 200, 224, 256):
        A = rng.standard_normal((n, n))
        mats.append((A + A.T) / 2)
    # structured / indefinite cases that force 2x2 pivots and interchanges
    mats.append(np.array([[0.0, 2.0], [2.0, 0.0]]))
    mats.append(np.diag([3.0, -1.0, 0.5, -2.0, 7.0]))
    mats.append(np.diag([1.0, 1e-9, -1.0]))
    Z = np.zeros((40, 40))
    Z[np.arange(39), np.arange(1, 40)] = 1.0
    mats.append(Z + Z.T)
    mats.append(np.diag([1.0, 0.0, -1.0]))  # breakdown
    out = {}
    for t, A in enumerate(mats):
        A = np.ascontiguousarray(A)
        n = A.shape[0]
        F = A.copy()
        ipiv = np.zeros(n, dtype=np.int64)
        tol = 1e3 * np.finfo(np.float64).eps * float(np.max(np.abs(A)))
        info = _core.bk_factor(F, ipiv, tol)
        counts = _core.bk_inertia(F, ipiv, 0.0) if info == 0 else (-1, -1, -1)
        out[f"A_{t}"] = A
        if n <= 48:
            out[f"F_{t}"] = F
        out[f"Fsha_{t}"] = np.array(hashlib.sha256(F.tobytes()).hexdigest())
        out[f"ipiv_{t}"] = ipiv
        out[f"info_{t}"] = np.array([info, *counts], dtype=np.int64)
        out[f"tol_{t}"] = np.array(tol)
    out["count"] = np.array(len(mats))
    np.savez_compressed(os.path.join(HERE, "bk_random.npz"), **out)


def _ref_cloud(kind, n):
    if kind == "circle":
        c = generate_circle(n)
    else:
        c = generate_grid(n, int(kind[-2]))
    return c.permuted(sfc_order(c))


def gen_sfc():
    out = {}
    rng = np.random.default_rng(3)
    clouds = {
        "cube": rng.uniform(0, 1, (3000, 3)),
        "plane": rng.standard_normal((2000, 2)),
        "line": rng.standard_normal((500, 1)),
        "grid2d": generate_grid(12, 2).coords,
        "grid3d": generate_grid(6, 3).coords,
    }
    from h2slice.geometry import PointCloud

    for name, xyz in clouds.items():
        pc = PointCloud(xyz)
        out[f"pts_{name}"] = xyz
        out[f"perm_{name}"] = sfc_order(pc)
        ordered = pc.permuted(sfc_order(pc))
        for leaf in (8, 32):
            tree = build_tree(ordered, leaf)
            st = classify(tree, strong(1.0))
            out[f"dense_{name}_{leaf}"] = np.array(st.dense, dtype=np.int64).reshape(-1, 2)
            out[f"low_{name}_{leaf}"] = np.array(
                [(l, i, j) for l in sorted(st.lowrank) for i, j in st.lowrank[l]],
                dtype=np.int64).reshape(-1, 3)
            out[f"def_{name}_{leaf}"] = np.array(
                [(l, i, j) for l in sorted(st.deferred) for i, j in st.deferred[l]],
                dtype=np.int64).reshape(-1, 3)
    np.savez_compressed(os.path.join(HERE, "sfc.npz"), **out)


# (name, builder) -- instances of test_gldl.py:31-47 / test_acceptance.py:63-88
def _instances():
    inst = []
    for fmt in ("blr2", "hss", "h2"):
        for kind, n, leaf in (("circle", 256, 32), ("grid1d", 256, 32), ("grid3d", 6, 16)):
            for eps in (1e-8, 1e-6):
                inst.append((f"{kind}{n}_{fmt}_e{int(-np.log10(eps))}", kind, n, leaf, fmt, eps))
    inst.append(("grid2d10_h2_e7", "grid2d", 10, 8, "h2", 1e-7))
    return inst


def _ref_H(kind, n, leaf, fmt, eps):
    cloud = _ref_cloud(kind, n)
    tree = build_tree(cloud, leaf)
    st = {"blr2": lambda: flat_structure(tree), "hss": lambda: classify(tree, WEAK),
          "h2": lambda: classify(tree, strong(1.0))}[fmt]()
    return construct(laplace_kernel(cloud), tree, st, eps)


def _ref_config_H(name, n, leaf):
    """Mini-config H built by the REFERENCE construct on our seeded cloud/kernel."""
    cloud, kern, tree, st = configs.config_problem(name, seed=0, n=n, leaf=leaf)
    from h2slice.geometry import PointCloud
    from h2slice.partition import build_tree as rbuild, classify as rclassify

    rcloud = PointCloud(cloud.coords)
    rtree = rbuild(rcloud, leaf)
    rst = rclassify(rtree, strong(1.0))
    with pin_host_fp.single_thread():
        return construct(kern, rtree, rst, configs.CONFIGS[name].eps)


def _record(name, H, nshift=40, seed=0):
    A = reconstruct_dense(H, cap=8192)
    w = np.linalg.eigvalsh(A)
    span = w[-1] - w[0]
    nrm = max(abs(w[0]), abs(w[-1]))
    rng = np.random.default_rng(seed + 7)
    mus = []
    guard = 10 * H.eps * nrm
    while len(mus) < nshift:
        if len(mus) % 3 == 0:  # uniform over the padded spectrum hull
            mu = float(rng.uniform(w[0] - 0.1 * span, w[-1] + 0.1 * span))
        else:  # inside a random spectral gap: exercises every count 0..n
            i = int(rng.integers(0, len(w) - 1))
            mu = float(w[i] + (w[i + 1] - w[i]) * rng.uniform(0.25, 0.75))
        if np.min(np.abs(w - mu)) >= guard:
            mus.append(mu)
    counts, stats = [], []
    for mu in mus:
        c = inertia(H, mu)
        f = generalized_ldl(shift_diagonal(H, mu))
        counts.append(c.as_tuple())
        s = f.stats
        stats.append((s["fill_blocks"], s["recompressions"], s["rank_added"], s["max_front"]))
    save_payload(os.path.join(HERE, f"h_{name}.npz"), _as_ours(H))
    np.savez_compressed(os.path.join(HERE, f"counts_{name}.npz"), mus=np.array(mus),
                        counts=np.array(counts, dtype=np.int64),
                        stats=np.array(stats, dtype=np.int64), eigs=w,
                        scale0=np.array(H.scale_estimate()))
    print(name, "n", H.n, "fills", stats[0][0], "recomp", stats[0][1], "ok")


def _as_ours(H):
    """Re-wrap the reference H into our container so save_payload can write it."""
    from paper_2311_08618_b200.cluster import BlockStructure, ClusterTree
    from paper_2311_08618_b200.h2matrix import BasisSplit, RankStructuredMatrix

    t = H.tree
    tree = ClusterTree(n=t.n, leaf_size=t.leaf_size, depth=t.depth, degenerate=t.degenerate,
                       ranges=t.ranges, boxes=t.boxes)
    s = H.structure
    st = BlockStructure(kind=s.kind, eta=s.eta, lowrank=dict(s.lowrank), dense=list(s.dense),
                        deferred=dict(s.deferred))
    bases = {k: BasisSplit(U_S=b.U_S, U_R=b.U_R) for k, b in H.bases.items()}
    return RankStructuredMatrix(fmt=H.fmt, tree=tree, structure=st, eps=H.eps,
                                leaf_diag=H.leaf_diag, leaf_offdiag=H.leaf_offdiag,
                                bases=bases, couplings=H.couplings)


def gen_instances():
    for name, kind, n, leaf, fmt, eps in _instances():
        _record(name, _ref_H(kind, n, leaf, fmt, eps), nshift=24)
    # strong-admissibility mini-configs with real fill / recompression / merges
    _record("mini_cfg1_1024", _ref_config_H("cfg1", 1024, 16), nshift=24)
    _record("mini_cfg3_1024", _ref_config_H("cfg3", 1024, 32), nshift=24)


def gen_cfg1():
    cfg = configs.CONFIGS["cfg1"]
    cloud, kern, tree, st = configs.config_problem("cfg1", seed=0)
    from h2slice.geometry import PointCloud

    rtree = build_tree(PointCloud(cloud.coords), cfg.leaf)
    rst = classify(rtree, strong(1.0))
    H = construct(kern, rtree, rst, cfg.eps)
    iv = default_interval(H)
    A = reconstruct_dense(H)
    w = np.linalg.eigvalsh(A)
    trace = []
    real = h2slice.spectrum.inertia

    def traced(Hx, mu=0.0, max_retries=3):
        c = real(Hx, mu, max_retries)
        trace.append((mu, c.neg, c.zero, c.pos))
        return c

    h2slice.spectrum.inertia = traced
    try:
        est = slice_spectrum(H, 1024, iv, cfg.eps_ev, cache=InertiaCache())
    finally:
        h2slice.spectrum.inertia = real
    sums = np.array([H.leaf_diag[i].sum() for i in range(16)]
                    + [H.leaf_offdiag[k].sum() for k in rst.dense])
    np.savez_compressed(os.path.join(HERE, "cfg1.npz"), points=cloud.coords,
                        interval=np.array(iv), trace=np.array(trace),
                        estimate=np.array([est.value, est.half_width, est.iterations,
                                           est.inertia_evals]),
                        eigs=w, block_sums=sums, dense=np.array(rst.dense, dtype=np.int64),
                        max_rank=np.array(H.max_rank()))
    print("cfg1 interval", iv, "estimate", est.value, "err", est.value - w[1023],
          "evals", est.inertia_evals)


def gen_mini():
    _record("mini_cfg1_1024", _ref_config_H("cfg1", 1024, 16), nshift=24)


# ---------------------------------------------------------------- production-size
# Same-recipe instances at each config's REAL leaf size (n = 16384): fronts of
# 300-450 rows, rank growth by recompression, cluster BK, chunked panels and
# large Gram orderings.  The payload is too large to commit (0.5-2 GB), so the
# fixture stores a sha256 digest of the reference-built payload instead: the
# GPU test rebuilds H with this package's host `construct` (bit-identical to the
# reference's, checked against the digest) and factorizes THAT H on the device.
PROD = (
    # name, config, n, leaf, shifts, k for a reference slice_spectrum (0: none)
    ("prod_cfg2_16k", "cfg2", 16384, 256, 12, 0),
    ("prod_cfg3_16k", "cfg3", 16384, 256, 16, 8192),
    ("prod_cfg4_16k", "cfg4", 16384, 256, 12, 0),
    ("prod_cfg5_16k", "cfg5", 16384, 512, 16, 8192),
)


def gen_prod(only=()):
    import time

    from paper_2311_08618_b200.h2matrix import payload_digest

    for name, cfgname, n, leaf, nshift, k in PROD:
        if only and name not in only:
            continue
        t0 = time.perf_counter()
        cfg = configs.CONFIGS[cfgname]
        assert not pin_host_fp.check(), pin_host_fp.check()
        H = _ref_config_H(cfgname, n, leaf)
        t_con = time.perf_counter() - t0
        digest = payload_digest(H)
        A = reconstruct_dense(H, cap=n)
        w = np.linalg.eigvalsh(A)
        del A
        span = w[-1] - w[0]
        nrm = max(abs(w[0]), abs(w[-1]))
        rng = np.random.default_rng(11)
        guard = 10 * H.eps * nrm
        mus = []
        while len(mus) < nshift:
            if len(mus) % 3 == 0:
                mu = float(rng.uniform(w[0] - 0.05 * span, w[-1] + 0.05 * span))
            else:
                i = int(rng.integers(0, len(w) - 1))
                mu = float(w[i] + (w[i + 1] - w[i]) * rng.uniform(0.25, 0.75))
            if np.min(np.abs(w - mu)) >= guard:
                mus.append(mu)
        counts, stats, secs = [], [], []
        for mu in mus:
            t1 = time.perf_counter()
            f = generalized_ldl(shift_diagonal(H, mu))
            secs.append(time.perf_counter() - t1)
            c = f.inertia_counts
            assert c.zero == 0, (name, mu)
            counts.append((c.neg, c.zero, c.pos))
            s = f.stats
            stats.append((s["fill_blocks"], s["recompressions"], s["rank_added"], s["max_front"]))
            print(name, f"mu={mu:.6g}", counts[-1], stats[-1], f"{secs[-1]:.1f}s", flush=True)
        extra = {}
        if k:
            iv = (float(w[0]) - 1.0, float(w[-1]) + 1.0)
            t1 = time.perf_counter()
            est = slice_spectrum(H, k, iv, cfg.eps_ev, cache=InertiaCache())
            extra = dict(est_k=np.array(k), est_interval=np.array(iv),
                         estimate=np.array([est.value, est.half_width, est.iterations,
                                            est.inertia_evals]),
                         est_seconds=np.array(time.perf_counter() - t1))
            print(name, "slice_spectrum k", k, est.value, "eigvalsh", w[k - 1],
                  "iters", est.iterations, flush=True)
        np.savez_compressed(os.path.join(HERE, f"{name}.npz"), config=np.array(cfgname),
                            n=np.array(n), leaf=np.array(leaf), digest=np.array(digest),
                            scale0=np.array(H.scale_estimate()), mus=np.array(mus),
                            counts=np.array(counts, dtype=np.int64),
                            stats=np.array(stats, dtype=np.int64), eigs=w,
                            ref_seconds=np.array(secs), construct_seconds=np.array(t_con),
                            **extra)
        print(name, "done: construct", f"{t_con:.1f}s", "digest", digest[:16], flush=True)


if __name__ == "__main__":
    which = set(sys.argv[1:]) or {"bk", "sfc", "inst", "cfg1"}
    if "mini" in which:
        gen_mini()
    prod = {w for w in which if w.startswith("prod")}
    if prod:
        gen_prod(() if "prod" in prod else tuple(prod))
    if "bk" in which:
        gen_bk()
    if "sfc" in which:
        gen_sfc()
    if "inst" in which:
        gen_instances()
    if "cfg1" in which:
        gen_cfg1()
