"""CPU: pin the oracle (oracle/) and the host-side mirror against the REFERENCE.

Golden fixtures in tests/golden/ were produced by the reference package itself
(tests/golden/make_golden.py): its compiled `_core.bk_factor`, its `sfc_order`
/ `classify`, its `construct`, and its `gldl.inertia` counts on exported H
payloads.  These tests prove that the oracle reproduces the reference
exactly before the oracle is used to check the CUDA engine.
"""

import hashlib

import numpy as np
import pytest

from conftest import golden, instance_names
from oracle import dense_ref, engine_ref
from paper_2311_08618_b200 import cluster, configs, geometry, h2matrix


def _bk_cases():
    z = golden("bk_random.npz")
    return [(t, z) for t in range(int(z["count"]))]


def test_bk_oracle_bit_identical_to_reference():
    z = golden("bk_random.npz")
    for t in range(int(z["count"])):
        A = np.ascontiguousarray(z[f"A_{t}"])
        F = A.copy()
        ipiv = np.zeros(A.shape[0], dtype=np.int64)
        info = dense_ref.bk_factor(F, ipiv, float(z[f"tol_{t}"]))
        ref = z[f"info_{t}"]
        assert info == ref[0], t
        if info == 0:
            assert np.array_equal(ipiv, z[f"ipiv_{t}"]), t
            assert dense_ref.bk_inertia(F, ipiv, 0.0) == tuple(ref[1:]), t
        assert hashlib.sha256(F.tobytes()).hexdigest() == str(z[f"Fsha_{t}"]), t
        if f"F_{t}" in z.files:
            assert np.array_equal(F, z[f"F_{t}"]), t


def test_oracle_ldl_kats():
    # reference test_dense.py:22-58
    res = dense_ref.ldl_symmetric(np.array([[0.0, 2.0], [2.0, 0.0]]))
    assert res.sizes == [2] and dense_ref.inertia_of(res) == (1, 0, 1)
    assert dense_ref.inertia_of(dense_ref.ldl_symmetric(np.diag([3.0, -1, .5, -2, 7]))) == (2, 0, 3)
    with pytest.raises(dense_ref.Breakdown):
        dense_ref.ldl_symmetric(np.diag([1.0, 0.0, -1.0]))
    res = dense_ref.ldl_symmetric(np.diag([1.0, 1e-9, -1.0]))
    assert dense_ref.inertia_of(res, zero_tol=1e-6) == (1, 1, 1)
    assert dense_ref.inertia_of(res, zero_tol=1e-12) == (1, 0, 2)


def test_morton_order_and_classification_match_reference():
    z = golden("sfc.npz")
    for name in ("cube", "plane", "line", "grid2d", "grid3d"):
        pc = geometry.PointCloud(z[f"pts_{name}"])
        perm = geometry.sfc_order(pc)
        assert np.array_equal(perm, z[f"perm_{name}"]), name
        ordered = pc.permuted(perm)
        for leaf in (8, 32):
            tree = cluster.build_tree(ordered, leaf)
            st = cluster.classify(tree, cluster.strong(1.0))
            assert np.array_equal(np.array(st.dense, dtype=np.int64).reshape(-1, 2),
                                  z[f"dense_{name}_{leaf}"]), (name, leaf)
            low = [(l, i, j) for l in sorted(st.lowrank) for i, j in st.lowrank[l]]
            assert np.array_equal(np.array(low, dtype=np.int64).reshape(-1, 3),
                                  z[f"low_{name}_{leaf}"]), (name, leaf)
            dfr = [(l, i, j) for l in sorted(st.deferred) for i, j in st.deferred[l]]
            assert np.array_equal(np.array(dfr, dtype=np.int64).reshape(-1, 3),
                                  z[f"def_{name}_{leaf}"]), (name, leaf)


SMALL = [n for n in instance_names() if not n.startswith("mini")]


@pytest.mark.parametrize("name", SMALL)
def test_oracle_engine_matches_reference_counts(name):
    H = h2matrix.load_payload(f"tests/golden/h_{name}.npz")
    z = golden(f"counts_{name}.npz")
    cache = {}
    for q, mu in enumerate(z["mus"]):
        got = engine_ref.inertia(H, float(mu), skel_cache=cache)
        assert got == tuple(z["counts"][q]), (name, q, mu)
        c, stats = engine_ref.generalized_ldl(h2matrix.shift_diagonal(H, float(mu)),
                                              skel_cache=cache)
        want = z["stats"][q]
        got_stats = (stats["fill_blocks"], stats["recompressions"], stats["rank_added"],
                     stats["max_front"])
        assert got_stats == tuple(want), (name, q)


@pytest.mark.parametrize("name", [n for n in instance_names() if n.startswith("mini")])
def test_oracle_engine_mini_configs(name):
    H = h2matrix.load_payload(f"tests/golden/h_{name}.npz")
    z = golden(f"counts_{name}.npz")
    cache = {}
    for q in range(0, len(z["mus"]), 4):  # every 4th shift keeps the CPU suite short
        mu = float(z["mus"][q])
        assert engine_ref.inertia(H, mu, skel_cache=cache) == tuple(z["counts"][q]), (name, q)


def test_counts_equal_lapack_on_instances():
    # the reference's own bar (test_gldl.py:31-47): counts == eigvalsh counts
    for name in SMALL:
        z = golden(f"counts_{name}.npz")
        w = z["eigs"]
        for mu, c in zip(z["mus"], z["counts"]):
            assert c[0] == int(np.sum(w < mu)) and c[1] == 0, name


def test_cfg1_construction_bitwise_equals_reference():
    z = golden("cfg1.npz")
    cloud, kern, tree, st = configs.config_problem("cfg1", seed=0)
    assert np.array_equal(cloud.coords, z["points"])
    assert np.array_equal(np.array(st.dense, dtype=np.int64), z["dense"])
    H = h2matrix.construct(kern, tree, st, 1e-8)
    assert H.max_rank() == int(z["max_rank"]) == 0
    sums = np.array([H.leaf_diag[i].sum() for i in range(16)]
                    + [H.leaf_offdiag[k].sum() for k in st.dense])
    assert np.array_equal(sums, z["block_sums"])


def test_cfg1_oracle_replays_reference_trace():
    z = golden("cfg1.npz")
    cloud, kern, tree, st = configs.config_problem("cfg1", seed=0)
    H = h2matrix.construct(kern, tree, st, 1e-8)
    trace = z["trace"]
    cache = {}
    for row in trace[[0, 7, 19, 39]]:
        mu = float(row[0])
        assert engine_ref.inertia(H, mu, skel_cache=cache) == tuple(int(v) for v in row[1:])


def test_oracle_deadline_sample_counts_elimination_flops():
    """bench.py's bounded CPU sample: a deadline stops the run after whole clusters
    and reports the elimination flops done so far (a prefix of the full count)."""
    name = SMALL[0]
    H = h2matrix.load_payload(f"tests/golden/h_{name}.npz")
    mu = float(golden(f"counts_{name}.npz")["mus"][0])
    cache = {}
    full = engine_ref.OracleEngine(H, mu, cache).run()
    assert full.elim_flops > 0
    with pytest.raises(engine_ref.Deadline) as ex:
        engine_ref.OracleEngine(H, mu, cache, deadline_s=0.0).run()
    d = ex.value
    assert d.clusters == 1 and 0 < d.elim_flops <= full.elim_flops
