"""GPU: level-batched elimination schedules, per-shift truncation, device-side
counts and the one-process multi-GPU entry point.

  * schedule 1 (wavefronts of the ascending order's dependency DAG) factors
    exactly what the reference's ascending sweep factors: with the full
    recompression ordering (qr_budget 0) counts AND structural statistics
    (fills, recompressions, rank added, max front, dropped norm) are identical
    to schedule 0, bit for bit;
  * schedule 2 (colour classes) re-orders the elimination: counts still equal
    the reference's on every golden shift (gldl.py:259-266 order-free inertia);
  * a shift-batched wave returns, for every shift, the count a single-shift
    call returns (each shift drops the fill directions its own rank drops,
    gldl.py:296-347), on an instance whose ranks differ across shifts;
  * h2l_inertia_device writes the packed rows into device memory;
  * h2l_comm_init / h2l_inertia_multi over the box's GPU(s) (NCCL all-gather
    between engine buffers) returns the single-engine counts.
"""

import numpy as np
import pytest

from conftest import golden, instance_names
from paper_2311_08618_b200 import _native, h2matrix, inertia, inertia_batch
from paper_2311_08618_b200.ldl import ldl_counts_array

pytestmark = pytest.mark.gpu


def _load(name):
    return h2matrix.load_payload(f"tests/golden/h_{name}.npz"), golden(f"counts_{name}.npz")


@pytest.mark.parametrize("name", instance_names())
def test_schedules_keep_reference_counts(name):
    H, z = _load(name)
    eng = _native.engine_for(H)
    mus = np.asarray(z["mus"], dtype=np.float64)
    try:
        for sched in (0, 1, 2):
            eng.set_option("schedule", sched)
            counts, status, _ = eng.inertia(mus)
            assert not status.any(), (name, sched)
            assert np.array_equal(counts, z["counts"]), (name, sched)
    finally:
        eng.set_option("schedule", 1)


@pytest.mark.parametrize("name", ["mini_cfg3_1024", "mini_cfg1_1024", "grid1d256_h2_e8",
                                  "circle256_hss_e8"])
def test_wavefront_schedule_is_the_ascending_sweep(name):
    H, z = _load(name)
    eng = _native.engine_for(H)
    mus = np.asarray(z["mus"], dtype=np.float64)
    out = {}
    try:
        eng.set_option("qr_budget", 0)
        for sched in (0, 1):
            eng.set_option("schedule", sched)
            out[sched] = eng.inertia(mus)
    finally:
        eng.set_option("qr_budget", 1)
        eng.set_option("schedule", 1)
    (c0, s0, st0), (c1, s1, st1) = out[0], out[1]
    assert np.array_equal(c0, c1) and np.array_equal(s0, s1)
    for key in ("fill_blocks", "recompressions", "rank_added", "max_front", "dropped_fro",
                "elim_flops"):
        assert st0[key] == st1[key], (name, key, st0[key], st1[key])
    assert st1["groups"] <= st0["groups"]


def test_colour_schedule_batches_clusters():
    H, z = _load("mini_cfg3_1024")
    eng = _native.engine_for(H)
    mus = np.asarray(z["mus"][:8], dtype=np.float64)
    try:
        eng.set_option("schedule", 0)
        _, _, st0 = eng.inertia(mus)
        eng.set_option("schedule", 2)
        _, _, st2 = eng.inertia(mus)
    finally:
        eng.set_option("schedule", 1)
    assert st2["groups"] < st0["groups"]
    assert st2["launches"] < st0["launches"]


@pytest.mark.parametrize("name", ["mini_cfg3_1024", "grid1d256_h2_e8", "circle256_h2_e6"])
def test_batched_wave_equals_single_shift_calls(name):
    """the wave keeps t = max rank over its shifts; each shift still drops
    the directions its own rank drops, so its count does not depend on the wave."""
    H, z = _load(name)
    mus = [float(m) for m in z["mus"]]
    batched = [c.as_tuple() for c in inertia_batch(H, mus)]
    single = [inertia(H, mu).as_tuple() for mu in mus]
    assert batched == single
    assert batched == [tuple(int(v) for v in c) for c in z["counts"]]
    # the instance does exercise different ranks across the wave's shifts
    ranks = [ldl_counts_array(H, [mu])[2]["rank_added"] for mu in mus[:8]]
    assert len(set(ranks)) > 1, ranks


def test_inertia_device_rows():
    import torch

    H, z = _load("mini_cfg3_1024")
    mus = np.asarray(z["mus"], dtype=np.float64)
    eng = _native.engine_for(H, 0)
    out = torch.full((len(mus), 4), -7, dtype=torch.int64, device="cuda:0")
    st = eng.inertia_device(mus, out)
    rows = out.cpu().numpy()
    assert np.array_equal(rows[:, :3], z["counts"])
    assert not rows[:, 3].any()
    assert st["launches"] > 0


def test_inertia_multi_matches_single_engine():
    import torch

    H, z = _load("mini_cfg3_1024")
    mus = np.asarray(z["mus"], dtype=np.float64)
    devs = list(range(torch.cuda.device_count()))
    multi = _native.MultiEngine(H, devs)
    counts, status, st = multi.inertia(mus)
    assert np.array_equal(counts, z["counts"])
    assert not status.any()
    # an uneven split (more ranks than some slices) and a single shift
    c1, s1, _ = multi.inertia(mus[:1])
    assert np.array_equal(c1, z["counts"][:1])
