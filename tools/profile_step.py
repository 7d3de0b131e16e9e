"""Run a few cfg1 shift-batched sweeps (for ncu launch lists / captures)."""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np  # noqa: E402

from bench import build_cfg1, cfg1_interval, shifts_for  # noqa: E402
from paper_2311_08618_b200 import _native  # noqa: E402
from paper_2311_08618_b200.ldl import ldl_counts_array  # noqa: E402

S = int(os.environ.get("S", "64"))
STEPS = int(os.environ.get("STEPS", "2"))
H = build_cfg1()
(lo, hi), eigs = cfg1_interval()
eng = _native.engine_for(H, 0)
eng.set_option("max_batch", int(os.environ.get("MB", S)))
eng.set_option("concurrency", int(os.environ.get("C", "2")))
for k in range(STEPS):
    mus = shifts_for(lo, hi, S, 100 + k, 0)
    c, st, stats = ldl_counts_array(H, mus)
    assert np.array_equal(c[:, 0], np.searchsorted(eigs, mus)) and not st.any()
    print(f"step {k}: {stats['ms_total']:.2f} ms, launches {stats['launches']}")
