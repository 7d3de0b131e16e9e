"""Counts and launch statistics of the three elimination schedules on the golden instances."""
import glob
import os
import sys
import time

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import numpy as np  # noqa: E402

from paper_2311_08618_b200 import _native, h2matrix  # noqa: E402
from paper_2311_08618_b200.ldl import ldl_counts_array  # noqa: E402

bad = 0
for path in sorted(glob.glob(os.path.join(ROOT, "tests/golden/h_*.npz"))):
    name = os.path.basename(path)[2:-4]
    H = h2matrix.load_payload(path)
    z = np.load(os.path.join(ROOT, f"tests/golden/counts_{name}.npz"))
    mus = [float(m) for m in z["mus"]]
    want = z["counts"]
    eng = _native.engine_for(H, 0)
    row = [name]
    for sched in (0, 1, 2):
        eng.set_option("schedule", sched)
        t0 = time.perf_counter()
        counts, status, st = ldl_counts_array(H, mus)
        dt = time.perf_counter() - t0
        ok = np.array_equal(counts, want) and not status.any()
        bad += not ok
        row.append(f"s{sched}:{'ok' if ok else 'BAD'} g={st['groups']} L={st['launches']} "
                   f"ra={st['rank_added']} {dt * 1e3:.0f}ms")
    print(" | ".join(row), flush=True)
print("BAD", bad)
