import os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np
from bench import build_cfg1, cfg1_interval, shifts_for
from paper_2311_08618_b200 import _native
from paper_2311_08618_b200.ldl import ldl_counts_array
S, MB, C = (int(v) for v in sys.argv[1:4])
H = build_cfg1()
(lo, hi), eigs = cfg1_interval()
eng = _native.engine_for(H, 0)
eng.set_option("max_batch", MB)
eng.set_option("concurrency", C)
for k in range(int(os.environ.get("IT", "4"))):
    mus = shifts_for(lo, hi, S, 100 + k, 0) if not os.environ.get('NARROW') else np.sort(np.random.default_rng(k).uniform(-20, 20, S))
    c, st, stats = ldl_counts_array(H, mus)
    want = np.searchsorted(eigs, mus)
    bad = np.nonzero(c[:, 0] != want)[0]
    print(k, "bad", len(bad), "got", c[bad, 0].tolist(), "want", want[bad].tolist(), "first", bad[:10].tolist(), "waves", sorted(set((bad // MB).tolist())), "status", st.sum(),
          "sum", (c.sum(axis=1) != 2048).sum())
