"""One shift-batched sweep of a config-2-recipe instance (n = 16384, leaf 256, host
construct) with the chosen Schur arithmetic -- a short workload for launch lists
and ncu captures of the Schur kernels.
    python tools/oz_step.py [schur_arith] [shifts] [n]"""
import os
import sys
import time

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np  # noqa: E402

from paper_2311_08618_b200 import _native, configs, construct  # noqa: E402

arith = int(sys.argv[1]) if len(sys.argv) > 1 else 1
S = int(sys.argv[2]) if len(sys.argv) > 2 else 7
n = int(sys.argv[3]) if len(sys.argv) > 3 else 16384
cloud, kern, tree, st = configs.config_problem("cfg2", seed=0, n=n, leaf=256)
H = construct(kern, tree, st, configs.CONFIGS["cfg2"].eps)
eng = _native.engine_for(H, 0)
eng.set_option("schur_arith", arith)
eng.set_option("time_kernels", 2)
mus = np.linspace(-50.0, 50.0, S)
for rep in range(2):
    t0 = time.perf_counter()
    counts, status, stt = eng.inertia(mus)
    print(f"arith={arith} rep={rep}: {time.perf_counter() - t0:.3f} s wall, device {stt['ms_total']:.1f} ms, "
          f"schur {stt['ms_schur']:.1f} ms ({stt['schur_flops'] / stt['ms_schur'] / 1e9:.1f} TF/s), "
          f"launches {stt['launches']}", flush=True)
print(counts[:, 0].tolist())
if os.environ.get("H2L_OZ_PROBE") == "8":
    import ctypes
    tl = _native.load_testing_library()
    buf = (ctypes.c_ulonglong * 16)()
    tl.h2l_internal_oz_prof(buf, 1)
    v = list(buf)
    items = max(1, v[0])
    names = ["items", "epi:tables", "epi:wait_mma", "epi:tmem+sum", "epi:stage", "epi:scatter", "", "",
             "mma:wait_epi", "mma:wait_tma", "mma:issue"]
    print("oz phases (cycles per item):",
          {n: round(v[k] / items) for k, n in enumerate(names) if n and k}, "items", items)
