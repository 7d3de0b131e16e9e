"""Time the INT8 Ozaki Schur product (k_schur_oz.cu, dense test target) on Schur-like
shapes; prints fp64-equivalent TF/s over the upper triangle (R (R+1) K per shift).
    python tools/oz_bench.py [probe]   probe 1: MMAs without waiting for loads, 2: loads only
"""
import ctypes
import os
import sys

import numpy as np

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_2311_08618_b200 import _native  # noqa: E402

_f64p = ctypes.POINTER(ctypes.c_double)
lib = _native.load_testing_library()
f = lib.h2l_internal_schur_oz
f.argtypes = [ctypes.c_int, ctypes.c_int, ctypes.c_int, ctypes.c_int, _f64p, _f64p, _f64p,
              ctypes.c_int, _f64p, ctypes.c_int]
probes = [int(a) for a in sys.argv[1:]] or [0]
for (s, R, K) in [(7, 4096, 448), (7, 16384, 160), (7, 16384, 256), (2, 40960, 192)]:
    rng = np.random.default_rng(0)
    X = rng.standard_normal((s, R, K))
    B = rng.standard_normal((s, R, K))
    C = np.zeros((s, R, R))
    for pr in probes:
        ms = ctypes.c_double(0)
        rc = f(0, R, K, s, X.ctypes.data_as(_f64p), B.ctypes.data_as(_f64p), C.ctypes.data_as(_f64p),
               10, ctypes.byref(ms), pr)
        assert rc == 0, lib.h2l_testing_last_error()
        fl = s * R * (R + 1) * K
        print(f"probe={pr} s={s} R={R} K={K}: {ms.value:.3f} ms  {fl / ms.value / 1e9:.1f} TF/s "
              f"fp64-equivalent", flush=True)
        if pr == 8:
            buf = (ctypes.c_ulonglong * 16)()
            lib.h2l_internal_oz_prof(buf, 1)
            v = list(buf)
            names = ["items", "epi:tables", "epi:wait_mma", "epi:tmem+sum", "epi:stage", "epi:scatter", "",
                     "", "mma:wait_epi", "mma:wait_tma", "mma:issue"]
            print("   cycles per item:", {n: round(v[k] / max(1, v[0])) for k, n in enumerate(names) if n and k})
