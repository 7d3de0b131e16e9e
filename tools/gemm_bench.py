"""Time the DMMA GEMM tile variants on Schur-shaped grouped workloads (GPU box).

    python tools/gemm_bench.py
Prints TFLOP/s per (variant, shape); variant 0 is the production config.
"""
import ctypes
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_2311_08618_b200 import _native  # noqa: E402

lib = _native.load_testing_library()
f = lib.h2l_internal_gemm_bench
f.argtypes = [ctypes.c_int] * 8 + [ctypes.POINTER(ctypes.c_double)] * 2
f.restype = ctypes.c_int
NAMES = ["64x64 w32x32 s3 Csm", "64x128 w32x64 s3 Csm", "64x64 w32x32 s2 min5",
         "64x64 w32x32 s3 min3", "64x64 w32x32 s2 min4", "128x64 w32x32 s2 min2",
         "64x64 w32x16 s2 min6", "128x64 w32x32 s3 min2", "64x64 BK32 s2 min3",
         "64x64 BK32 s3 min2"]
shapes = [(128, 128, 128, 91, 256), (256, 256, 192, 60, 32), (64, 64, 64, 300, 64),
          (200, 200, 160, 400, 4), (256, 256, 32, 200, 4)]
if len(sys.argv) > 1:
    shapes = [tuple(int(v) for v in a.split(",")) for a in sys.argv[1:]]
for (M, N, K, nt, ns) in shapes:
    for v in range(len(NAMES)):
        ms, md = ctypes.c_double(), ctypes.c_double()
        rc = f(0, v, M, N, K, nt, ns, 10, ctypes.byref(ms), ctypes.byref(md))
        if rc:
            print("rc", rc, lib.h2l_last_error(None))
            continue
        tf = 2.0 * M * N * K * nt * ns / (ms.value / 1e3) / 1e12
        print(f"M={M} N={N} K={K} tasks={nt} shifts={ns}  v{v} {NAMES[v]:18s} "
              f"{ms.value:8.3f} ms  {tf:6.2f} TF/s  maxdiff={md.value:.2e}", flush=True)
