"""tcgen05 INT8 MMA issue rate (M=128, K=32) vs N and accumulator order (testing library)."""
import ctypes
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_2311_08618_b200 import _native  # noqa: E402

lib = _native.load_testing_library()
f = lib.h2l_internal_umma_rate
f.argtypes = [ctypes.c_int, ctypes.c_int, ctypes.c_int, ctypes.c_int, ctypes.POINTER(ctypes.c_double)]
for n in (64, 128, 256):
    for order in (0, 1):
        c = ctypes.c_double()
        rc = f(0, n, order, 4096, ctypes.byref(c))
        assert rc == 0, lib.h2l_testing_last_error()
        macs = 128 * n * 32
        print(f"N={n} order={order}: {c.value:.1f} cycles/MMA  {macs / c.value:.0f} MACs/clk/SM", flush=True)
