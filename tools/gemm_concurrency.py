"""Run the production GEMM vs a naive kernel from several host threads at once."""
import ctypes, os, sys, threading
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_2311_08618_b200 import _native
lib = _native.load_testing_library()
f = lib.h2l_internal_gemm_check
f.argtypes = [ctypes.c_int] * 7 + [ctypes.POINTER(ctypes.c_double)]
f.restype = ctypes.c_int
NT = int(sys.argv[1]) if len(sys.argv) > 1 else 4
out = {}
def run(t):
    md = ctypes.c_double()
    rc = f(0, 128, 128, 128, 60, 16, 20, ctypes.byref(md))
    out[t] = (rc, md.value)
th = [threading.Thread(target=run, args=(t,)) for t in range(NT)]
[x.start() for x in th]; [x.join() for x in th]
print(NT, "threads:", [out[t] for t in range(NT)])
