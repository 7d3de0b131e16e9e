"""Probe cusolverDnXsyevd buffer sizes for large n (64-bit API) via ctypes."""
import ctypes
import glob
import sys

import torch

torch.linalg.eigvalsh(torch.eye(4, dtype=torch.float64, device="cuda"))  # loads torch's cusolver
libs = sorted(glob.glob(torch.__path__[0] + "/../nvidia/cusolver/lib/libcusolver.so*")) + \
    sorted(glob.glob(torch.__path__[0] + "/../nvidia/cu*/lib/libcusolver.so*"))
print(libs)
cs = ctypes.CDLL(libs[0])
h = ctypes.c_void_p()
print("create", cs.cusolverDnCreate(ctypes.byref(h)))
p = ctypes.c_void_p()
print("params", cs.cusolverDnCreateParams(ctypes.byref(p)))
for n in [int(a) for a in sys.argv[1:]] or [32768, 46340, 46341, 49152, 65536]:
    dev = ctypes.c_size_t(0)
    host = ctypes.c_size_t(0)
    A = torch.empty(1, dtype=torch.float64, device="cuda")
    W = torch.empty(1, dtype=torch.float64, device="cuda")
    # jobz N = 0, uplo lower = 0 (CUBLAS_FILL_MODE_LOWER), CUDA_R_64F = 1
    rc = cs.cusolverDnXsyevd_bufferSize(h, p, 0, 0, ctypes.c_int64(n), 1, ctypes.c_void_p(A.data_ptr()),
                                        ctypes.c_int64(n), 1, ctypes.c_void_p(W.data_ptr()), 1,
                                        ctypes.byref(dev), ctypes.byref(host))
    print(n, "rc", rc, "device ws GB", dev.value / 1e9, "host ws", host.value, flush=True)
