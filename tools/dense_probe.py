"""Largest n for which torch.linalg.eigvalsh (cuSOLVER syevd, fp64) accepts a matrix."""
import sys
import torch
for n in [int(a) for a in sys.argv[1:]]:
    A = torch.randn(n, n, dtype=torch.float64, device="cuda")
    A = A + A.T
    try:
        w = torch.linalg.eigvalsh(A)
        print(n, "ok", float(w[0]), flush=True)
    except Exception as e:  # noqa: BLE001
        print(n, "fail", repr(e)[:120], flush=True)
    del A
    torch.cuda.empty_cache()
