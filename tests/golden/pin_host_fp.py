"""Pin host floating point so a payload rebuilt on any x86-64 host is bit-identical.

The production-size fixtures (prod_*.npz) record the sha256 digest of the payload the
REFERENCE built in this container; the GPU-box tests rebuild H with this package's host
`construct` and factor it on the device, so both sides must round identically.  Two
things make numpy/scipy results host-dependent:

  * OpenBLAS picks its kernels by CPU (SkylakeX here, something else on the box) and
    splits some routines over threads -> force the Haswell (AVX2+FMA) kernels, which
    every x86-64 host we run on has, and construct under one BLAS thread;
  * numpy dispatches its float64 exp/log/... loops to AVX-512 variants when present
    -> disable the AVX-512 dispatch targets.

Import this module BEFORE numpy (make_golden.py and tests/conftest.py do);
`check()` verifies it took effect.
"""

import os

_ENV = {
    "OPENBLAS_CORETYPE": "Haswell",
    "NPY_DISABLE_CPU_FEATURES": ("AVX512F AVX512CD AVX512_KNL AVX512_KNM AVX512_SKX AVX512_CLX "
                                 "AVX512_CNL AVX512_ICL AVX512_SPR"),
}
for _k, _v in _ENV.items():
    os.environ.setdefault(_k, _v)


def check():
    """-> '' when the pin is active in this process, else why not."""
    try:
        from numpy._core._multiarray_umath import __cpu_features__ as feats
        from threadpoolctl import threadpool_info
    except Exception as e:  # noqa: BLE001
        return f"cannot inspect: {e}"
    if feats.get("AVX512F"):
        return "numpy AVX-512 dispatch active (numpy imported before pin_host_fp)"
    arch = {d.get("architecture") for d in threadpool_info() if d.get("internal_api") == "openblas"}
    if arch - {"Haswell"}:
        return f"OpenBLAS core type {sorted(arch)} (numpy imported before pin_host_fp)"
    return ""


def single_thread():
    """Context manager: one BLAS thread (thread splits change some reductions)."""
    from threadpoolctl import threadpool_limits

    return threadpool_limits(1)
