"""Build libh2ldl.so (the product) and libh2ldl_testing.so (test / benchmark entry
points, linked against the product library) in-tree with nvcc for sm_100a
(no JIT, no torch extension).

    python -m paper_2311_08618_b200.build_native [--force]
"""

import os
import subprocess
import sys

HERE = os.path.dirname(os.path.abspath(__file__))
SRC = os.path.join(HERE, "csrc")
OUT = os.path.join(HERE, "libh2ldl.so")
OUT_TESTING = os.path.join(HERE, "libh2ldl_testing.so")
SOURCES = ["engine.cu", "k_copy.cu", "k_gemm.cu", "k_bk.cu", "k_panel.cu", "k_qr.cu", "k_rrqr.cu",
           "k_bk_cluster.cu", "k_schur_oz.cu"]
TESTING_SOURCES = ["testing.cu", "k_gemm_variants.cu"]
NVCC = os.environ.get("NVCC", "/usr/local/cuda/bin/nvcc")
FLAGS = ["-O3", "-std=c++17", "-gencode", "arch=compute_100a,code=sm_100a", "-lineinfo",
         "-Xcompiler", "-fPIC", "-shared", "-Xcompiler", "-O2"]


def _stale(out, sources):
    if not os.path.exists(out):
        return True
    t = os.path.getmtime(out)
    deps = [os.path.join(SRC, f) for f in os.listdir(SRC) if f.endswith((".cuh", ".h"))]
    deps += [os.path.join(SRC, f) for f in sources]
    deps.append(os.path.join(os.path.dirname(HERE), "include", "h2ldl.h"))
    return any(os.path.getmtime(d) > t for d in deps)


def _nvcc(out, sources, extra, verbose):
    cmd = [NVCC, *FLAGS, *[os.path.join(SRC, s) for s in sources], *extra, "-o", out + ".tmp"]
    if verbose:
        print(" ".join(cmd), flush=True)
    subprocess.check_call(cmd)
    os.replace(out + ".tmp", out)


def build(force=False, verbose=False):
    if force or _stale(OUT, SOURCES):
        _nvcc(OUT, SOURCES, [], verbose)
    if force or _stale(OUT_TESTING, TESTING_SOURCES) or os.path.getmtime(OUT_TESTING) < os.path.getmtime(OUT):
        _nvcc(OUT_TESTING, TESTING_SOURCES,
              ["-L" + HERE, "-lh2ldl", "-Xlinker", "-rpath,$ORIGIN"], verbose)
    return OUT


if __name__ == "__main__":
    print(build(force="--force" in sys.argv, verbose=True))
