"""Build a BASELINE config on the device and time inertia sweeps under engine options.

    OPTS="schedule=3,window=64,max_batch=8,concurrency=2" S=15 REPS=2 python tools/step_probe.py cfg5

Prints per sweep: device ms, groups, launches, memory peak and (time_kernels=1)
the device ms per launch kind.  Exploration / profiling tool (not the bench)."""
import os
import sys
import time

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np  # noqa: E402
import torch  # noqa: E402

from paper_2311_08618_b200 import _native, gpu_build  # noqa: E402
from paper_2311_08618_b200.ldl import ldl_counts_array  # noqa: E402

KINDS = ["panel_gemm", "schur", "rot_merge", "bk", "panel", "copies", "rec_products", "rec_order"]


def main():
    name = sys.argv[1]
    S = int(os.environ.get("S", "15"))
    t0 = time.perf_counter()
    H, cloud = gpu_build.config_device(name)
    torch.cuda.synchronize()
    iv = gpu_build.gershgorin_device(H._kernel)
    print(f"{name}: construct {time.perf_counter() - t0:.1f} s, interval {iv}", flush=True)
    eng = _native.engine_for(H, 0)
    a, b = iv
    mus = [a + (b - a) * (j + 1) / (S + 1) for j in range(S)]
    ref = counts = status = None
    for opts in os.environ.get("OPTS", "").split(";"):
        for kv in filter(None, opts.split(",")):
            k, v = kv.split("=")
            eng.set_option(k, int(v))
        reps = int(os.environ.get("REPS", "2"))
        for rep in range(reps):
            eng.set_option("time_kernels", 1 if rep == reps - 1 and reps > 1 else 0)
            t1 = time.perf_counter()
            try:
                counts, status, st = ldl_counts_array(H, mus)
            except Exception as exc:  # noqa: BLE001
                print(f"[{opts}] rep {rep}: FAILED {exc}", flush=True)
                break
            wall = time.perf_counter() - t1
            kinds = {k: round(v, 1) for k, v in zip(KINDS, st["ms_kind"]) if v}
            print(f"[{opts}] rep {rep}: {st['ms_total']:.1f} ms dev, {wall * 1e3:.1f} ms wall, "
                  f"groups {st['groups']}, launches {st['launches']}, mem {st['mem_peak'] / 1e9:.1f} GB, "
                  f"rank_added {st['rank_added']}, fills {st['fill_blocks']}, paths {st['paths']}, "
                  f"kinds {kinds}", flush=True)
            if ref is None:
                ref = counts
            elif not np.array_equal(ref, counts):
                print(f"[{opts}] COUNTS DIFFER: {np.nonzero((ref != counts).any(axis=1))[0].tolist()}",
                      flush=True)
    if counts is not None:
        print("neg counts", counts[:, 0].tolist(), "status", status.tolist(), flush=True)


if __name__ == "__main__":
    main()
