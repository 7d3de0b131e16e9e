"""Build cfg2 once on the GPU, time inertia sweeps for several (max_batch, concurrency, shifts)."""
import os, sys, time
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np
import torch
from paper_2311_08618_b200 import _native, gpu_build

name = os.environ.get("CFG", "cfg2")
Hd, cloud = gpu_build.config_device(name)
torch.cuda.synchronize()
eng = _native.engine_for(Hd, 0)
eng.set_option("time_kernels", 0)
combos = [tuple(int(v) for v in c.split("x")) for c in sys.argv[1:]]  # MBxCxS
base = [-10.0, -8.0, -6.0, -4.0, -2.0, 0.0, 2.0, 4.0, 6.0, 8.0, 10.0, 12.0, 14.0, 16.0, 18.0, 20.0]
for rep in range(int(os.environ.get("REPS", "2"))):
    for mb, c, s in combos:
        eng.set_option("max_batch", mb)
        eng.set_option("concurrency", c)
        mus = base[:s]
        t0 = time.perf_counter()
        counts, status, st = eng.inertia(mus)
        dt = time.perf_counter() - t0
        print(f"rep {rep} MB={mb} C={c} S={s}: {dt:.2f} s wall, {st['ms_total'] / 1e3:.2f} s device, "
              f"{dt / s:.3f} s/shift, mem {st['mem_peak'] / 1e9:.0f} GB, ok={not status.any()}",
              flush=True)
