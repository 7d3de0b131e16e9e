"""A/B an engine option on one device-built config: alternate values, print device times.

    python tools/ab_option.py OPTION v0,v1 [S] [REPS]     (env CFG=cfg2)
"""
import os, sys, time
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch
from paper_2311_08618_b200 import _native, gpu_build

opt = sys.argv[1]
vals = [int(v) for v in sys.argv[2].split(",")]
S = int(sys.argv[3]) if len(sys.argv) > 3 else 7
reps = int(sys.argv[4]) if len(sys.argv) > 4 else 3
nn = int(os.environ["N"]) if "N" in os.environ else None
Hd, cloud = gpu_build.config_device(os.environ.get("CFG", "cfg2"), n=nn)
torch.cuda.synchronize()
eng = _native.engine_for(Hd, 0)
eng.set_option("max_batch", S)
eng.set_option("concurrency", 1)
eng.set_option("time_kernels", int(os.environ.get("TK", "2")))
mus = [float(os.environ.get("MU0", "-10")) + float(os.environ.get("DMU", "2")) * q for q in range(S)]
eng.inertia(mus[:1])
for r in range(reps):
    for v in vals:
        eng.set_option(opt, v)
        counts, status, st = eng.inertia(mus)
        print(f"rep {r} {opt}={v}: total {st['ms_total']:.0f} ms, schur {st['ms_schur']:.0f} ms, "
              f"qr {st['ms_kind'][6]:.0f} ms, rank_added {st['rank_added']}, counts0 {counts[0].tolist()}",
              flush=True)
