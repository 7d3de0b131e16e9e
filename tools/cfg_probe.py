"""Build a config on the GPU and time a few inertia sweeps (exploration tool)."""
import os, sys, time
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np
import torch
from paper_2311_08618_b200 import _native, gpu_build

name = sys.argv[1]
n = int(sys.argv[2]) if len(sys.argv) > 2 and sys.argv[2] != "-" else None
mus = [float(v) for v in sys.argv[3].split(",")] if len(sys.argv) > 3 else [-10.0]
mb = int(os.environ.get("MB", "4"))
t0 = time.perf_counter()
Hd, cloud = gpu_build.config_device(name, n=n)
torch.cuda.synchronize()
t1 = time.perf_counter()
L = Hd.tree.depth
ranks = [b.rank for (l, i), b in Hd.bases.items() if l == L]
print(f"{name} n={cloud.n} depth={L} build {t1 - t0:.1f}s arena {Hd._arena.numel() * 8 / 1e9:.2f} GB "
      f"dense pairs {len(Hd.structure.dense)} leaf rank mean {np.mean(ranks):.1f} max {max(ranks)} "
      f"max rank all {Hd.max_rank()}", flush=True)
t_up = time.perf_counter()
eng = _native.engine_for(Hd, 0)
print(f"upload {time.perf_counter() - t_up:.2f} s", flush=True)
eng.set_option("max_batch", mb)
eng.set_option("time_kernels", int(os.environ.get("TK", "1")))
eng.set_option("concurrency", int(os.environ.get("C", "2")))
t2 = time.perf_counter()
eng_t = time.perf_counter() - t2
for rep in range(int(os.environ.get("REPS", "1"))):
    t2 = time.perf_counter()
    counts, status, st = eng.inertia(mus)
    dt = time.perf_counter() - t2
    print(f"rep {rep}: {len(mus)} shifts in {dt:.2f}s ({st['ms_total']:.0f} ms device), "
          f"counts {counts.tolist()} status {status.tolist()}", flush=True)
    print({k: (round(v, 3) if isinstance(v, float) else v) for k, v in st.items()}, flush=True)
print("schur TF/s", st["schur_flops"] / (st["ms_schur"] / 1e3) / 1e12 if st["ms_schur"] else None,
      "alg TF/s", st["flops"] / (st["ms_total"] / 1e3) / 1e12, flush=True)
print("mem peak GB", torch.cuda.max_memory_allocated() / 1e9, "device free/total GB",
      [v / 1e9 for v in torch.cuda.mem_get_info()])
