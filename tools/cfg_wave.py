"""One production wave of a BASELINE config on the device-built H, for each Schur
arithmetic given (set H2L_SCHURLOG=1 for a per-launch Schur log on stderr).
    python tools/cfg_wave.py cfg2 [arith ...] [--shifts S]"""
import os
import sys
import time

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np  # noqa: E402


def main():
    import torch

    from paper_2311_08618_b200 import _native, gpu_build
    args = sys.argv[1:]
    S = 7
    if "--shifts" in args:
        i = args.index("--shifts")
        S = int(args[i + 1])
        del args[i:i + 2]
    name = args[0]
    ariths = [int(a) for a in args[1:]] or [0, 1]
    H, cloud = gpu_build.config_device(name)
    iv = gpu_build.gershgorin_device(H._kernel)
    eng = _native.engine_for(H, 0)
    eng.set_option("max_batch", S)
    eng.set_option("concurrency", 1)
    eng.set_option("schedule", 1 if name == "cfg2" else 2)
    if name == "cfg4":
        eng.set_option("elim_order", 1)
    a, b = iv
    mus = [a + (b - a) * (j + 1) / (S + 1) for j in range(S)]
    for ar in ariths:
        eng.set_option("schur_arith", ar)
        eng.set_option("time_kernels", 1)
        print(f"=== arith {ar}", file=sys.stderr, flush=True)
        t0 = time.perf_counter()
        counts, status, st = eng.inertia(np.asarray(mus))
        torch.cuda.synchronize()
        print(f"arith={ar}: wall {time.perf_counter() - t0:.2f} s device {st['ms_total']:.0f} ms "
              f"schur {st['ms_kind'][1]:.0f} ms kinds {[round(x) for x in st['ms_kind']]} "
              f"neg {counts[:, 0].tolist()}", flush=True)


if __name__ == "__main__":
    main()
