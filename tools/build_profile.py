"""Phase times of the device construction (H2L_BUILD_PROFILE=1).
    python tools/build_profile.py cfg5 [n] ..."""
import json
import os
import sys
import time

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
os.environ["H2L_BUILD_PROFILE"] = "1"


def main():
    import torch

    from paper_2311_08618_b200 import gpu_build

    args = sys.argv[1:]
    out = []
    while args:
        name = args.pop(0)
        n = int(args.pop(0)) if args and args[0].isdigit() else None
        t0 = time.perf_counter()
        H, cloud = gpu_build.config_device(name, n=n)
        torch.cuda.synchronize()
        rec = {"config": name, "n": cloud.n, "total_s": time.perf_counter() - t0,
               "phases_s": H._build_profile,
               "ranks_leaf_max": max(b.rank for (l, i), b in H.bases.items() if l == H.tree.depth)}
        print(json.dumps(rec), flush=True)
        out.append(rec)
        del H
        torch.cuda.empty_cache()


if __name__ == "__main__":
    main()
