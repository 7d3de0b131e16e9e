"""Rebuild a production-size fixture's H exactly as the reference built it, in a fresh
process whose host floating point is pinned before numpy loads (pin_host_fp), and save
its payload; prints the payload digest.  Used by tests/test_gpu_prod.py (a pytest
plugin may import numpy before any conftest can pin it).

    python tests/golden/build_prod_payload.py prod_cfg2_16k /tmp/out.npz
"""
import os
import sys

HERE = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, HERE)
sys.path.insert(0, os.path.dirname(os.path.dirname(HERE)))
import pin_host_fp  # noqa: E402  (before numpy)
import numpy as np  # noqa: E402

from paper_2311_08618_b200 import configs, construct  # noqa: E402
from paper_2311_08618_b200.h2matrix import payload_digest, save_payload  # noqa: E402


def main():
    name, out = sys.argv[1:3]
    why = pin_host_fp.check()
    if why:
        raise SystemExit(f"host floating point not pinned: {why}")
    z = np.load(os.path.join(HERE, f"{name}.npz"))
    cfg, n, leaf = str(z["config"]), int(z["n"]), int(z["leaf"])
    cloud, kern, tree, st = configs.config_problem(cfg, seed=0, n=n, leaf=leaf)
    with pin_host_fp.single_thread():
        H = construct(kern, tree, st, configs.CONFIGS[cfg].eps)
    save_payload(out, H, compress=False)
    print(payload_digest(H))


if __name__ == "__main__":
    main()
