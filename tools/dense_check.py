"""Full-size parity against dense LAPACK-class eigenvalues (run on the GPU box).

    python tools/dense_check.py cfg2 [--n N] [--out gpurun_out/dense_check_cfg2.json] [--no-eig]

cuSOLVER's syevd rejects n = 65536 (CUSOLVER_STATUS_INVALID_VALUE from the 64-bit
Xsyevd buffer query; MAGMA's dsytrd overflows 32-bit indices and faults), and host
LAPACK needs hours at that size, so the dense spectrum is taken at the largest size
cuSOLVER accepts: the config's own recipe (leaf, eta, eps, kernel, point law) at
n = 32768 (--n), fronts and ranks of the full-size run.

Builds the config's H on the device, realises it densely on the device
(gpu_build.reconstruct_dense_device: 34 GB for config 2) and takes its exact spectrum
with cuSOLVER (torch.linalg.eigvalsh, fp64).  Then, with the engine in its production
settings:
  * counts at shifts inside spectral gaps wider than twice the parity guard
    (10 eps max|lambda|, the guard of the reference fixtures) must equal the number of
    eigenvalues below the shift -- bit-exact inertia on the full-size matrix;
  * the multisection estimates of lambda_k, k in {1, n/2, n} (BASELINE config 2), must
    lie within eps_ev + the truncation band of the exact eigenvalue.
"""

import json
import os
import sys
import time

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

import numpy as np  # noqa: E402


def main():
    import torch

    from paper_2311_08618_b200 import _native, configs, gpu_build, multisection
    from paper_2311_08618_b200.bisection import InertiaCache
    from paper_2311_08618_b200.ldl import ldl_counts_array

    args = sys.argv[1:]
    name = args[0] if args and not args[0].startswith("--") else "cfg2"
    out = f"gpurun_out/dense_check_{name}.json"
    if "--out" in args:
        out = args[args.index("--out") + 1]
    cfg = configs.CONFIGS[name]
    nreq = int(args[args.index("--n") + 1]) if "--n" in args else None
    rec = {"config": name}
    t0 = time.perf_counter()
    H, cloud = gpu_build.config_device(name, n=nreq)
    torch.cuda.synchronize()
    rec["construct_s"] = time.perf_counter() - t0
    n = cloud.n
    iv = gpu_build.gershgorin_device(H._kernel)
    t0 = time.perf_counter()
    A = gpu_build.reconstruct_dense_device(H)
    torch.cuda.synchronize()
    rec["reconstruct_s"] = time.perf_counter() - t0
    t0 = time.perf_counter()
    w = torch.linalg.eigvalsh(A).cpu().numpy()
    rec["eigvalsh_backend"] = "cuSOLVER syevd (torch.linalg.eigvalsh, fp64)"
    rec["eigvalsh_s"] = time.perf_counter() - t0
    del A
    torch.cuda.empty_cache()
    print(name, "eigvalsh", rec["eigvalsh_s"], "s; range", w[0], w[-1], flush=True)
    nrm = max(abs(w[0]), abs(w[-1]))
    guard = 10 * cfg.eps * nrm
    gaps = np.diff(w)
    wide = np.nonzero(gaps > 2 * guard)[0]
    rng = np.random.default_rng(3)
    pick = sorted(rng.choice(wide, size=min(14, len(wide)), replace=False).tolist()) if len(wide) else []
    mus = [float(0.5 * (w[i] + w[i + 1])) for i in pick]
    want = [int(i + 1) for i in pick]
    eng = _native.engine_for(H, 0)
    eng.set_option("max_batch", 7)
    eng.set_option("concurrency", 1)
    t0 = time.perf_counter()
    counts, status, st = ldl_counts_array(H, mus)
    rec["counts_s"] = time.perf_counter() - t0
    got = [int(c) for c in counts[:, 0]]
    rec.update({"n": n, "interval": list(iv), "lambda_min": float(w[0]), "lambda_max": float(w[-1]),
                "guard": guard, "wide_gaps": int(len(wide)), "mus": mus, "eigvalsh_neg": want,
                "engine_neg": got, "engine_zero": [int(c) for c in counts[:, 1]],
                "status": [int(s) for s in status], "counts_equal": got == want,
                "stats": {k: st[k] for k in ("fill_blocks", "recompressions", "rank_added",
                                             "max_front", "groups", "launches")}})
    print(name, "counts equal:", got == want, list(zip(want, got)), flush=True)
    with open(out, "w") as f:
        json.dump(rec, f, indent=1)
    if "--no-eig" not in args:
        ks = [1, n // 2, n] if name == "cfg2" else [k for k in cfg.ks if k <= n]
        t0 = time.perf_counter()
        ests = multisection(H, ks, iv, cfg.eps_ev, cache=InertiaCache(), batch=7)
        rec["eig_s"] = time.perf_counter() - t0
        band = 10 * cfg.eps * nrm
        rec["eigenvalues"] = [{"k": e.k, "estimate": e.value, "half_width": e.half_width,
                               "exact": float(w[e.k - 1]), "abs_err": abs(e.value - float(w[e.k - 1])),
                               "within": abs(e.value - float(w[e.k - 1])) <= cfg.eps_ev + band,
                               "evals": e.inertia_evals} for e in ests]
        rec["eig_band"] = band
        print(name, "eigenvalues", rec["eigenvalues"], flush=True)
        with open(out, "w") as f:
            json.dump(rec, f, indent=1)


if __name__ == "__main__":
    main()
