"""Full-size same-H parity and a measured CPU factorization (run on the GPU box).

    python tools/fullsize_parity.py cfg5 cfg3 cfg2 [--out gpurun_out/fullsize.json]

For each BASELINE config at its full size: build H on the device, factor it on
the GPU at a shift (reference order and the bench's production settings), then
export the SAME H to host memory and run the oracle port (oracle/engine_ref.py,
numpy/scipy BLAS on every host core) to completion at the same shift.  Records
both counts, the structural statistics and the wall time of the complete CPU
factorization (the measured CPU baseline of one inertia evaluation).
"""

import json
import os
import sys
import time

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

import numpy as np  # noqa: E402

# shifts: one across the widest gap among the ENDS lowest eigenvalues and one across the
# widest among the ENDS highest (the interior of these spectra is too dense for gaps wider
# than the parity guard DELTA); counts there are non-trivial (k and n - k negatives)
ENDS = 4
GUARD = 10.0  # DELTA = GUARD * eps * max(|lo|, |hi|): the guard of the reference fixtures
PROD = {"cfg2": (7, 1, 1, 0), "cfg3": (8, 2, 2, 0), "cfg4": (2, 1, 2, 1), "cfg5": (8, 2, 3, 0)}


def main():
    import torch

    from oracle import engine_ref
    from paper_2311_08618_b200 import _native, gpu_build, multisection
    from paper_2311_08618_b200.bisection import InertiaCache
    from paper_2311_08618_b200.ldl import ldl_counts_array

    out_path = "gpurun_out/fullsize.json"
    names = []
    args = sys.argv[1:]
    while args:
        a = args.pop(0)
        if a == "--out":
            out_path = args.pop(0)
        else:
            names.append(a)
    results = []
    for name in names:
        t0 = time.perf_counter()
        H, cloud = gpu_build.config_device(name)
        torch.cuda.synchronize()
        t_con = time.perf_counter() - t0
        iv = gpu_build.gershgorin_device(H._kernel)
        eng = _native.engine_for(H, 0)
        delta = GUARD * H.eps * max(abs(iv[0]), abs(iv[1]))
        eng.set_option("max_batch", 8)
        eng.set_option("concurrency", 1)
        # locate the J lowest and J highest eigenvalues of the factored matrix to a quarter of
        # the guard (device multisection); a shift midway across a gap wider than 3 delta has
        # no eigenvalue within delta: a certified, non-trivial parity shift (count k or n - k)
        n = cloud.n
        ks = list(range(1, ENDS + 1)) + list(range(n - ENDS + 1, n + 1))
        t_loc = time.perf_counter()
        ests = multisection(H, ks, iv, delta / 4, cache=InertiaCache(), batch=32)
        t_loc = time.perf_counter() - t_loc
        lam = {e.k: (e.value, e.half_width) for e in ests}
        located = [[e.k, e.value, e.half_width] for e in ests]
        print(name, "located", located, f"{t_loc:.1f}s", flush=True)
        mus, rejected = [], []
        for side in (range(1, ENDS), range(n - ENDS + 1, n)):
            best = None
            for k in side:
                (a, ha), (b, hb) = lam[k], lam[k + 1]
                gap = (b - hb) - (a + ha)
                if gap > 3 * delta and (best is None or gap > best[0]):
                    best = (gap, 0.5 * (a + ha + b - hb), k)
            if best is not None:
                mus.append(best[1])
            else:
                rejected.append(list(side))
        # independent check of the certification: equal counts at mu - delta, mu, mu + delta
        probe = [x for m in mus for x in (m - delta, m, m + delta)]
        pc, _, _ = ldl_counts_array(H, probe) if probe else (np.zeros((0, 3)), None, None)
        certified = [[int(pc[3 * q + d, 0]) for d in range(3)] for q in range(len(mus))]
        print(name, "shifts", mus, "negatives at -d/0/+d", certified, flush=True)
        gpu = {}
        for label, (mb, conc, sched, order, budget, arith) in (
                ("reference_order", (4, 1, 0, 1 if name == "cfg4" else 0, 0, 0)),
                ("production", PROD[name] + (1, 1))):
            eng.set_option("schur_arith", arith)
            eng.set_option("max_batch", mb)
            eng.set_option("concurrency", conc)
            eng.set_option("schedule", sched)
            eng.set_option("elim_order", order)
            eng.set_option("qr_budget", budget)
            counts, status, st = ldl_counts_array(H, mus)
            gpu[label] = {"counts": counts.tolist(), "status": status.tolist(),
                          "ms_total": st["ms_total"], "rank_added": st["rank_added"],
                          "fill_blocks": st["fill_blocks"], "recompressions": st["recompressions"],
                          "max_front": st["max_front"], "groups": st["groups"],
                          "launches": st["launches"], "elim_flops": st["elim_flops"]}
            print(name, label, gpu[label], flush=True)
        t1 = time.perf_counter()
        host_H = gpu_build.to_host(H)
        t_exp = time.perf_counter() - t1
        del eng, H
        _native.engine_for  # noqa: B018 (engines are cached on the device H, freed with it)
        torch.cuda.empty_cache()
        cpu = []
        cache = {}
        for mu in mus:
            t2 = time.perf_counter()
            try:
                oe = engine_ref.OracleEngine(host_H, host_H.shift + mu, cache).run()
                c = tuple(oe.counts)
                stats = dict(oe.stats)
                flops = oe.elim_flops
                err = None
            except engine_ref.ShiftHit as exc:
                c, stats, flops, err = None, {}, 0.0, repr(exc)
            dt = time.perf_counter() - t2
            cpu.append({"mu": mu, "counts": c, "stats": stats, "seconds": dt, "elim_flops": flops,
                        "error": err})
            print(name, "oracle", mu, c, stats, f"{dt:.1f}s", flush=True)
        try:
            from threadpoolctl import threadpool_info

            threads = max([d.get("num_threads", 1) for d in threadpool_info()] or [1])
        except Exception:  # noqa: BLE001
            threads = os.cpu_count()
        rec = {"config": name, "n": cloud.n, "interval": list(iv), "mus": mus,
               "located_eigenvalues": located, "locate_s": t_loc, "probe_negatives": certified,
               "guard_delta": delta, "rejected_candidates": rejected,
               "construct_device_s": t_con, "export_s": t_exp, "gpu": gpu, "oracle": cpu,
               "host_threads": threads, "cpu_count": os.cpu_count(),
               "counts_equal": all(
                   cpu[q]["counts"] is not None
                   and [list(cpu[q]["counts"])] == [gpu["reference_order"]["counts"][q]]
                   and gpu["production"]["counts"][q] == gpu["reference_order"]["counts"][q]
                   for q in range(len(mus)))}
        results.append(rec)
        with open(out_path, "w") as f:
            json.dump(results, f, indent=1)
        del host_H, cache


if __name__ == "__main__":
    main()
