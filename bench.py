"""Benchmark: H2-LDL inertia evaluations per second on B200 (BASELINE.json metric).

    python bench.py [--gpus N] [--steps K] [--warmup W] [--impl ours|reference]
                    [--config cfg1] [--batch S]

Workload (config.workload): BASELINE config 1 -- 3D 1/r kernel, n = 2048
uniform points in [0,1]^3 (seed 0, Morton order), leaf 128, eta = 1,
eps = 1e-8.  This is the only configuration whose input (the H2 matrix) can
be built today (configs 2-5 need the GPU construction that SURVEY.md §8f
lists next).  A step = one shift-batched sweep of the generalized LDL^T over
S shifts (default 256) spread over the spectrum; `value` = shifts factorized
per second over K timed steps (device time, CUDA events on the engine's
stream, max over ranks); inputs (the uploaded H payload, 17.8 MB, and its
s-batched working copies, 4.6 GB per step at S = 256) are resident in HBM and exceed L2,
so no flush is needed.  `e2e` = the same metric through the public API
`inertia_batch(H, mus)` with host shift lists and host counts (H2D of the
shifts and D2H of the counts inside the timed region, wall clock).

Multi-GPU (torchrun): one rank per GPU, each with its own replica and S
shifts per step (weak scaling; the path shards over shifts, no collective in
the data path -- SURVEY.md §8e).

`--impl reference`: the reference algorithm on the host CPU through the
oracle port (oracle/engine_ref.py, the reference's engine restated in
numpy/scipy with the reference kernel's C restatement), all host cores as
worker processes, rank 0 only.
"""

import argparse
import json
import os
import subprocess
import sys
import threading
import time

ROOT = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, ROOT)

import numpy as np  # noqa: E402

METRIC = "H2-LDL inertia evals/s (cfg1 n=2048 3D 1/r leaf 128, shift-batched)"
UNIT = "inertia evals/s"


def _dist():
    world = int(os.environ.get("WORLD_SIZE", "1"))
    rank = int(os.environ.get("RANK", "0"))
    local = int(os.environ.get("LOCAL_RANK", "0"))
    return world, rank, local


def shifts_for(eigs_lo, eigs_hi, s, step, rank):
    """Deterministic shifts spread over [lo, hi] (distinct per step and rank)."""
    rng = np.random.default_rng(1000 * step + rank)
    return np.sort(rng.uniform(eigs_lo, eigs_hi, s))


class ClockSampler:
    """nvidia-smi sampling of SM clocks and throttle reasons during the timed region."""

    Q = ("clocks.sm,clocks.max.sm,power.draw,clocks_event_reasons.hw_slowdown,"
         "clocks_event_reasons.hw_thermal_slowdown,clocks_event_reasons.sw_thermal_slowdown,"
         "clocks_event_reasons.sw_power_cap")

    def __init__(self, index):
        self.index = index
        self.rows = []
        self._stop = threading.Event()
        self._t = None

    def _run(self):
        while not self._stop.is_set():
            try:
                out = subprocess.run(["nvidia-smi", "-i", str(self.index), f"--query-gpu={self.Q}",
                                      "--format=csv,noheader,nounits"], capture_output=True,
                                     text=True, timeout=5).stdout.strip()
                if out:
                    self.rows.append([v.strip() for v in out.split(",")])
            except Exception:  # noqa: BLE001
                pass
            self._stop.wait(0.2)

    def start(self):
        self._t = threading.Thread(target=self._run, daemon=True)
        self._t.start()

    def stop(self):
        self._stop.set()
        if self._t:
            self._t.join(timeout=10)
        sm = [float(r[0]) for r in self.rows if r[0].replace(".", "").isdigit()]
        mx = [float(r[1]) for r in self.rows if r[1].replace(".", "").isdigit()]
        names = ["hw_slowdown", "hw_thermal_slowdown", "sw_thermal_slowdown", "sw_power_cap"]
        reasons = sorted({names[q] for r in self.rows for q in range(4)
                          if len(r) > 3 + q and "Active" in r[3 + q] and "Not" not in r[3 + q]})
        return {"sm_mhz": float(np.median(sm)) if sm else None,
                "sm_max_mhz": max(mx) if mx else None, "reasons": reasons,
                "samples": len(self.rows)}


def measure_fp64_peak(torch, dev):
    """cuBLAS DGEMM 8192^3 (torch.matmul fp64), best of 5 -> TFLOP/s."""
    n = 8192
    a = torch.randn(n, n, dtype=torch.float64, device=dev)
    b = torch.randn(n, n, dtype=torch.float64, device=dev)
    torch.matmul(a, b)
    torch.cuda.synchronize()
    best = 1e9
    for _ in range(5):
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record()
        torch.matmul(a, b)
        e1.record()
        torch.cuda.synchronize()
        best = min(best, e0.elapsed_time(e1) / 1e3)
    del a, b
    torch.cuda.empty_cache()
    return 2.0 * n ** 3 / best / 1e12


def build_cfg1():
    from paper_2311_08618_b200 import configs, construct

    cloud, kern, tree, st = configs.config_problem("cfg1", seed=0)
    return construct(kern, tree, st, configs.CONFIGS["cfg1"].eps)


def cfg1_interval():
    z = np.load(os.path.join(ROOT, "tests", "golden", "cfg1.npz"))
    return tuple(float(v) for v in z["interval"]), z["eigs"]


# ------------------------------------------------------------------ reference
def _ref_worker(args):
    os.environ["OPENBLAS_NUM_THREADS"] = "1"
    mus, = args
    from oracle import engine_ref

    H = build_cfg1()
    cache = {}
    out = []
    for mu in mus:
        out.append(engine_ref.inertia(H, float(mu), skel_cache=cache))
    return out


def run_reference(args):
    world, rank, _ = _dist()
    if rank != 0:
        return
    import multiprocessing as mp

    # spawn (not fork): a forked child inherits the parent's OpenBLAS thread pool
    # in a broken state and can deadlock on its first BLAS call
    for var in ("OPENBLAS_NUM_THREADS", "OMP_NUM_THREADS", "MKL_NUM_THREADS"):
        os.environ[var] = "1"
    cores = os.cpu_count() or 1
    (lo, hi), _ = cfg1_interval()
    ctx = mp.get_context("spawn")
    with ctx.Pool(cores) as pool:
        # warm the per-process skeleton caches / imports
        pool.map(_ref_worker, [([0.0],)] * cores)
        per = 1  # shifts per worker per step: one factorization each (~0.5 s)
        for w in range(args.warmup):
            pool.map(_ref_worker, [(shifts_for(lo, hi, per, w, q),) for q in range(cores)])
        t0 = time.perf_counter()
        for k in range(args.steps):
            pool.map(_ref_worker, [(shifts_for(lo, hi, per, 100 + k, q),) for q in range(cores)])
        dt = time.perf_counter() - t0
    total = cores * per * args.steps
    v = total / dt
    line = {
        "impl": "reference", "metric": METRIC, "value": v, "unit": UNIT, "n_gpus": args.gpus,
        "steps": args.steps, "warmup": args.warmup, "ms_per_step": 1e3 * dt / args.steps,
        "higher_is_better": True, "scaling": "weak", "vs_baseline": None, "dtype": "f64",
        "data": "synthetic", "config": {"workload": "cfg1", "n": 2048, "leaf": 128,
                                       "kernel": "1/r", "eps": 1e-8, "shifts_per_step": total // args.steps},
        "cpu_baseline": {"value": v, "unit": UNIT, "cores": cores, "kind": "port",
                         "sample": f"{cores} worker processes x {per} factorization per step "
                                   f"(oracle/engine_ref.py, OPENBLAS_NUM_THREADS=1)"},
        "e2e": {"value": v, "unit": UNIT, "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0},
    }
    print(json.dumps(line), flush=True)


def cpu_baseline_sample(seconds=15.0):
    """Oracle port on one host core, bounded sample of cfg1 shifts."""
    os.environ["OPENBLAS_NUM_THREADS"] = "1"
    try:
        from threadpoolctl import threadpool_limits
        lim = threadpool_limits(1)
    except Exception:  # noqa: BLE001
        lim = None
    from oracle import engine_ref

    H = build_cfg1()
    (lo, hi), _ = cfg1_interval()
    cache = {}
    engine_ref.inertia(H, 0.0, skel_cache=cache)  # warm the skeleton cache
    t0 = time.perf_counter()
    n = 0
    while time.perf_counter() - t0 < seconds:
        engine_ref.inertia(H, float(shifts_for(lo, hi, 1, 7, n)[0]), skel_cache=cache)
        n += 1
    dt = time.perf_counter() - t0
    if lim is not None:
        lim.unregister() if hasattr(lim, "unregister") else None
    return {"value": n / dt, "unit": UNIT, "cores": 1, "kind": "port",
            "sample": f"{n} single-shift factorizations of cfg1 in {dt:.1f} s "
                      f"(oracle/engine_ref.py, 1 thread)"}


# ----------------------------------------------------------------------- ours
def run_ours(args):
    import torch

    world, rank, local = _dist()
    if world > 1:
        import torch.distributed as dist

        dist.init_process_group("nccl", device_id=torch.device(f"cuda:{local}"))
    torch.cuda.set_device(local)
    from paper_2311_08618_b200 import _native, inertia_batch
    from paper_2311_08618_b200.ldl import ldl_counts_array

    _native.set_default_device(local)
    H = build_cfg1()
    (lo, hi), eigs = cfg1_interval()
    eng = _native.engine_for(H, local)
    eng.set_option("max_batch", args.batch)
    eng.set_option("time_kernels", 1)
    S = args.batch
    for w in range(max(3, args.warmup)):
        ldl_counts_array(H, shifts_for(lo, hi, S, w, rank))
    # ---- device-timed region
    if world > 1:
        dist.barrier()
    torch.cuda.synchronize()
    clocks = ClockSampler(local)
    clocks.start()
    ms = 0.0
    ms_schur = 0.0
    schur_flops = 0.0
    schur_bytes = 0.0
    gemm_exec = 0.0
    flops = 0.0
    launches = 0
    ok = True
    for k in range(args.steps):
        mus = shifts_for(lo, hi, S, 100 + k, rank)
        counts, status, st = ldl_counts_array(H, mus)
        ms += st["ms_total"]
        ms_schur += st["ms_schur"]
        schur_flops += st["schur_flops"]
        schur_bytes += st["bytes"]
        gemm_exec += st["gemm_flops_exec"]
        flops += st["flops"]
        launches += st["launches"]
        if k == 0:  # spot-check against the exact spectrum (rank-0 H2: exact matrix)
            want = np.searchsorted(eigs, mus)
            ok = ok and bool(np.array_equal(counts[:, 0], want)) and not status.any()
    torch.cuda.synchronize()
    clk = clocks.stop()
    t_dev = ms / 1e3
    if world > 1:
        tt = torch.tensor([t_dev], dtype=torch.float64, device="cuda")
        dist.all_reduce(tt, op=dist.ReduceOp.MAX)
        t_dev = float(tt.item())
    value = world * S * args.steps / t_dev
    # ---- e2e through the public API (host shifts in, host counts out)
    if world > 1:
        dist.barrier()
    t0 = time.perf_counter()
    for k in range(args.steps):
        inertia_batch(H, list(shifts_for(lo, hi, S, 200 + k, rank)))
    t_e2e = time.perf_counter() - t0
    if world > 1:
        tt = torch.tensor([t_e2e], dtype=torch.float64, device="cuda")
        dist.all_reduce(tt, op=dist.ReduceOp.MAX)
        t_e2e = float(tt.item())
    e2e = world * S * args.steps / t_e2e
    if rank != 0:
        dist.destroy_process_group()
        return
    peak = measure_fp64_peak(torch, "cuda")
    achieved = schur_flops / (ms_schur / 1e3) / 1e12 if ms_schur > 0 else None
    # ---- seconds per eigenvalue (k = n/2, eps_ev = 1e-8), sequential and multisection
    from paper_2311_08618_b200 import multisection, slice_spectrum

    eng.set_option("time_kernels", 0)
    torch.cuda.synchronize()
    t0 = time.perf_counter()
    est = slice_spectrum(H, 1024, (lo, hi), 1e-8)
    t_seq = time.perf_counter() - t0
    t0 = time.perf_counter()
    (mest,) = multisection(H, [1024], (lo, hi), 1e-8, batch=63)
    t_ms = time.perf_counter() - t0
    line = {
        "metric": METRIC, "value": value, "unit": UNIT, "n_gpus": world, "steps": args.steps,
        "warmup": args.warmup, "ms_per_step": 1e3 * t_dev / args.steps, "higher_is_better": True,
        "scaling": "weak", "vs_baseline": None, "dtype": "f64", "data": "synthetic",
        "config": {"workload": "cfg1", "n": 2048, "leaf": 128, "kernel": "1/r", "eps": 1e-8,
                   "shifts_per_step": S, "parallelism": f"shift-replicas x{world}",
                   "l2": "inputs larger than L2 (s x 17.8 MB per step)"},
        "roofline": {"bound": "tensor", "kernel": "gemm_kernel (Schur update, DMMA fp64)",
                     "achieved": achieved, "peak": peak, "unit": "TFLOP/s",
                     "frac": (achieved / peak) if achieved else None, "traffic": None,
                     "peak_source": "measured in-run: cuBLAS DGEMM fp64 8192^3 best of 5 "
                                    "(MEASURED_PEAKS.json has no fp64 figure)",
                     "schur_share_of_step": ms_schur / ms if ms else None,
                     "algorithmic_flops_per_eval": schur_flops / (S * args.steps),
                     "algorithmic_bytes_per_eval": schur_bytes / (S * args.steps),
                     "flops_rule": "SURVEY.md §8d: Schur 2 nR [sum_{a<b} l_a l_b + 1/2 sum_a l_a^2] "
                                   "per elimination step, live rows only"},
        "step_rates": {"algorithmic_tflops": flops / t_dev / 1e12 / max(1, 1),
                       "dmma_executed_tflops": gemm_exec / (ms / 1e3) / 1e12 if ms else None},
        "e2e": {"value": e2e, "unit": UNIT, "h2d_bytes_per_step": 8 * S,
                "d2h_bytes_per_step": (3 * 8 + 4) * S},
        "gpu_launches": launches,
        "clocks": clk,
        "parity_spot_check": ok,
        "eigenvalue": {"k": 1024, "eps_ev": 1e-8, "sequential_s": t_seq,
                       "sequential_evals": est.inertia_evals, "multisection_s": t_ms,
                       "multisection_evals": mest.inertia_evals,
                       "value": est.value, "multisection_equal": mest.value == est.value,
                       "abs_err_vs_eigvalsh": abs(est.value - float(eigs[1023]))},
        "algorithmic_flops_per_step": flops / args.steps,
    }
    if not args.no_cpu_baseline:
        line["cpu_baseline"] = cpu_baseline_sample(args.cpu_seconds)
    print(json.dumps(line), flush=True)
    if world > 1:
        dist.destroy_process_group()


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=10)
    ap.add_argument("--warmup", type=int, default=3)
    ap.add_argument("--impl", default="ours", choices=["ours", "reference"])
    ap.add_argument("--config", default="cfg1", choices=["cfg1"])
    ap.add_argument("--batch", type=int, default=256)
    ap.add_argument("--cpu-seconds", type=float, default=15.0)
    ap.add_argument("--no-cpu-baseline", action="store_true")
    args = ap.parse_args()
    if args.impl == "reference":
        run_reference(args)
    else:
        run_ours(args)


if __name__ == "__main__":
    main()
