// libh2ldl_testing.so: test and benchmark entry points that are NOT part of the
// product ABI (include/h2ldl.h).  Linked against libh2ldl.so; used by tests/ and
// tools/ only (GEMM tile variants, naive GEMM cross-check, Gram ordering, BK
// kernels on host matrices, the INT8 Ozaki Schur kernel against a dense target).
#include <algorithm>
#include <chrono>
#include <cmath>
#include <cstdio>
#include <cstring>
#include <string>
#include <vector>

#include "common.cuh"
#include "host_util.h"

static thread_local std::string g_terr;

template <class F>
static int guarded(void *, F &&f) {
    try {
        f();
        return H2L_OK;
    } catch (const h2l::CudaFail &x) {
        g_terr = x.what();
        return x.code;
    } catch (const std::exception &x) {
        g_terr = x.what();
        return H2L_EINVAL;
    }
}

extern "C" const char *h2l_testing_last_error(void) { return g_terr.c_str(); }

// ------------------------------------------------------------ internal tooling
// Not part of the ABI (absent from h2ldl.h): micro-benchmark of the DMMA GEMM
// tile variants on a Schur-shaped grouped workload (tools/gemm_bench.py).
namespace h2l {
int gemm_variant_tiles(int v, int M, int N);
void launch_gemm_variant(int v, const GemmTask *dev_tasks, const int *dev_tile_prefix, int ntasks,
                         int total_tiles, int nshift, cudaStream_t st);
}

extern "C" int h2l_internal_gemm_bench(int device, int variant, int M, int N, int K, int ntasks,
                                       int nshift, int reps, double *ms_out, double *maxdiff_out) {
    return guarded(nullptr, [&] {
        CK(cudaSetDevice(device));
        const int64_t sa = (int64_t)M * K, sb = (int64_t)N * K, sc = (int64_t)M * N;
        const int64_t per = (sa + sb + sc) * ntasks;
        double *buf, *ref;
        CK(cudaMalloc(&buf, sizeof(double) * per * nshift));
        CK(cudaMalloc(&ref, sizeof(double) * sc * ntasks * nshift));
        std::vector<double> h(per * nshift);
        uint64_t x = 88172645463325252ull;
        for (auto &v : h) { x ^= x << 13; x ^= x >> 7; x ^= x << 17; v = (double)(x % 2001) / 1000.0 - 1.0; }
        CK(cudaMemcpy(buf, h.data(), sizeof(double) * h.size(), cudaMemcpyHostToDevice));
        std::vector<h2l::GemmTask> tasks(ntasks);
        for (int t = 0; t < ntasks; ++t) {
            h2l::GemmTask &g = tasks[t];
            g = h2l::GemmTask{};
            g.A = buf + t * sa; g.B = buf + ntasks * sa + t * sb; g.C = buf + ntasks * (sa + sb) + t * sc;
            g.sA = g.sB = g.sC = per;
            g.M = M; g.N = N; g.K = K; g.lda = K; g.ldb = K; g.ldc = N; g.tA = 0; g.tB = 1;
            g.alpha = -1.0; g.beta = 1.0;
        }
        auto run = [&](int v, int nrep, float *ms) {
            std::vector<int> pre(ntasks);
            int tiles = 0;
            for (int t = 0; t < ntasks; ++t) { pre[t] = tiles; tiles += h2l::gemm_variant_tiles(v, M, N); }
            h2l::GemmTask *dt; int *dp;
            CK(cudaMalloc(&dt, sizeof(h2l::GemmTask) * ntasks));
            CK(cudaMalloc(&dp, sizeof(int) * ntasks));
            CK(cudaMemcpy(dt, tasks.data(), sizeof(h2l::GemmTask) * ntasks, cudaMemcpyHostToDevice));
            CK(cudaMemcpy(dp, pre.data(), sizeof(int) * ntasks, cudaMemcpyHostToDevice));
            cudaEvent_t e0, e1;
            cudaEventCreate(&e0); cudaEventCreate(&e1);
            h2l::launch_gemm_variant(v, dt, dp, ntasks, tiles, nshift, 0);  // warm
            CK(cudaDeviceSynchronize());
            cudaEventRecord(e0);
            for (int r = 0; r < nrep; ++r) h2l::launch_gemm_variant(v, dt, dp, ntasks, tiles, nshift, 0);
            cudaEventRecord(e1);
            CK(cudaEventSynchronize(e1));
            cudaEventElapsedTime(ms, e0, e1);
            cudaEventDestroy(e0); cudaEventDestroy(e1);
            cudaFree(dt); cudaFree(dp);
        };
        // correctness: one launch of `variant` vs one of variant 0 from the same inputs
        const size_t cbytes = sizeof(double) * sc * ntasks;
        std::vector<double> c0(sc * ntasks), c1(sc * ntasks);
        double *Cz = buf + ntasks * (sa + sb);
        float ms = 0.f;
        CK(cudaMemcpy(ref, Cz, cbytes, cudaMemcpyDeviceToDevice));
        run(0, 0, &ms);
        CK(cudaMemcpy(c0.data(), Cz, cbytes, cudaMemcpyDeviceToHost));
        CK(cudaMemcpy(Cz, ref, cbytes, cudaMemcpyDeviceToDevice));
        run(variant, 0, &ms);
        CK(cudaMemcpy(c1.data(), Cz, cbytes, cudaMemcpyDeviceToHost));
        double md = 0.0;
        for (size_t q = 0; q < c0.size(); ++q) md = std::max(md, std::fabs(c0[q] - c1[q]));
        run(variant, reps, &ms);
        *ms_out = ms / std::max(1, reps);
        *maxdiff_out = md;
        cudaFree(buf); cudaFree(ref);
    });
}

// Debug: production GEMM vs a naive reference kernel on a Schur-shaped
// grouped workload; returns the max abs difference (tools/gemm_concurrency.py).
namespace h2l {
__global__ void naive_gemm_kernel(const GemmTask *tasks, int ntasks) {
    const int t = blockIdx.x, z = blockIdx.y;
    if (t >= ntasks) return;
    const GemmTask tk = tasks[t];
    const double *A = tk.A + z * tk.sA, *B = tk.B + z * tk.sB;
    double *C = tk.C + z * tk.sC;
    for (int e = threadIdx.x; e < tk.M * tk.N; e += blockDim.x) {
        const int r = e / tk.N, c = e % tk.N;
        double s = 0.0;
        for (int k = 0; k < tk.K; ++k) {
            const double a = tk.tA ? A[(int64_t)k * tk.lda + r] : A[(int64_t)r * tk.lda + k];
            const double b = tk.tB ? B[(int64_t)c * tk.ldb + k] : B[(int64_t)k * tk.ldb + c];
            s += a * b;
        }
        C[(int64_t)r * tk.ldc + c] = tk.alpha * s + tk.beta * C[(int64_t)r * tk.ldc + c];
    }
}
}  // namespace h2l

// Gram-matrix ordering of the recompression (k_qr.cu): `count` symmetric n x n
// matrices (host, row-major) -> Q^T (count x n x n), tau, piv; mode 0 the cluster
// kernel pair, mode 1 the single-CTA fallback pair
extern "C" int h2l_internal_gram_order(int device, int mode, int n, int count, const double *m,
                                       double *qt, double *tau, int *piv) {
    return guarded(nullptr, [&] {
        CK(cudaSetDevice(device));
        const int64_t nn = (int64_t)n * n, ts = n;
        double *dm, *dq, *dt, *dnorm, *dtol, *ddrop;
        int *dp, *du, *drank;
        CK(cudaMalloc(&dm, sizeof(double) * nn * count));
        CK(cudaMalloc(&dq, sizeof(double) * nn * count));
        CK(cudaMalloc(&dt, sizeof(double) * ts * count));
        CK(cudaMalloc(&dnorm, sizeof(double) * ts * count));
        CK(cudaMalloc(&dtol, sizeof(double) * count));
        CK(cudaMalloc(&ddrop, sizeof(double) * count));
        CK(cudaMalloc(&dp, sizeof(int) * ts * count));
        CK(cudaMalloc(&du, sizeof(int) * ts * count));
        CK(cudaMalloc(&drank, sizeof(int) * count));
        CK(cudaMemcpy(dm, m, sizeof(double) * nn * count, cudaMemcpyHostToDevice));
        CK(cudaMemset(dtol, 0, sizeof(double) * count));
        if (mode == 0) {
            if (!h2l::pqr_cluster_size(n)) throw h2l::CudaFail(H2L_EINVAL, "n too large for the cluster QR");
            CK(h2l::launch_pqr_cluster(dm, nn, n, dt, dp, ts, nullptr, count, 0));
            CK(h2l::launch_form_q_rows(dm, nn, n, dt, ts, dq, nn, nullptr, count, 0));
        } else {
            CK(h2l::launch_pqr(dm, nn, n, n, n, dt, dp, du, dnorm, ts, ts, dtol, drank, ddrop, nullptr,
                               -2, count, 0));
            CK(h2l::launch_form_tr(dm, nn, n, dt, dp, ts, n, n, dq, nn, nullptr, count, 0));
        }
        CK(cudaDeviceSynchronize());
        CK(cudaMemcpy(qt, dq, sizeof(double) * nn * count, cudaMemcpyDeviceToHost));
        CK(cudaMemcpy(tau, dt, sizeof(double) * ts * count, cudaMemcpyDeviceToHost));
        CK(cudaMemcpy(piv, dp, sizeof(int) * ts * count, cudaMemcpyDeviceToHost));
        for (void *p : {(void *)dm, (void *)dq, (void *)dt, (void *)dnorm, (void *)dtol, (void *)ddrop,
                        (void *)dp, (void *)du, (void *)drank})
            cudaFree(p);
    });
}

// engine-mode BK of `count` n x n row-major matrices (host), single-CTA (mode 0)
// or cluster (mode 1) kernel: factor (lower triangle), perm, dinfo, counts, status
extern "C" int h2l_internal_bk_engine(int device, int mode, int n, int count, double *a, int *perm,
                                      double *dinfo, int64_t *counts, int *status) {
    return guarded(nullptr, [&] {
        CK(cudaSetDevice(device));
        const int64_t nn = (int64_t)n * n, ps = n;
        double *da, *dd, *scr = nullptr;
        int *dp, *dst;
        int64_t *dc;
        h2l::BkJob *dj;
        CK(cudaMalloc(&da, sizeof(double) * nn * count));
        CK(cudaMalloc(&dd, sizeof(double) * 3 * ps * count));
        CK(cudaMalloc(&dp, sizeof(int) * ps * count));
        CK(cudaMalloc(&dst, sizeof(int) * count));
        CK(cudaMalloc(&dc, sizeof(int64_t) * 3 * count));
        CK(cudaMalloc(&dj, sizeof(h2l::BkJob)));
        CK(cudaMemcpy(da, a, sizeof(double) * nn * count, cudaMemcpyHostToDevice));
        CK(cudaMemset(dst, 0, sizeof(int) * count));
        CK(cudaMemset(dc, 0, sizeof(int64_t) * 3 * count));
        h2l::BkJob jb{da, nn, n, n, dp, dd, ps};
        CK(cudaMemcpy(dj, &jb, sizeof(jb), cudaMemcpyHostToDevice));
        if (mode == 1) {
            if (!h2l::bk_cluster_size(n)) throw h2l::CudaFail(H2L_EINVAL, "n too large for the cluster BK");
            CK(h2l::launch_bk_cluster(dj, 1, count, n, dc, dst, 0));
        } else {
            const int64_t sd = h2l::bk_scratch_doubles(n);
            if (sd) CK(cudaMalloc(&scr, sizeof(double) * sd * count));
            CK(h2l::launch_bk_engine(dj, 1, count, n, dc, dst, scr, sd, 0));
        }
        CK(cudaDeviceSynchronize());
        CK(cudaMemcpy(a, da, sizeof(double) * nn * count, cudaMemcpyDeviceToHost));
        CK(cudaMemcpy(perm, dp, sizeof(int) * ps * count, cudaMemcpyDeviceToHost));
        CK(cudaMemcpy(dinfo, dd, sizeof(double) * 3 * ps * count, cudaMemcpyDeviceToHost));
        CK(cudaMemcpy(counts, dc, sizeof(int64_t) * 3 * count, cudaMemcpyDeviceToHost));
        CK(cudaMemcpy(status, dst, sizeof(int) * count, cudaMemcpyDeviceToHost));
        for (void *p : {(void *)da, (void *)dd, (void *)dp, (void *)dst, (void *)dc, (void *)dj})
            cudaFree(p);
        if (scr) cudaFree(scr);
    });
}

extern "C" int h2l_internal_gemm_check(int device, int M, int N, int K, int ntasks, int nshift,
                                       int reps, double *maxdiff_out) {
    return guarded(nullptr, [&] {
        CK(cudaSetDevice(device));
        cudaStream_t st;
        CK(cudaStreamCreateWithFlags(&st, cudaStreamNonBlocking));
        const int64_t sa = (int64_t)M * K, sb = (int64_t)N * K, sc = (int64_t)M * N;
        const int64_t per = (sa + sb + 2 * sc) * ntasks;
        double *buf;
        CK(cudaMalloc(&buf, sizeof(double) * per * nshift));
        std::vector<double> h(per * nshift);
        uint64_t x = 0x9E3779B97F4A7C15ull ^ (uint64_t)(M * 131 + N * 7 + ntasks);
        for (auto &v : h) { x ^= x << 13; x ^= x >> 7; x ^= x << 17; v = (double)(x % 2001) / 1000.0 - 1.0; }
        CK(cudaMemcpy(buf, h.data(), sizeof(double) * h.size(), cudaMemcpyHostToDevice));
        std::vector<h2l::GemmTask> t1(ntasks), t2(ntasks);
        std::vector<int> pre(ntasks);
        int tiles = 0;
        for (int t = 0; t < ntasks; ++t) {
            h2l::GemmTask g{};
            g.A = buf + t * sa; g.B = buf + ntasks * sa + t * sb;
            g.sA = g.sB = g.sC = per;
            g.M = M; g.N = N; g.K = K; g.lda = K; g.ldb = K; g.ldc = N; g.tA = 0; g.tB = 1;
            g.alpha = -1.0; g.beta = 1.0;
            g.C = buf + ntasks * (sa + sb) + t * sc;
            t1[t] = g;
            g.C = buf + ntasks * (sa + sb + sc) + t * sc;
            t2[t] = g;
            pre[t] = tiles;
            tiles += h2l::gemm_tiles(M, N);
        }
        h2l::GemmTask *d1, *d2; int *dp;
        CK(cudaMalloc(&d1, sizeof(h2l::GemmTask) * ntasks));
        CK(cudaMalloc(&d2, sizeof(h2l::GemmTask) * ntasks));
        CK(cudaMalloc(&dp, sizeof(int) * ntasks));
        CK(cudaMemcpy(d1, t1.data(), sizeof(h2l::GemmTask) * ntasks, cudaMemcpyHostToDevice));
        CK(cudaMemcpy(d2, t2.data(), sizeof(h2l::GemmTask) * ntasks, cudaMemcpyHostToDevice));
        CK(cudaMemcpy(dp, pre.data(), sizeof(int) * ntasks, cudaMemcpyHostToDevice));
        // both C copies start equal (copy C1 -> C2)
        for (int z = 0; z < nshift; ++z)
            CK(cudaMemcpyAsync(buf + z * per + ntasks * (sa + sb + sc), buf + z * per + ntasks * (sa + sb),
                               sizeof(double) * sc * ntasks, cudaMemcpyDeviceToDevice, st));
        CK(cudaStreamSynchronize(st));
        double md = 0.0;
        for (int r = 0; r < reps; ++r) {
            h2l::launch_gemm(d1, dp, ntasks, tiles, nshift, st);
            cudaError_t e1 = cudaGetLastError();
            h2l::naive_gemm_kernel<<<dim3(ntasks, nshift), 256, 0, st>>>(d2, ntasks);
            cudaError_t e2 = cudaGetLastError();
            cudaError_t e3 = cudaStreamSynchronize(st);
            if (e1 || e2 || e3)
                fprintf(stderr, "LAUNCH rep %d: gemm=%s naive=%s sync=%s\n", r, cudaGetErrorString(e1),
                        cudaGetErrorString(e2), cudaGetErrorString(e3));
        }
        std::vector<double> c1(sc * ntasks * nshift), c2(sc * ntasks * nshift);
        for (int z = 0; z < nshift; ++z) {
            CK(cudaMemcpy(c1.data() + z * sc * ntasks, buf + z * per + ntasks * (sa + sb),
                          sizeof(double) * sc * ntasks, cudaMemcpyDeviceToHost));
            CK(cudaMemcpy(c2.data() + z * sc * ntasks, buf + z * per + ntasks * (sa + sb + sc),
                          sizeof(double) * sc * ntasks, cudaMemcpyDeviceToHost));
        }
        int64_t nbad = 0;
        for (size_t q = 0; q < c1.size(); ++q) {
            const double d = std::fabs(c1[q] - c2[q]);
            md = std::max(md, d);
            if (d > 1e-9) {
                if (nbad < 12) {
                    const int64_t z = q / (sc * ntasks), rem = q % (sc * ntasks);
                    const int64_t t = rem / sc, e = rem % sc;
                    fprintf(stderr, "BAD z=%lld task=%lld r=%lld c=%lld got=%g want=%g\n", (long long)z,
                            (long long)t, (long long)(e / N), (long long)(e % N), c1[q], c2[q]);
                }
                ++nbad;
            }
        }
        if (nbad) fprintf(stderr, "BAD total %lld of %zu\n", (long long)nbad, c1.size());
        *maxdiff_out = md;
        cudaFree(buf); cudaFree(d1); cudaFree(d2); cudaFree(dp);
        cudaStreamDestroy(st);
    });
}

// INT8-tensor-core (Ozaki) Schur update on dense inputs through the production
// epilogue: one segment whose target is C itself, so for each of `nshift` shifts
// C -= X Bg^T (X, Bg: R x K row-major, host, shift-major; C: R x R, host) on the upper
// triangle and, the segment being diagonal, the mirrored lower triangle.  reps > 0
// times `reps` further launches (split + GEMM, C keeps accumulating) -> mean ms.
extern "C" int h2l_internal_schur_oz(int device, int R, int K, int nshift, const double *X,
                                     const double *Bg, double *C, int reps, double *ms_out,
                                     int probe) {
    return guarded(nullptr, [&] {
        CK(cudaSetDevice(device));
        const int64_t rk = (int64_t)R * K, rr = (int64_t)R * R;
        const int rpad = (R + 127) / 128 * 128, kpad = (K + 63) / 64 * 64;
        double *dx, *db, *dc;
        CK(cudaMalloc(&dx, sizeof(double) * rk * nshift));
        CK(cudaMalloc(&db, sizeof(double) * rk * nshift));
        CK(cudaMalloc(&dc, sizeof(double) * rr * nshift));
        CK(cudaMemcpy(dx, X, sizeof(double) * rk * nshift, cudaMemcpyHostToDevice));
        CK(cudaMemcpy(db, Bg, sizeof(double) * rk * nshift, cudaMemcpyHostToDevice));
        CK(cudaMemcpy(dc, C, sizeof(double) * rr * nshift, cudaMemcpyHostToDevice));
        std::vector<int> seg(R, 0);
        int start0 = 0;
        h2l::SchurTarget tgt{dc, rr, R, 0};
        int *dseg, *dstart;
        h2l::SchurTarget *dtbl;
        CK(cudaMalloc(&dseg, sizeof(int) * std::max(1, R)));
        CK(cudaMalloc(&dstart, sizeof(int)));
        CK(cudaMalloc(&dtbl, sizeof(tgt)));
        CK(cudaMemcpy(dseg, seg.data(), sizeof(int) * R, cudaMemcpyHostToDevice));
        CK(cudaMemcpy(dstart, &start0, sizeof(int), cudaMemcpyHostToDevice));
        CK(cudaMemcpy(dtbl, &tgt, sizeof(tgt), cudaMemcpyHostToDevice));
        h2l::OzJob jb{};
        jb.X = dx; jb.Bg = db; jb.sx = rk; jb.ld = K; jb.R = R; jb.K = K; jb.nseg = 1;
        jb.seg_of = dseg; jb.seg_start = dstart; jb.tbl = dtbl;
        jb.row0 = 0; jb.tile0 = 0;
        const int tiles = h2l::schur_oz_tiles(R);
        std::vector<int> row_job(rpad / 128, 0);
        std::vector<int2> tile_ij;
        h2l::schur_oz_tile_order(R, 0, tile_ij);
        h2l::OzJob *djob; int *drj; int2 *dtj; void *scratch;
        CK(cudaMalloc(&djob, sizeof(jb)));
        CK(cudaMalloc(&drj, sizeof(int) * row_job.size()));
        CK(cudaMalloc(&dtj, sizeof(int2) * std::max(1, tiles)));
        CK(cudaMalloc(&scratch, h2l::schur_oz_scratch_bytes(rpad, kpad, nshift)));
        CK(cudaMemcpy(djob, &jb, sizeof(jb), cudaMemcpyHostToDevice));
        CK(cudaMemcpy(drj, row_job.data(), sizeof(int) * row_job.size(), cudaMemcpyHostToDevice));
        CK(cudaMemcpy(dtj, tile_ij.data(), sizeof(int2) * tiles, cudaMemcpyHostToDevice));
        CK(h2l::launch_schur_oz(djob, drj, dtj, rpad, kpad, tiles, nshift, scratch, 0));
        CK(cudaDeviceSynchronize());
        CK(cudaMemcpy(C, dc, sizeof(double) * rr * nshift, cudaMemcpyDeviceToHost));
        if (reps > 0 && ms_out) {
            cudaEvent_t e0, e1;
            CK(cudaEventCreate(&e0));
            CK(cudaEventCreate(&e1));
            CK(cudaEventRecord(e0));
            for (int q = 0; q < reps; ++q)
                CK(h2l::launch_schur_oz(djob, drj, dtj, rpad, kpad, tiles, nshift, scratch, 0, probe));
            CK(cudaEventRecord(e1));
            CK(cudaEventSynchronize(e1));
            float ms = 0.f;
            CK(cudaEventElapsedTime(&ms, e0, e1));
            *ms_out = ms / reps;
            cudaEventDestroy(e0);
            cudaEventDestroy(e1);
        }
        for (void *p : {(void *)dx, (void *)db, (void *)dc, (void *)djob, (void *)drj, (void *)dtj,
                        scratch, (void *)dseg, (void *)dstart, (void *)dtbl})
            cudaFree(p);
    });
}

// phase counters of schur_oz_kernel under probe 8 (H2L_OZ_PROBE=8 in the engine)
extern "C" int h2l_internal_oz_prof(unsigned long long *out16, int reset) {
    return guarded(nullptr, [&] { h2l::oz_prof_fetch(out16, reset != 0); });
}

// ---- tcgen05 INT8 MMA issue-rate probe: one CTA per SM issues `count` MMAs of shape
// M=128 x N=n x K=32 (SWIZZLE_32B K-major operands, zeroed shared memory) from one
// thread and reports cycles per MMA.  order 0: runs of 8 MMAs into the same
// accumulator; 1: consecutive MMAs rotate over accumulators.
#include "tcgen05.cuh"
namespace h2l {
__global__ void umma_rate_kernel(int n, int order, int count, long long *cycles) {
    using namespace tc;
    extern __shared__ __align__(1024) unsigned char sm_raw[];
    unsigned char *sm = (unsigned char *)(((uintptr_t)sm_raw + 1023) & ~(uintptr_t)1023);
    __shared__ uint32_t slot;
    __shared__ __align__(8) uint64_t bar;
    for (int q = threadIdx.x; q < 96 * 1024 / 16; q += blockDim.x) ((int4 *)sm)[q] = make_int4(0, 0, 0, 0);
    if (threadIdx.x < 32) {
        asm volatile("tcgen05.alloc.cta_group::1.sync.aligned.shared::cta.b32 [%0], 512;" ::"r"(su32(&slot)) : "memory");
        asm volatile("tcgen05.relinquish_alloc_permit.cta_group::1.sync.aligned;" ::: "memory");
    }
    if (threadIdx.x == 0) {
        mbar_init(&bar, 1);
        asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
    }
    asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
    tc_fence_before();
    __syncthreads();
    tc_fence_after();
    const uint32_t tmem = slot;
    if (threadIdx.x == 0) {
        auto sdesc32 = [](uint32_t a) {
            uint64_t d = (uint64_t)((a >> 4) & 0x3FFF) | ((uint64_t)1 << 16) | ((uint64_t)16 << 32) |
                         ((uint64_t)1 << 46) | ((uint64_t)6 << 61);
            return d;
        };
        const uint32_t idesc = (2u << 4) | (1u << 7) | (1u << 10) | ((uint32_t)(n >> 3) << 17) |
                               ((uint32_t)(128 >> 4) << 24);
        const int nacc = 512 / n;
        const uint32_t a0 = su32(sm), b0 = a0 + 8 * 4096;
        const long long t0 = clock64();
        for (int c = 0; c < count; ++c) {
            const int g = order == 0 ? (c / 8) % nacc : c % nacc;
            mma_i8(tmem + g * n, sdesc32(a0 + (c & 7) * 4096), sdesc32(b0 + (c & 7) * (n * 32)), idesc, 1);
        }
        tc_commit(&bar);
        mbar_wait(&bar, 0);
        cycles[blockIdx.x] = clock64() - t0;
    }
    tc_fence_before();
    __syncthreads();
    if (threadIdx.x < 32) {
        tc_fence_after();
        asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, 512;" ::"r"(tmem) : "memory");
    }
}
}  // namespace h2l

extern "C" int h2l_internal_umma_rate(int device, int n, int order, int count, double *cyc_per_mma) {
    return guarded(nullptr, [&] {
        CK(cudaSetDevice(device));
        int nsm = 0;
        CK(cudaDeviceGetAttribute(&nsm, cudaDevAttrMultiProcessorCount, device));
        long long *d;
        CK(cudaMalloc(&d, sizeof(long long) * nsm));
        const int smem = 96 * 1024 + 1024 + 8 * 256 * 32;
        CK(cudaFuncSetAttribute(h2l::umma_rate_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, 200 * 1024));
        h2l::umma_rate_kernel<<<nsm, 128, 200 * 1024>>>(n, order, count, d);
        (void)smem;
        CK(cudaGetLastError());
        CK(cudaDeviceSynchronize());
        std::vector<long long> h(nsm);
        CK(cudaMemcpy(h.data(), d, sizeof(long long) * nsm, cudaMemcpyDeviceToHost));
        double mx = 0;
        for (auto v : h) mx = std::max(mx, (double)v);
        *cyc_per_mma = mx / count;
        cudaFree(d);
    });
}
