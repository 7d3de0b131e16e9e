// Batched Bunch-Kaufman LDL^T with fused inertia count (K2 + K3).
//
// Restates the reference's native kernel `_core.bk_factor`
// (_core/_kernels.pyx:21-125: dsytf2 lower, alpha = (1+sqrt(17))/8,
// symmetric interchange on the lower triangle, 1x1 and 2x2 pivots, singular
// test |d| <= tol or |det| <= tol*max|block|) and `inertia_of`
// (dense.py:127-168: zero_tol = 1e3*eps*max|D|, 2x2 blocks by det/trace).
//
// One CTA factors one (block, shift).  The lower triangle is held packed and
// column-major (column j contiguous from row j, start offsets in a table) in
// shared memory when n <= BK_SMEM_MAX (201,600 B at n = 224), else in an
// L2-resident global scratch.  One column step costs two block barriers:
//   [finish previous pivot: deferred column scaling / 2x2 L write-back]
//   [pivot decision from the column arg-max computed in the previous step;
//    row-max reduction only when the 1x1 test fails]
//   swap  | barrier | rank-1/rank-2 update, warps over columns, lanes over
//   rows; warp 0 owns the next pivot column and reduces its arg-max as it
//   updates it | barrier
// The interchanges of finished L columns that the reference's _unpack
// applies on the host (dense.py:72-107) are replayed once at the end (engine
// mode), leaving an explicit unit-lower L and the permutation.
//
// Arithmetic uses explicitly rounded __dmul_rn/__dsub_rn/__dadd_rn in the
// reference's operation order (the reference is compiled without FMA
// contraction), so the packed factor and ipiv are bit-identical to the
// reference kernel (tests/test_gpu_engine.py against tests/golden/bk_random.npz).
#include <cfloat>
#include "common.cuh"

namespace h2l {

constexpr int BK_SMEM_MAX = 224;
constexpr int BK_THREADS = 256;
constexpr int BK_NMAX = 4096;

namespace {

struct Packed {
    double *p;
    const int *cs;  // column start offsets: element (i, j), i >= j, at p[cs[j] + i]
    __device__ __forceinline__ double &at(int i, int j) const { return p[cs[j] + i]; }
};

struct ArgMax {
    double v;
    int i;
};

__device__ __forceinline__ ArgMax better(ArgMax a, ArgMax b) {
    if (b.v > a.v || (b.v == a.v && b.i < a.i)) return b;
    return a;
}

__device__ __forceinline__ ArgMax warp_argmax(ArgMax x) {
#pragma unroll
    for (int off = 16; off; off >>= 1) {
        ArgMax o;
        o.v = __shfl_xor_sync(0xffffffffu, x.v, off);
        o.i = __shfl_xor_sync(0xffffffffu, x.i, off);
        x = better(x, o);
    }
    return x;
}

__device__ ArgMax block_argmax(ArgMax mine, ArgMax *red) {
    const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
    mine = warp_argmax(mine);
    if (lane == 0) red[warp] = mine;
    __syncthreads();
    ArgMax x = lane < (int)(blockDim.x >> 5) ? red[lane] : ArgMax{0.0, 0x7fffffff};
    x = warp_argmax(x);
    __syncthreads();
    return x;
}

__device__ double block_max(double v, double *red) {
    const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
#pragma unroll
    for (int off = 16; off; off >>= 1) v = fmax(v, __shfl_xor_sync(0xffffffffu, v, off));
    if (lane == 0) red[warp] = v;
    __syncthreads();
    double x = lane < (int)(blockDim.x >> 5) ? red[lane] : 0.0;
#pragma unroll
    for (int off = 16; off; off >>= 1) x = fmax(x, __shfl_xor_sync(0xffffffffu, x, off));
    __syncthreads();
    return x;
}

struct BkShared {
    ArgMax red_a[32];
    double red_d[32];
    ArgMax next;      // arg-max of the next pivot column (rows below its diagonal)
    int info;
};

// Rank-1 update of the trailing lower triangle for a 1x1 pivot at column k,
// rows owned by lane (i = lane + 32 t), pivot column cached in registers.
// Returns (in nx, warp 0 only) the arg-max of the updated column k+1.
template <int NT>
__device__ __forceinline__ void update1(Packed A, int n, int k, double r1, ArgMax &nx) {
    const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5, nwarp = blockDim.x >> 5;
    double ak[NT];
#pragma unroll
    for (int t = 0; t < NT; ++t) {
        const int i = lane + 32 * t;
        ak[t] = (i > k && i < n) ? A.at(i, k) : 0.0;
    }
    for (int j = k + 1 + warp; j < n; j += nwarp) {
        const double wj = __dmul_rn(r1, A.at(j, k));
        double *col = A.p + A.cs[j];
        double v[NT];
#pragma unroll
        for (int t = 0; t < NT; ++t) {
            const int i = lane + 32 * t;
            if (i >= j && i < n) v[t] = col[i];
        }
#pragma unroll
        for (int t = 0; t < NT; ++t) {
            const int i = lane + 32 * t;
            if (i >= j && i < n) {
                v[t] = __dsub_rn(v[t], __dmul_rn(ak[t], wj));
                col[i] = v[t];
            }
        }
        if (j == k + 1) {
#pragma unroll
            for (int t = 0; t < NT; ++t) {
                const int i = lane + 32 * t;
                if (i > j && i < n && fabs(v[t]) > nx.v) { nx.v = fabs(v[t]); nx.i = i; }
            }
        }
    }
}

// Rank-2 update for a 2x2 pivot at columns k, k+1 (w0/w1 receive the new L columns).
template <int NT>
__device__ __forceinline__ void update2(Packed A, int n, int k, double d11, double d22,
                                        double d21, double *w0, double *w1, ArgMax &nx) {
    const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5, nwarp = blockDim.x >> 5;
    double ak[NT], ak1[NT];
#pragma unroll
    for (int t = 0; t < NT; ++t) {
        const int i = lane + 32 * t;
        const bool ok = i > k + 1 && i < n;
        ak[t] = ok ? A.at(i, k) : 0.0;
        ak1[t] = ok ? A.at(i, k + 1) : 0.0;
    }
    for (int j = k + 2 + warp; j < n; j += nwarp) {
        const double ajk = A.at(j, k), ajk1 = A.at(j, k + 1);
        const double wk = __dmul_rn(d21, __dsub_rn(__dmul_rn(d11, ajk), ajk1));
        const double wk1 = __dmul_rn(d21, __dsub_rn(__dmul_rn(d22, ajk1), ajk));
        double *col = A.p + A.cs[j];
        double v[NT];
#pragma unroll
        for (int t = 0; t < NT; ++t) {
            const int i = lane + 32 * t;
            if (i >= j && i < n) v[t] = col[i];
        }
#pragma unroll
        for (int t = 0; t < NT; ++t) {
            const int i = lane + 32 * t;
            if (i >= j && i < n) {
                const double s = __dadd_rn(__dmul_rn(ak[t], wk), __dmul_rn(ak1[t], wk1));
                v[t] = __dsub_rn(v[t], s);
                col[i] = v[t];
            }
        }
        if (lane == 0) { w0[j] = wk; w1[j] = wk1; }
        if (j == k + 2) {
#pragma unroll
            for (int t = 0; t < NT; ++t) {
                const int i = lane + 32 * t;
                if (i > j && i < n && fabs(v[t]) > nx.v) { nx.v = fabs(v[t]); nx.i = i; }
            }
        }
    }
}

// Factor packed A (n x n) in place.  w0/w1: n-entry scratch; swaps: 2n ints.
// perm != nullptr: engine mode (explicit L + permutation).  ipiv/dinfo optional.
__device__ __forceinline__ int bk_core(Packed A, int n, double tol, double *w0, double *w1, int *swaps, int *perm,
                       int64_t *ipiv, double *dinfo, BkShared &sh) {
    const double alpha = (1.0 + sqrt(17.0)) / 8.0;
    const int tid = threadIdx.x, nthr = blockDim.x;
    const int lane = tid & 31, warp = tid >> 5, nwarp = nthr >> 5;
    {   // arg-max of column 0
        ArgMax mine{0.0, 0x7fffffff};
        for (int i = 1 + tid; i < n; i += nthr) {
            const double v = fabs(A.at(i, 0));
            if (v > mine.v) { mine.v = v; mine.i = i; }
        }
        ArgMax r = block_argmax(mine, sh.red_a);
        if (tid == 0) sh.next = r;
        __syncthreads();
    }
    int prev = -1, prev_step = 0;
    double prev_r1 = 0.0;
    int k = 0, info = 0;
    while (k < n) {
        // ---- finish the previous pivot (no reader until the end)
        if (prev_step == 1) {
            for (int i = prev + 1 + tid; i < n; i += nthr) A.at(i, prev) = __dmul_rn(A.at(i, prev), prev_r1);
        } else if (prev_step == 2) {
            for (int j = prev + 2 + tid; j < n; j += nthr) {
                A.at(j, prev) = w0[j];
                A.at(j, prev + 1) = w1[j];
            }
        }
        // ---- pivot decision
        const ArgMax cm = sh.next;
        const double colmax = cm.v;
        const int imax = cm.v > 0.0 ? cm.i : k;
        const double absakk = fabs(A.at(k, k));
        int kp, kstep = 1;
        if (absakk >= __dmul_rn(alpha, colmax)) {
            kp = k;
        } else {
            // every decision input is read before the barrier inside block_max:
            // past it, thread 0 may already be interchanging (kk,kk) <-> (kp,kp)
            const double aii = fabs(A.at(imax, imax));
            double r = 0.0;
            for (int j = k + tid; j < imax; j += nthr) r = fmax(r, fabs(A.at(imax, j)));
            for (int i = imax + 1 + tid; i < n; i += nthr) r = fmax(r, fabs(A.at(i, imax)));
            const double rowmax = block_max(r, sh.red_d);
            if (__dmul_rn(absakk, rowmax) >= __dmul_rn(__dmul_rn(alpha, colmax), colmax)) {
                kp = k;
            } else if (aii >= __dmul_rn(alpha, rowmax)) {
                kp = imax;
            } else {
                kp = imax;
                kstep = 2;
            }
        }
        const int kk = k + kstep - 1;
        if (kp != kk) {
            for (int i = kp + 1 + tid; i < n; i += nthr) {
                const double t = A.at(i, kk); A.at(i, kk) = A.at(i, kp); A.at(i, kp) = t;
            }
            for (int j = kk + 1 + tid; j < kp; j += nthr) {
                const double t = A.at(j, kk); A.at(j, kk) = A.at(kp, j); A.at(kp, j) = t;
            }
            if (tid == 0) {
                double t = A.at(kk, kk); A.at(kk, kk) = A.at(kp, kp); A.at(kp, kp) = t;
                if (kstep == 2) { t = A.at(kk, k); A.at(kk, k) = A.at(kp, k); A.at(kp, k) = t; }
                if (perm) { const int q = perm[kk]; perm[kk] = perm[kp]; perm[kp] = q; }
            }
        }
        if (tid == 0 && swaps) { swaps[2 * k] = kk; swaps[2 * k + 1] = kp; }
        __syncthreads();
        if (kstep == 1) {
            const double d = A.at(k, k);
            if (fabs(d) <= tol) { info = k + 1; break; }
            const double r1 = 1.0 / d;
            ArgMax nx{0.0, 0x7fffffff};
            if (n <= 32) update1<1>(A, n, k, r1, nx);
            else if (n <= 64) update1<2>(A, n, k, r1, nx);
            else if (n <= 128) update1<4>(A, n, k, r1, nx);
            else if (n <= 256) update1<8>(A, n, k, r1, nx);
            else {
                for (int j = k + 1 + warp; j < n; j += nwarp) {
                    const double wj = __dmul_rn(r1, A.at(j, k));
                    for (int i = j + lane; i < n; i += 32) {
                        const double v = __dsub_rn(A.at(i, j), __dmul_rn(A.at(i, k), wj));
                        A.at(i, j) = v;
                        if (j == k + 1 && i > j && fabs(v) > nx.v) { nx.v = fabs(v); nx.i = i; }
                    }
                }
            }
            if (warp == 0 && k + 1 < n) {
                nx = warp_argmax(nx);
                if (lane == 0) sh.next = nx;
            }
            if (tid == 0) {
                if (ipiv) ipiv[k] = kp;
                if (dinfo) { dinfo[3 * k] = d; dinfo[3 * k + 1] = 0.0; dinfo[3 * k + 2] = 1.0; }
            }
            prev_r1 = r1;
        } else {
            const double a11 = A.at(k, k), a22 = A.at(k + 1, k + 1);
            double d21 = A.at(k + 1, k);
            const double det = __dsub_rn(__dmul_rn(a11, a22), __dmul_rn(d21, d21));
            double bmax = fabs(d21);
            if (fabs(a11) > bmax) bmax = fabs(a11);
            if (fabs(a22) > bmax) bmax = fabs(a22);
            if (fabs(det) <= __dmul_rn(tol, bmax)) { info = k + 1; break; }
            if (k < n - 2) {
                const double d11 = a22 / d21;
                const double d22 = a11 / d21;
                const double t = 1.0 / __dsub_rn(__dmul_rn(d11, d22), 1.0);
                d21 = t / d21;
                ArgMax nx{0.0, 0x7fffffff};
                if (n <= 32) update2<1>(A, n, k, d11, d22, d21, w0, w1, nx);
                else if (n <= 64) update2<2>(A, n, k, d11, d22, d21, w0, w1, nx);
                else if (n <= 128) update2<4>(A, n, k, d11, d22, d21, w0, w1, nx);
                else if (n <= 256) update2<8>(A, n, k, d11, d22, d21, w0, w1, nx);
                else {
                    for (int j = k + 2 + warp; j < n; j += nwarp) {
                        const double ajk = A.at(j, k), ajk1 = A.at(j, k + 1);
                        const double wk = __dmul_rn(d21, __dsub_rn(__dmul_rn(d11, ajk), ajk1));
                        const double wk1 = __dmul_rn(d21, __dsub_rn(__dmul_rn(d22, ajk1), ajk));
                        for (int i = j + lane; i < n; i += 32) {
                            const double s = __dadd_rn(__dmul_rn(A.at(i, k), wk),
                                                       __dmul_rn(A.at(i, k + 1), wk1));
                            const double v = __dsub_rn(A.at(i, j), s);
                            A.at(i, j) = v;
                            if (j == k + 2 && i > j && fabs(v) > nx.v) { nx.v = fabs(v); nx.i = i; }
                        }
                        if (lane == 0) { w0[j] = wk; w1[j] = wk1; }
                    }
                }
                if (warp == 0 && k + 2 < n) {
                    nx = warp_argmax(nx);
                    if (lane == 0) sh.next = nx;
                }
            }
            if (tid == 0) {
                if (ipiv) { ipiv[k] = -(kp + 1); ipiv[k + 1] = -(kp + 1); }
                if (dinfo) {
                    dinfo[3 * k] = a11; dinfo[3 * k + 1] = A.at(k + 1, k); dinfo[3 * k + 2] = 2.0;
                    dinfo[3 * k + 3] = a22; dinfo[3 * k + 4] = 0.0; dinfo[3 * k + 5] = 0.0;
                }
            }
        }
        __syncthreads();
        prev = k;
        prev_step = kstep;
        k += kstep;
    }
    // ---- finish the last pivot
    if (!info) {
        if (prev_step == 1) {
            for (int i = prev + 1 + tid; i < n; i += nthr) A.at(i, prev) = __dmul_rn(A.at(i, prev), prev_r1);
        } else if (prev_step == 2) {
            for (int j = prev + 2 + tid; j < n; j += nthr) {
                A.at(j, prev) = w0[j];
                A.at(j, prev + 1) = w1[j];
            }
        }
    }
    __syncthreads();
    // ---- engine mode: replay the interchanges on the finished L columns
    if (perm && !info) {
        for (int c = tid; c < n; c += nthr) {
            for (int s = c + 1; s < n; ++s) {
                const int kk = swaps[2 * s], kp = swaps[2 * s + 1];
                if (kk < 0) continue;  // second column of a 2x2 step
                if (kp != kk) {
                    const double t = A.at(kk, c); A.at(kk, c) = A.at(kp, c); A.at(kp, c) = t;
                }
            }
        }
        __syncthreads();
    }
    return info;
}

// sign counts of the pivot blocks (dense.py:127-168), single thread
__device__ void count_inertia(const double *dinfo, int n, double zt, long long *c) {
    long long neg = 0, zero = 0, pos = 0;
    for (int k = 0; k < n;) {
        if (dinfo[3 * k + 2] < 1.5) {
            const double d = dinfo[3 * k];
            if (fabs(d) <= zt) ++zero; else if (d < 0.0) ++neg; else ++pos;
            k += 1;
        } else {
            const double x = dinfo[3 * k], y = dinfo[3 * k + 3], e = dinfo[3 * k + 1];
            const double det = __dsub_rn(__dmul_rn(x, y), __dmul_rn(e, e));
            const double tr = __dadd_rn(x, y);
            const double zt2 = __dmul_rn(zt, zt);
            if (det < -zt2) { ++neg; ++pos; }
            else if (det > zt2) { if (tr < 0.0) neg += 2; else pos += 2; }
            else {
                ++zero;
                if (tr < -zt) ++neg; else if (tr > zt) ++pos; else ++zero;
            }
            k += 2;
        }
    }
    c[0] = neg; c[1] = zero; c[2] = pos;
}

// dynamic smem: [packed | w0 | w1] doubles, then [cs | swaps] ints
__device__ __forceinline__ void carve(double *smem, int n, bool in_smem, double *scratch, double **store,
                      double **w0, double **w1, int **cs, int **swaps) {
    const int64_t packed = in_smem ? (int64_t)n * (n + 1) / 2 : 0;
    *store = in_smem ? smem : scratch;
    *w0 = smem + packed;
    *w1 = *w0 + n;
    *cs = (int *)(*w1 + n);
    *swaps = *cs + n;
    for (int j = threadIdx.x; j < n; j += blockDim.x) {
        (*cs)[j] = j * n - (j * (j + 1)) / 2;
        (*swaps)[2 * j] = -1;
        (*swaps)[2 * j + 1] = -1;
    }
    __syncthreads();
}

size_t bk_smem_bytes(int n) {
    const size_t packed = n <= BK_SMEM_MAX ? (size_t)n * (n + 1) / 2 : 0;
    return sizeof(double) * (packed + 2 * (size_t)n) + sizeof(int) * 3 * (size_t)n;
}

// Engine mode: jobs x shifts, explicit L + perm + dinfo + counts.
template <bool SMEM>
__global__ void __launch_bounds__(BK_THREADS) bk_engine_kernel(const BkJob *jobs, int nmax,
                                                               long long *counts, int *status,
                                                               double *scratch,
                                                               int64_t scratch_stride) {
    constexpr bool use_smem = SMEM;
    extern __shared__ __align__(16) double smem[];
    __shared__ BkShared sh;
    const BkJob jb = jobs[blockIdx.x];
    const int z = blockIdx.y;
    const int n = jb.n;
    if (n <= 0) return;
    double *a = jb.a + z * jb.astride;
    int *perm = jb.perm + z * jb.pstride;
    double *dinfo = jb.dinfo + 3 * z * jb.pstride;
    double *store, *w0, *w1;
    int *cs, *swaps;
    carve(smem, use_smem ? nmax : n, use_smem,
          scratch + ((int64_t)blockIdx.y * gridDim.x + blockIdx.x) * scratch_stride, &store, &w0,
          &w1, &cs, &swaps);
    // carve() sized the column table for nmax when in smem; rebuild for n
    for (int j = threadIdx.x; j < n; j += blockDim.x) cs[j] = j * n - (j * (j + 1)) / 2;
    __syncthreads();
    Packed A{store, cs};
    // tolerance from max |entry| of the full leading n x n block (dense.py:50-53)
    double m = 0.0;
    for (int i = threadIdx.x >> 5; i < n; i += blockDim.x >> 5)
        for (int j = threadIdx.x & 31; j < n; j += 32) m = fmax(m, fabs(a[(int64_t)i * jb.ld + j]));
    const double amax = block_max(m, sh.red_d);
    const double tol = 1e3 * DBL_EPSILON * amax;
    for (int i = threadIdx.x >> 5; i < n; i += blockDim.x >> 5)
        for (int j = threadIdx.x & 31; j <= i; j += 32) A.at(i, j) = a[(int64_t)i * jb.ld + j];
    for (int i = threadIdx.x; i < n; i += blockDim.x) perm[i] = i;
    __syncthreads();
    const int info = bk_core(A, n, tol, w0, w1, swaps, perm, nullptr, dinfo, sh);
    for (int i = threadIdx.x >> 5; i < n; i += blockDim.x >> 5)
        for (int j = threadIdx.x & 31; j <= i; j += 32) a[(int64_t)i * jb.ld + j] = A.at(i, j);
    if (info) {
        if (threadIdx.x == 0) atomicOr(status + z, 1);
        return;
    }
    double dm = 0.0;
    for (int k = threadIdx.x; k < n; k += blockDim.x)
        dm = fmax(dm, fmax(fabs(dinfo[3 * k]), fabs(dinfo[3 * k + 1])));
    const double dmax = block_max(dm, sh.red_d);
    if (threadIdx.x == 0) {
        long long c[3];
        count_inertia(dinfo, n, 1e3 * DBL_EPSILON * dmax, c);
        atomicAdd((unsigned long long *)(counts + 3 * z + 0), (unsigned long long)c[0]);
        atomicAdd((unsigned long long *)(counts + 3 * z + 1), (unsigned long long)c[1]);
        atomicAdd((unsigned long long *)(counts + 3 * z + 2), (unsigned long long)c[2]);
    }
}

// KAT mode (the reference contract): matrix q of `count`, packed output in place.
template <bool SMEM>
__global__ void __launch_bounds__(BK_THREADS) bk_kat_kernel(double *a, int n, const double *tol,
                                                            int64_t *ipiv, int64_t *info,
                                                            double *scratch) {
    extern __shared__ __align__(16) double smem[];
    __shared__ BkShared sh;
    const int q = blockIdx.x;
    double *aq = a + (int64_t)q * n * n;
    double *store, *w0, *w1;
    int *cs, *swaps;
    constexpr bool in_smem = SMEM;
    carve(smem, n, in_smem, scratch + (int64_t)q * n * (n + 1) / 2, &store, &w0, &w1, &cs, &swaps);
    Packed A{store, cs};
    for (int i = threadIdx.x >> 5; i < n; i += blockDim.x >> 5)
        for (int j = threadIdx.x & 31; j <= i; j += 32) A.at(i, j) = aq[(int64_t)i * n + j];
    __syncthreads();
    const int r = bk_core(A, n, tol[q], w0, w1, nullptr, nullptr, ipiv + (int64_t)q * n, nullptr, sh);
    for (int i = threadIdx.x >> 5; i < n; i += blockDim.x >> 5)
        for (int j = threadIdx.x & 31; j <= i; j += 32) aq[(int64_t)i * n + j] = A.at(i, j);
    if (threadIdx.x == 0) info[q] = r;
}

__global__ void bk_inertia_kernel(const double *a, int n, const int64_t *ipiv,
                                  const double *zero_tol, int64_t *counts) {
    if (threadIdx.x) return;
    const int q = blockIdx.x;
    const double *aq = a + (int64_t)q * n * n;
    const int64_t *ip = ipiv + (int64_t)q * n;
    const double zt = zero_tol[q];
    long long neg = 0, zero = 0, pos = 0;
    for (int k = 0; k < n;) {
        if (ip[k] >= 0) {
            const double d = aq[(int64_t)k * n + k];
            if (fabs(d) <= zt) ++zero; else if (d < 0.0) ++neg; else ++pos;
            k += 1;
        } else {
            const double x = aq[(int64_t)k * n + k], y = aq[(int64_t)(k + 1) * n + k + 1];
            const double e = aq[(int64_t)(k + 1) * n + k];
            const double det = __dsub_rn(__dmul_rn(x, y), __dmul_rn(e, e));
            const double tr = __dadd_rn(x, y);
            const double zt2 = __dmul_rn(zt, zt);
            if (det < -zt2) { ++neg; ++pos; }
            else if (det > zt2) { if (tr < 0.0) neg += 2; else pos += 2; }
            else {
                ++zero;
                if (tr < -zt) ++neg; else if (tr > zt) ++pos; else ++zero;
            }
            k += 2;
        }
    }
    counts[3 * q] = neg; counts[3 * q + 1] = zero; counts[3 * q + 2] = pos;
}

}  // namespace

int64_t bk_scratch_doubles(int n) {
    return n <= BK_SMEM_MAX ? 0 : ((int64_t)n * (n + 1) / 2 + 31) / 32 * 32;
}

cudaError_t launch_bk_engine(const BkJob *dev_jobs, int njobs, int nshift, int nmax,
                             int64_t *counts, int *status, double *scratch,
                             int64_t scratch_stride, cudaStream_t st) {
    if (njobs <= 0 || nshift <= 0 || nmax <= 0) return cudaSuccess;
    if (nmax > BK_NMAX) return cudaErrorInvalidValue;
    const size_t sm = bk_smem_bytes(nmax);
    dim3 grid(njobs, nshift);
    if (nmax <= BK_SMEM_MAX) {
        cudaError_t e = smem_optin(bk_engine_kernel<true>);
        if (e != cudaSuccess) return e;
        bk_engine_kernel<true><<<grid, BK_THREADS, sm, st>>>(dev_jobs, nmax, (long long *)counts,
                                                             status, scratch, scratch_stride);
    } else {
        cudaError_t e = smem_optin(bk_engine_kernel<false>);
        if (e != cudaSuccess) return e;
        bk_engine_kernel<false><<<grid, BK_THREADS, sm, st>>>(dev_jobs, nmax, (long long *)counts,
                                                              status, scratch, scratch_stride);
    }
    return cudaGetLastError();
}

cudaError_t launch_bk_kat(double *a, int n, int count, const double *tol, int64_t *ipiv,
                          int64_t *info, double *scratch, cudaStream_t st) {
    if (count <= 0 || n <= 0) return cudaSuccess;
    if (n > BK_NMAX) return cudaErrorInvalidValue;
    const size_t sm = bk_smem_bytes(n);
    if (n <= BK_SMEM_MAX) {
        cudaError_t e = smem_optin(bk_kat_kernel<true>);
        if (e != cudaSuccess) return e;
        bk_kat_kernel<true><<<count, BK_THREADS, sm, st>>>(a, n, tol, ipiv, info, scratch);
    } else {
        cudaError_t e = smem_optin(bk_kat_kernel<false>);
        if (e != cudaSuccess) return e;
        bk_kat_kernel<false><<<count, BK_THREADS, sm, st>>>(a, n, tol, ipiv, info, scratch);
    }
    return cudaGetLastError();
}

cudaError_t launch_bk_inertia(const double *a, int n, int count, const int64_t *ipiv,
                              const double *zero_tol, int64_t *counts, cudaStream_t st) {
    if (count <= 0 || n <= 0) return cudaSuccess;
    bk_inertia_kernel<<<count, 32, 0, st>>>(a, n, ipiv, zero_tol, counts);
    return cudaGetLastError();
}

}  // namespace h2l
