// Batched Bunch-Kaufman LDL^T with fused inertia count (K2 + K3).
//
// Restates the reference's native kernel `_core.bk_factor`
// (_core/_kernels.pyx:21-125: dsytf2 lower, alpha = (1+sqrt(17))/8,
// symmetric interchange on the lower triangle, 1x1 and 2x2 pivots, singular
// test |d| <= tol or |det| <= tol*max|block|) and `inertia_of`
// (dense.py:127-168: zero_tol = 1e3*eps*max|D|, 2x2 blocks by det/trace).
//
// One CTA factors one (block, shift).  The lower triangle is held packed and
// column-major (column j contiguous from row j) in shared memory when
// n <= BK_SMEM_MAX (201,600 B at n = 224), else in an L2-resident global
// scratch.  Every column step is: block arg-max reduction (first index on
// ties, as the scalar loop), optional row-max, uniform pivot decision,
// parallel swap, parallel rank-1/rank-2 update of the trailing lower
// triangle with warps over columns and lanes over rows.
//
// Arithmetic is done with explicitly rounded __dmul_rn/__dsub_rn/__dadd_rn
// in the reference's operation order (the reference is compiled without FMA
// contraction), so the packed factor and ipiv are bit-identical to the
// reference kernel (tests/test_bk_gpu.py against tests/golden/bk_random.npz).
//
// Engine mode additionally applies each interchange to the finished L
// columns and records the permutation (what the reference's _unpack does on
// the host, dense.py:72-107), leaving an explicit unit-lower L for the panel.
#include <cfloat>
#include "common.cuh"

namespace h2l {

constexpr int BK_SMEM_MAX = 224;
constexpr int BK_THREADS = 512;

namespace {

struct Packed {
    double *p;
    int n;
    __device__ __forceinline__ double &at(int i, int j) const {  // i >= j
        return p[(int64_t)j * n - ((int64_t)j * (j - 1)) / 2 + (i - j)];
    }
};

struct ArgMax {
    double v;
    int i;
};

__device__ __forceinline__ ArgMax better(ArgMax a, ArgMax b) {
    if (b.v > a.v || (b.v == a.v && b.i < a.i)) return b;
    return a;
}

// block-wide arg-max; result broadcast through smem
__device__ ArgMax block_argmax(ArgMax mine, ArgMax *red) {
    const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
#pragma unroll
    for (int off = 16; off; off >>= 1) {
        ArgMax o;
        o.v = __shfl_down_sync(0xffffffffu, mine.v, off);
        o.i = __shfl_down_sync(0xffffffffu, mine.i, off);
        mine = better(mine, o);
    }
    if (lane == 0) red[warp] = mine;
    __syncthreads();
    if (warp == 0) {
        ArgMax x = lane < (int)(blockDim.x >> 5) ? red[lane] : ArgMax{0.0, 0x7fffffff};
#pragma unroll
        for (int off = 16; off; off >>= 1) {
            ArgMax o;
            o.v = __shfl_down_sync(0xffffffffu, x.v, off);
            o.i = __shfl_down_sync(0xffffffffu, x.i, off);
            x = better(x, o);
        }
        if (lane == 0) red[32] = x;
    }
    __syncthreads();
    ArgMax r = red[32];
    __syncthreads();
    return r;
}

__device__ double block_max(double v, double *red) {
    const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
#pragma unroll
    for (int off = 16; off; off >>= 1) v = fmax(v, __shfl_down_sync(0xffffffffu, v, off));
    if (lane == 0) red[warp] = v;
    __syncthreads();
    if (warp == 0) {
        double x = lane < (int)(blockDim.x >> 5) ? red[lane] : 0.0;
#pragma unroll
        for (int off = 16; off; off >>= 1) x = fmax(x, __shfl_down_sync(0xffffffffu, x, off));
        if (lane == 0) red[32] = x;
    }
    __syncthreads();
    double r = red[32];
    __syncthreads();
    return r;
}

struct BkOut {
    int info;  // 0 or k+1
};

// Factor the packed matrix A (n x n) in place.  w0/w1: n-entry scratch.
// perm != nullptr: engine mode (swap finished L rows, record permutation).
// ipiv/dinfo may be nullptr.
__device__ int bk_core(Packed A, int n, double tol, double *w0, double *w1, int *perm,
                       int64_t *ipiv, double *dinfo, double *red_d, ArgMax *red_a) {
    const double alpha = (1.0 + sqrt(17.0)) / 8.0;
    const int tid = threadIdx.x, nthr = blockDim.x;
    const int lane = tid & 31, warp = tid >> 5, nwarp = nthr >> 5;
    int k = 0;
    while (k < n) {
        // ---- column max below the diagonal
        ArgMax mine{0.0, 0x7fffffff};
        for (int i = k + 1 + tid; i < n; i += nthr) {
            double v = fabs(A.at(i, k));
            if (v > mine.v) { mine.v = v; mine.i = i; }
        }
        ArgMax cm = block_argmax(mine, red_a);
        const double colmax = cm.v;
        const int imax = cm.v > 0.0 ? cm.i : k;
        const double absakk = fabs(A.at(k, k));
        int kp, kstep = 1;
        if (absakk >= __dmul_rn(alpha, colmax)) {
            kp = k;
        } else {
            double r = 0.0;
            for (int j = k + tid; j < imax; j += nthr) r = fmax(r, fabs(A.at(imax, j)));
            for (int i = imax + 1 + tid; i < n; i += nthr) r = fmax(r, fabs(A.at(i, imax)));
            const double rowmax = block_max(r, red_d);
            if (__dmul_rn(absakk, rowmax) >= __dmul_rn(__dmul_rn(alpha, colmax), colmax)) {
                kp = k;
            } else if (fabs(A.at(imax, imax)) >= __dmul_rn(alpha, rowmax)) {
                kp = imax;
            } else {
                kp = imax;
                kstep = 2;
            }
        }
        const int kk = k + kstep - 1;
        if (kp != kk) {
            for (int i = kp + 1 + tid; i < n; i += nthr) {
                double t = A.at(i, kk); A.at(i, kk) = A.at(i, kp); A.at(i, kp) = t;
            }
            for (int j = kk + 1 + tid; j < kp; j += nthr) {
                double t = A.at(j, kk); A.at(j, kk) = A.at(kp, j); A.at(kp, j) = t;
            }
            if (tid == 0) {
                double t = A.at(kk, kk); A.at(kk, kk) = A.at(kp, kp); A.at(kp, kp) = t;
                if (kstep == 2) { t = A.at(kk, k); A.at(kk, k) = A.at(kp, k); A.at(kp, k) = t; }
                if (perm) { int q = perm[kk]; perm[kk] = perm[kp]; perm[kp] = q; }
            }
            if (perm) {  // apply the interchange to the finished columns of L
                for (int j = tid; j < k; j += nthr) {
                    double t = A.at(kk, j); A.at(kk, j) = A.at(kp, j); A.at(kp, j) = t;
                }
            }
        }
        __syncthreads();
        if (kstep == 1) {
            const double d = A.at(k, k);
            if (fabs(d) <= tol) return k + 1;
            const double r1 = 1.0 / d;
            for (int j = k + 1 + warp; j < n; j += nwarp) {
                const double wj = __dmul_rn(r1, A.at(j, k));
                for (int i = j + lane; i < n; i += 32)
                    A.at(i, j) = __dsub_rn(A.at(i, j), __dmul_rn(A.at(i, k), wj));
            }
            __syncthreads();
            for (int i = k + 1 + tid; i < n; i += nthr) A.at(i, k) = __dmul_rn(A.at(i, k), r1);
            if (tid == 0) {
                if (ipiv) ipiv[k] = kp;
                if (dinfo) { dinfo[3 * k] = d; dinfo[3 * k + 1] = 0.0; dinfo[3 * k + 2] = 1.0; }
            }
        } else {
            const double a11 = A.at(k, k), a22 = A.at(k + 1, k + 1);
            double d21 = A.at(k + 1, k);
            const double det = __dsub_rn(__dmul_rn(a11, a22), __dmul_rn(d21, d21));
            double bmax = fabs(d21);
            if (fabs(a11) > bmax) bmax = fabs(a11);
            if (fabs(a22) > bmax) bmax = fabs(a22);
            if (fabs(det) <= __dmul_rn(tol, bmax)) return k + 1;
            if (k < n - 2) {
                const double d11 = a22 / d21;
                const double d22 = a11 / d21;
                const double t = 1.0 / __dsub_rn(__dmul_rn(d11, d22), 1.0);
                d21 = t / d21;
                for (int j = k + 2 + tid; j < n; j += nthr) {
                    const double ajk = A.at(j, k), ajk1 = A.at(j, k + 1);
                    w0[j] = __dmul_rn(d21, __dsub_rn(__dmul_rn(d11, ajk), ajk1));
                    w1[j] = __dmul_rn(d21, __dsub_rn(__dmul_rn(d22, ajk1), ajk));
                }
                __syncthreads();
                for (int j = k + 2 + warp; j < n; j += nwarp) {
                    const double wk = w0[j], wk1 = w1[j];
                    for (int i = j + lane; i < n; i += 32) {
                        const double s = __dadd_rn(__dmul_rn(A.at(i, k), wk),
                                                   __dmul_rn(A.at(i, k + 1), wk1));
                        A.at(i, j) = __dsub_rn(A.at(i, j), s);
                    }
                }
                __syncthreads();
                for (int j = k + 2 + tid; j < n; j += nthr) {
                    A.at(j, k) = w0[j];
                    A.at(j, k + 1) = w1[j];
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
        k += kstep;
    }
    return 0;
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


// Engine mode: jobs x shifts, explicit L + perm + dinfo + counts.
__global__ void __launch_bounds__(BK_THREADS) bk_engine_kernel(const BkJob *jobs, int nmax,
                                                               long long *counts, int *status,
                                                               double *scratch,
                                                               int64_t scratch_stride,
                                                               int use_smem) {
    extern __shared__ __align__(16) double smem[];
    __shared__ double red_d[40];
    __shared__ ArgMax red_a[40];
    __shared__ int s_info;
    const BkJob jb = jobs[blockIdx.x];
    const int z = blockIdx.y;
    const int n = jb.n;
    if (n <= 0) return;
    double *a = jb.a + z * jb.astride;
    int *perm = jb.perm + z * jb.pstride;
    double *dinfo = jb.dinfo + 3 * z * jb.pstride;
    double *wbuf = smem + (use_smem ? (int64_t)nmax * (nmax + 1) / 2 : 0);
    double *store = use_smem ? smem
                             : scratch + ((int64_t)blockIdx.y * gridDim.x + blockIdx.x) *
                                             scratch_stride;
    Packed A{store, n};
    // tolerance from max |entry| of the full leading n x n block (dense.py:50-53)
    double m = 0.0;
    for (int64_t q = threadIdx.x; q < (int64_t)n * n; q += blockDim.x)
        m = fmax(m, fabs(a[(q / n) * jb.ld + q % n]));
    const double amax = block_max(m, red_d);
    const double tol = 1e3 * DBL_EPSILON * amax;
    // load lower triangle (row-major global -> packed column-major)
    for (int i = threadIdx.x >> 5; i < n; i += blockDim.x >> 5)
        for (int j = threadIdx.x & 31; j <= i; j += 32) A.at(i, j) = a[(int64_t)i * jb.ld + j];
    for (int i = threadIdx.x; i < n; i += blockDim.x) perm[i] = i;
    __syncthreads();
    int info = bk_core(A, n, tol, wbuf, wbuf + n, perm, nullptr, dinfo, red_d, red_a);
    if (threadIdx.x == 0) s_info = info;
    __syncthreads();
    info = s_info;
    // write back explicit L / D (lower triangle)
    for (int i = threadIdx.x >> 5; i < n; i += blockDim.x >> 5)
        for (int j = threadIdx.x & 31; j <= i; j += 32) a[(int64_t)i * jb.ld + j] = A.at(i, j);
    if (info) {
        if (threadIdx.x == 0) atomicOr(status + z, 1);
        return;
    }
    // zero tolerance from max |D| (dense.py:134-136) and counts
    double dm = 0.0;
    for (int k = threadIdx.x; k < n; k += blockDim.x)
        dm = fmax(dm, fmax(fabs(dinfo[3 * k]), fabs(dinfo[3 * k + 1])));
    const double dmax = block_max(dm, red_d);
    if (threadIdx.x == 0) {
        long long c[3];
        count_inertia(dinfo, n, 1e3 * DBL_EPSILON * dmax, c);
        atomicAdd((unsigned long long *)(counts + 3 * z + 0), (unsigned long long)c[0]);
        atomicAdd((unsigned long long *)(counts + 3 * z + 1), (unsigned long long)c[1]);
        atomicAdd((unsigned long long *)(counts + 3 * z + 2), (unsigned long long)c[2]);
    }
}

// KAT mode (the reference contract): matrix q of `count`, packed output in place.
__global__ void __launch_bounds__(BK_THREADS) bk_kat_kernel(double *a, int n, const double *tol,
                                                            int64_t *ipiv, int64_t *info,
                                                            double *scratch) {
    extern __shared__ __align__(16) double smem[];
    __shared__ double red_d[40];
    __shared__ ArgMax red_a[40];
    const int q = blockIdx.x;
    double *aq = a + (int64_t)q * n * n;
    const bool use_smem = n <= BK_SMEM_MAX;
    double *wbuf = smem + (use_smem ? (int64_t)n * (n + 1) / 2 : 0);
    double *store = use_smem ? smem : scratch + (int64_t)q * n * (n + 1) / 2;
    Packed A{store, n};
    for (int i = threadIdx.x >> 5; i < n; i += blockDim.x >> 5)
        for (int j = threadIdx.x & 31; j <= i; j += 32) A.at(i, j) = aq[(int64_t)i * n + j];
    __syncthreads();
    int r = bk_core(A, n, tol[q], wbuf, wbuf + n, nullptr, ipiv + (int64_t)q * n, nullptr, red_d,
                    red_a);
    __syncthreads();
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

size_t bk_smem_bytes(int n) {
    if (n <= BK_SMEM_MAX) return sizeof(double) * ((size_t)n * (n + 1) / 2 + 2 * (size_t)n);
    return sizeof(double) * 2 * (size_t)n;
}

}  // namespace

int64_t bk_scratch_doubles(int n) {
    return n <= BK_SMEM_MAX ? 0 : ((int64_t)n * (n + 1) / 2 + 31) / 32 * 32;
}

cudaError_t launch_bk_engine(const BkJob *dev_jobs, int njobs, int nshift, int nmax,
                             int64_t *counts, int *status, double *scratch,
                             int64_t scratch_stride, cudaStream_t st) {
    if (njobs <= 0 || nshift <= 0 || nmax <= 0) return cudaSuccess;
    size_t sm = bk_smem_bytes(nmax);
    cudaError_t e = cudaFuncSetAttribute(bk_engine_kernel,
                                         cudaFuncAttributeMaxDynamicSharedMemorySize, (int)sm);
    if (e != cudaSuccess) return e;
    dim3 grid(njobs, nshift);
    bk_engine_kernel<<<grid, BK_THREADS, sm, st>>>(dev_jobs, nmax, (long long *)counts, status,
                                                   scratch, scratch_stride,
                                                   nmax <= BK_SMEM_MAX ? 1 : 0);
    return cudaGetLastError();
}

cudaError_t launch_bk_kat(double *a, int n, int count, const double *tol, int64_t *ipiv,
                          int64_t *info, double *scratch, cudaStream_t st) {
    if (count <= 0 || n <= 0) return cudaSuccess;
    size_t sm = bk_smem_bytes(n);
    cudaError_t e = cudaFuncSetAttribute(bk_kat_kernel,
                                         cudaFuncAttributeMaxDynamicSharedMemorySize, (int)sm);
    if (e != cudaSuccess) return e;
    bk_kat_kernel<<<count, BK_THREADS, sm, st>>>(a, n, tol, ipiv, info, scratch);
    return cudaGetLastError();
}

cudaError_t launch_bk_inertia(const double *a, int n, int count, const int64_t *ipiv,
                              const double *zero_tol, int64_t *counts, cudaStream_t st) {
    if (count <= 0 || n <= 0) return cudaSuccess;
    bk_inertia_kernel<<<count, 32, 0, st>>>(a, n, ipiv, zero_tol, counts);
    return cudaGetLastError();
}

}  // namespace h2l
