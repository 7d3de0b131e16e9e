// Recompression rank-reveal for wide fill rows (K7), Gram-ordered, exact tail.
// (engine.cu drives it: M = G G^T, pivoted QR of M for the order, D = Q^T G,
// one deflation pass on the directions the Gram matrix cannot resolve, rank
// from the exact energies of D.)
//
// Reference: gldl.py:67-79 - scipy.linalg.qr(G, pivoting=True) of
// G = [fill rows] (n_R x c, c up to ~10^5 at config 2) and
// rank = first r with ||R[r:, :]||_F <= drop_tol.  A column-pivoted QR of
// such a wide G is a long chain of dependent reflections; here:
//   1. M = G G^T                         (DMMA GEMM, engine.cu)
//   2. pivoted Cholesky of M            pchol_kernel   -> L (greedy order)
//      (= the pivoted QR of G^T: at step j it picks the direction with the
//       largest remaining energy, exactly the rank-revealing greedy choice)
//   3. Householder QR of L              hqr_kernel     -> Q, nested spans
//   4. D = Q^T G                        (DMMA GEMM)
//   5. rank from the exact row energies of D: tail(r) = sqrt(sum_{i>=r}
//      ||D_i||^2) = ||(I - Q_r Q_r^T) G||_F (Q orthogonal), first r with
//      tail(r) <= drop_tol                               tail kernels
// Steps 1-3 only choose the ORDER of the directions (their rounding is
// harmless); the rank test in step 5 uses energies computed directly from G,
// so the dropped part is <= drop_tol as in the reference, for any Q.
#include <algorithm>
#include <cfloat>
#include "common.cuh"

namespace h2l {

namespace {

constexpr int RR_THREADS = 256;

struct ArgMaxD {
    double v;
    int i;
};

__device__ __forceinline__ ArgMaxD better(ArgMaxD a, ArgMaxD b) {
    return (b.v > a.v || (b.v == a.v && b.i < a.i)) ? b : a;
}

__device__ ArgMaxD block_argmax(ArgMaxD x, ArgMaxD *red) {
    const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
#pragma unroll
    for (int off = 16; off; off >>= 1) {
        ArgMaxD o{__shfl_xor_sync(0xffffffffu, x.v, off), __shfl_xor_sync(0xffffffffu, x.i, off)};
        x = better(x, o);
    }
    if (lane == 0) red[warp] = x;
    __syncthreads();
    ArgMaxD y = lane < (int)(blockDim.x >> 5) ? red[lane] : ArgMaxD{-1.0, 0x7fffffff};
#pragma unroll
    for (int off = 16; off; off >>= 1) {
        ArgMaxD o{__shfl_xor_sync(0xffffffffu, y.v, off), __shfl_xor_sync(0xffffffffu, y.i, off)};
        y = better(y, o);
    }
    __syncthreads();
    return y;
}

__device__ double block_sum(double v, double *red) {
    const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
#pragma unroll
    for (int off = 16; off; off >>= 1) v += __shfl_xor_sync(0xffffffffu, v, off);
    if (lane == 0) red[warp] = v;
    __syncthreads();
    double y = lane < (int)(blockDim.x >> 5) ? red[lane] : 0.0;
#pragma unroll
    for (int off = 16; off; off >>= 1) y += __shfl_xor_sync(0xffffffffu, y, off);
    __syncthreads();
    return y;
}

// Pivoted Cholesky of M (n x n, row-major, one shift per CTA) without explicit
// interchanges: column j of L (row-major L[i*n + j], original row order) is the
// j-th greedy pivot.  S: n x n scratch (Schur complement), rem/d in smem.
__global__ void __launch_bounds__(RR_THREADS) pchol_kernel(const double *M, int64_t mstride, int n,
                                                           double *S, double *L,
                                                           const int *active) {
    extern __shared__ double dsm[];
    double *d = dsm;             // n
    int *rem = (int *)(d + n);   // n
    __shared__ ArgMaxD red[32];
    __shared__ double s_piv;
    const int z = blockIdx.x;
    const double *Mz = M + z * mstride;
    double *Sz = S + z * mstride;
    double *Lz = L + z * mstride;
    for (int64_t e = threadIdx.x; e < (int64_t)n * n; e += blockDim.x) {
        Sz[e] = Mz[e];
        Lz[e] = 0.0;
    }
    for (int i = threadIdx.x; i < n; i += blockDim.x) {
        d[i] = Mz[(int64_t)i * n + i];
        rem[i] = 1;
    }
    __syncthreads();
    if (active && !active[z]) return;
    const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5, nwarp = blockDim.x >> 5;
    for (int j = 0; j < n; ++j) {
        ArgMaxD mine{-1.0, 0x7fffffff};
        for (int i = threadIdx.x; i < n; i += blockDim.x)
            if (rem[i] && d[i] > mine.v) { mine.v = d[i]; mine.i = i; }
        const ArgMaxD pv = block_argmax(mine, red);
        if (!(pv.v > 0.0)) break;  // remaining energy exhausted (or rounding noise)
        const int p = pv.i;
        if (threadIdx.x == 0) s_piv = sqrt(pv.v);
        __syncthreads();
        const double piv = s_piv;
        for (int i = threadIdx.x; i < n; i += blockDim.x)
            Lz[(int64_t)i * n + j] = (i == p) ? piv : (rem[i] ? Sz[(int64_t)i * n + p] / piv : 0.0);
        __syncthreads();
        if (threadIdx.x == 0) rem[p] = 0;
        __syncthreads();
        // S[i][k] -= L[i][j] L[k][j] over remaining rows (warps over i, lanes over k)
        for (int i = warp; i < n; i += nwarp) {
            if (!rem[i]) continue;
            const double li = Lz[(int64_t)i * n + j];
            double *srow = Sz + (int64_t)i * n;
            for (int k = lane; k < n; k += 32)
                if (rem[k]) srow[k] -= li * Lz[(int64_t)k * n + j];
        }
        __syncthreads();
        for (int i = threadIdx.x; i < n; i += blockDim.x)
            if (rem[i]) d[i] = Sz[(int64_t)i * n + i];
        __syncthreads();
    }
}

// Householder QR of A (n x n, row-major, one shift per CTA), unpivoted; writes
// QT = Q^T (row q = column q of Q).  W: n x n scratch (column-major copy).
__global__ void __launch_bounds__(RR_THREADS) hqr_kernel(const double *A, int64_t astride, int n,
                                                         double *W, double *QT, double *tau,
                                                         int64_t tstride, const int *active) {
    __shared__ double red[32];
    __shared__ double s_beta, s_tau, s_scale;
    const int z = blockIdx.x;
    const double *Az = A + z * astride;
    double *Wz = W + z * astride;   // Wz[j*n + i] = A[i][j]
    double *Qz = QT + z * astride;
    double *tz = tau + z * tstride;
    const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5, nwarp = blockDim.x >> 5;
    for (int64_t e = threadIdx.x; e < (int64_t)n * n; e += blockDim.x) {
        const int i = (int)(e / n), j = (int)(e % n);
        Wz[(int64_t)j * n + i] = Az[e];
        Qz[e] = (i == j) ? 1.0 : 0.0;
    }
    __syncthreads();
    if (active && !active[z]) return;
    for (int j = 0; j < n; ++j) {
        double *x = Wz + (int64_t)j * n;
        double part = 0.0;
        for (int r = j + 1 + threadIdx.x; r < n; r += blockDim.x) part += x[r] * x[r];
        const double xn2 = block_sum(part, red);
        if (threadIdx.x == 0) {
            const double alpha = x[j];
            if (xn2 == 0.0) {
                s_tau = 0.0; s_beta = alpha; s_scale = 0.0;
            } else {
                const double beta = -copysign(sqrt(alpha * alpha + xn2), alpha);
                s_tau = (beta - alpha) / beta;
                s_scale = 1.0 / (alpha - beta);
                s_beta = beta;
            }
            tz[j] = s_tau;
        }
        __syncthreads();
        const double tj = s_tau;
        for (int r = j + 1 + threadIdx.x; r < n; r += blockDim.x) x[r] *= s_scale;
        __syncthreads();
        if (threadIdx.x == 0) x[j] = s_beta;
        for (int k = j + 1 + warp; k < n; k += nwarp) {
            double *y = Wz + (int64_t)k * n;
            double s = (lane == 0) ? y[j] : 0.0;
            for (int r = j + 1 + lane; r < n; r += 32) s += x[r] * y[r];
#pragma unroll
            for (int off = 16; off; off >>= 1) s += __shfl_xor_sync(0xffffffffu, s, off);
            const double f = tj * s;
            if (lane == 0) y[j] -= f;
            for (int r = j + 1 + lane; r < n; r += 32) y[r] -= f * x[r];
        }
        __syncthreads();
    }
    // Q = H_0 ... H_{n-1}: apply in reverse to the identity, rows of QT = columns of Q
    for (int j = n - 1; j >= 0; --j) {
        const double *x = Wz + (int64_t)j * n;
        const double tj = tz[j];
        for (int q = j + warp; q < n; q += nwarp) {
            double *y = Qz + (int64_t)q * n;
            double s = (lane == 0) ? y[j] : 0.0;
            for (int r = j + 1 + lane; r < n; r += 32) s += x[r] * y[r];
#pragma unroll
            for (int off = 16; off; off >>= 1) s += __shfl_xor_sync(0xffffffffu, s, off);
            const double f = tj * s;
            if (lane == 0) y[j] -= f;
            for (int r = j + 1 + lane; r < n; r += 32) y[r] -= f * x[r];
        }
        __syncthreads();
    }
}

// partial column energies of DT (c x n row-major): part[z][chunk][i]
__global__ void __launch_bounds__(RR_THREADS) colenergy_kernel(const double *DT, int64_t dstride,
                                                               int c, int n, int rows_per_chunk,
                                                               double *part, int nchunk) {
    const int z = blockIdx.y, ch = blockIdx.x;
    const double *D = DT + z * dstride;
    const int q0 = ch * rows_per_chunk, q1 = min(c, q0 + rows_per_chunk);
    double *out = part + ((int64_t)z * nchunk + ch) * n;
    for (int i = threadIdx.x; i < n; i += blockDim.x) {
        double s = 0.0;
        for (int q = q0; q < q1; ++q) {
            const double v = D[(int64_t)q * n + i];
            s += v * v;
        }
        out[i] = s;
    }
}

// rank per shift: first r with sqrt(sum_{i>=r} e_i) <= tol (fixed-order sums);
// also r1 = leading directions whose energy is >= 1e-10 of the first one (the
// directions a Gram-based ordering resolves reliably), and the energies.
__global__ void __launch_bounds__(RR_THREADS) tail_rank_kernel(const double *part, int nchunk, int n,
                                                               const double *tol, int *rank,
                                                               double *dropped, int *r1out,
                                                               const int *active) {
    extern __shared__ double e[];
    const int z = blockIdx.x;
    for (int i = threadIdx.x; i < n; i += blockDim.x) {
        double s = 0.0;
        for (int ch = 0; ch < nchunk; ++ch) s += part[((int64_t)z * nchunk + ch) * n + i];
        e[i] = s;
    }
    __syncthreads();
    if (threadIdx.x == 0) {
        if (active && !active[z]) {
            rank[z] = 0;
            dropped[z] = 0.0;
            if (r1out) r1out[z] = n;
            return;
        }
        double acc = 0.0;
        int r = n;
        // walk from the end: tail(r) = sqrt(sum_{i>=r} e_i), monotone in r
        for (int i = n - 1; i >= 0; --i) {
            if (sqrt(acc + e[i]) > tol[z]) break;
            acc += e[i];
            r = i;
        }
        rank[z] = r;
        dropped[z] = sqrt(acc);
        if (r1out) {
            int r1 = 0;
            const double e0 = n ? e[0] : 0.0;
            while (r1 < n && e[r1] >= 1e-10 * e0 && e0 > 0.0) ++r1;
            r1out[z] = r1;
        }
    }
}

}  // namespace

cudaError_t launch_pchol(const double *M, int64_t mstride, int n, double *S, double *L,
                         const int *active, int nshift, cudaStream_t st) {
    if (n <= 0 || nshift <= 0) return cudaSuccess;
    const size_t sm = (sizeof(double) + sizeof(int)) * (size_t)n;
    pchol_kernel<<<nshift, RR_THREADS, sm, st>>>(M, mstride, n, S, L, active);
    return cudaGetLastError();
}

cudaError_t launch_hqr(const double *A, int64_t astride, int n, double *W, double *QT,
                       double *tau, int64_t tstride, const int *active, int nshift,
                       cudaStream_t st) {
    if (n <= 0 || nshift <= 0) return cudaSuccess;
    hqr_kernel<<<nshift, RR_THREADS, 0, st>>>(A, astride, n, W, QT, tau, tstride, active);
    return cudaGetLastError();
}

cudaError_t launch_tail_rank(const double *DT, int64_t dstride, int c, int n, double *part,
                             const double *tol, int *rank, double *dropped, int *r1out,
                             const int *active, int nshift, cudaStream_t st) {
    if (n <= 0 || nshift <= 0) return cudaSuccess;
    const int rows = 256;
    const int nchunk = std::max(1, (c + rows - 1) / rows);
    colenergy_kernel<<<dim3(nchunk, nshift), RR_THREADS, 0, st>>>(DT, dstride, c, n, rows, part,
                                                                  nchunk);
    cudaError_t e = cudaGetLastError();
    if (e != cudaSuccess) return e;
    tail_rank_kernel<<<nshift, RR_THREADS, sizeof(double) * n, st>>>(part, nchunk, n, tol, rank,
                                                                     dropped, r1out, active);
    return cudaGetLastError();
}

int64_t tail_rank_part_doubles(int c, int n) {
    const int nchunk = std::max(1, (c + 255) / 256);
    return (int64_t)nchunk * n;
}

}  // namespace h2l
