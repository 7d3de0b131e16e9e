// Recompression rank reveal for wide fill rows (K7): exact energies and the
// reference's tail rule.
//
// Reference: gldl.py:67-79 - scipy.linalg.qr(G, pivoting=True) of
// G = [fill rows] (n_R x c, c up to ~10^5 at config 2) and
// rank = first r with ||R[r:, :]||_F <= drop_tol.  The engine (recompress)
// orders the directions with a pivoted QR of the Gram matrix M = G G^T
// (k_qr.cu, cluster kernel), forms D = Q^T G by GEMM and takes the rank here
// from the exact row energies of D: tail(r) = sqrt(sum_{i>=r} ||D_i||^2) =
// ||(I - Q_r Q_r^T) G||_F (Q orthogonal), first r with tail(r) <= drop_tol.
// The ordering only decides how small r is; the dropped part is <= drop_tol as
// in the reference, for any orthonormal Q.
#include <algorithm>
#include <cfloat>
#include "common.cuh"

namespace h2l {

namespace {

constexpr int RR_THREADS = 256;

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
__device__ __forceinline__ void tail_rank_body(const double *part, int nchunk, int n,
                                               const double *tol, int *rank, double *dropped,
                                               int *r1out, const int *active) {
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

__global__ void __launch_bounds__(RR_THREADS) tail_rank_kernel(const double *part, int nchunk, int n,
                                                               const double *tol, int *rank,
                                                               double *dropped, int *r1out,
                                                               const int *active) {
    tail_rank_body(part, nchunk, n, tol, rank, dropped, r1out, active);
}

__global__ void __launch_bounds__(RR_THREADS) colenergy_multi_kernel(const RankJob *jobs,
                                                                     int rows_per_chunk) {
    const RankJob jb = jobs[blockIdx.z];
    const int nchunk = max(1, (jb.c + rows_per_chunk - 1) / rows_per_chunk);
    const int ch = blockIdx.x, z = blockIdx.y;
    if (ch >= nchunk) return;
    const double *D = jb.DT + z * jb.dstride;
    const int q0 = ch * rows_per_chunk, q1 = min(jb.c, q0 + rows_per_chunk);
    double *out = jb.part + ((int64_t)z * nchunk + ch) * jb.n;
    for (int i = threadIdx.x; i < jb.n; i += blockDim.x) {
        double s = 0.0;
        for (int q = q0; q < q1; ++q) {
            const double v = D[(int64_t)q * jb.n + i];
            s += v * v;
        }
        out[i] = s;
    }
}

__global__ void __launch_bounds__(RR_THREADS) tail_rank_multi_kernel(const RankJob *jobs,
                                                                     int rows_per_chunk,
                                                                     const double *tol,
                                                                     const int *active) {
    const RankJob jb = jobs[blockIdx.y];
    const int nchunk = max(1, (jb.c + rows_per_chunk - 1) / rows_per_chunk);
    tail_rank_body(jb.part, nchunk, jb.n, tol, jb.rank, jb.dropped, jb.r1, active);
}

}  // namespace

cudaError_t launch_tail_rank_multi(const RankJob *jobs, int njobs, int cmax, int nmax,
                                   const double *tol, const int *active, int nshift,
                                   cudaStream_t st) {
    if (njobs <= 0 || nmax <= 0 || nshift <= 0) return cudaSuccess;
    const int rows = 256;
    const int nchunk = std::max(1, (cmax + rows - 1) / rows);
    colenergy_multi_kernel<<<dim3(nchunk, nshift, njobs), RR_THREADS, 0, st>>>(jobs, rows);
    cudaError_t e = cudaGetLastError();
    if (e != cudaSuccess) return e;
    tail_rank_multi_kernel<<<dim3(nshift, njobs), RR_THREADS, sizeof(double) * nmax, st>>>(
        jobs, rows, tol, active);
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
