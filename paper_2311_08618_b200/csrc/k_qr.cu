// Fill recompression rank-reveal (K7): column-pivoted Householder QR with the
// reference's absolute Frobenius-tail stopping rule.
//
// Reference: gldl.py:67-79 runs scipy.linalg.qr(G, mode="full",
// pivoting=True) (dgeqp3 + dorgqr) on the full G and then picks
// rank = first r with sqrt(sum_{i>=r} ||R[i,:]||^2) <= drop_tol.  After r
// Householder steps that tail is exactly the Frobenius norm of the not yet
// reduced trailing block, so the factorization can stop as soon as it drops
// under the tolerance: only t << min(G.shape) steps are performed, and the
// completion Q[:, t:] is taken from the same reflectors (any orthonormal
// completion spans the same redundant space; inertia is invariant to the
// choice).  Column norms are recomputed exactly after every step (no
// downdating), ties pick the lowest column.
//
// Storage: GT = G^T (cols(G) x rows(G), row-major) so each column of G is a
// contiguous row; one CTA per shift; warps own columns, lanes own rows.
// Phase A stops on the tolerance; phase B continues every shift to the
// common rank t = max over shifts (shift-batched structure); form_q builds
// Tr = [U_r^T ; U_s^T] (rows(G) x rows(G)) from the reflectors.
#include "common.cuh"

namespace h2l {

namespace {

constexpr int QR_THREADS = 512;

__device__ double block_sum(double v, double *red) {
    const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
#pragma unroll
    for (int off = 16; off; off >>= 1) v += __shfl_down_sync(0xffffffffu, v, off);
    if (lane == 0) red[warp] = v;
    __syncthreads();
    if (warp == 0) {
        double x = lane < (int)(blockDim.x >> 5) ? red[lane] : 0.0;
#pragma unroll
        for (int off = 16; off; off >>= 1) x += __shfl_down_sync(0xffffffffu, x, off);
        if (lane == 0) red[32] = x;
    }
    __syncthreads();
    double r = red[32];
    __syncthreads();
    return r;
}

__device__ int block_argmax_unused(const double *norms, const int *used, int c, double *redv,
                                   int *redi) {
    const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
    double bv = -1.0;
    int bi = 0x7fffffff;
    for (int q = threadIdx.x; q < c; q += blockDim.x) {
        if (used[q]) continue;
        double v = norms[q];
        if (v > bv) { bv = v; bi = q; }
    }
#pragma unroll
    for (int off = 16; off; off >>= 1) {
        double ov = __shfl_down_sync(0xffffffffu, bv, off);
        int oi = __shfl_down_sync(0xffffffffu, bi, off);
        if (ov > bv || (ov == bv && oi < bi)) { bv = ov; bi = oi; }
    }
    if (lane == 0) { redv[warp] = bv; redi[warp] = bi; }
    __syncthreads();
    if (warp == 0) {
        double xv = lane < (int)(blockDim.x >> 5) ? redv[lane] : -1.0;
        int xi = lane < (int)(blockDim.x >> 5) ? redi[lane] : 0x7fffffff;
#pragma unroll
        for (int off = 16; off; off >>= 1) {
            double ov = __shfl_down_sync(0xffffffffu, xv, off);
            int oi = __shfl_down_sync(0xffffffffu, xi, off);
            if (ov > xv || (ov == xv && oi < xi)) { xv = ov; xi = oi; }
        }
        if (lane == 0) redi[32] = xi;
    }
    __syncthreads();
    int r = redi[32];
    __syncthreads();
    return r;
}

struct QrArgs {
    double *GT;          // c x nR per shift (row q = column q of G)
    int64_t gstride;
    int c, nR, ldg;
    double *tau;         // [shift][nR]
    int *piv;            // [shift][nR]
    int *used;           // [shift][c]
    double *norms;       // [shift][c]
    int64_t vstride;     // stride of tau/piv (>= nR)
    int64_t cstride;     // stride of used/norms (>= c)
    const double *tol;   // [shift] (phase A)
    int *rank;           // [shift] in/out
    double *dropped;     // [shift]
    const int *active;   // [shift] 0 -> skip this shift (singular)
    int target;          // -1: phase A (tolerance); else phase B (continue to target)
};

__global__ void __launch_bounds__(QR_THREADS) pqr_kernel(QrArgs a) {
    __shared__ double redv[40];
    __shared__ int redi[40];
    __shared__ double s_beta, s_tau, s_scale;
    const int z = blockIdx.x;
    if (a.active && !a.active[z]) {
        if (threadIdx.x == 0 && a.target == -1) { a.rank[z] = 0; a.dropped[z] = 0.0; }
        return;
    }
    double *GT = a.GT + z * a.gstride;
    double *tau = a.tau + z * a.vstride;
    int *piv = a.piv + z * a.vstride;
    int *used = a.used + z * a.cstride;
    double *norms = a.norms + z * a.cstride;
    const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5, nwarp = blockDim.x >> 5;
    const int c = a.c, nR = a.nR, kmax = min(c, nR);
    int j;
    const bool full = a.target == -2;  // init and run to min(c, nR) steps (no tolerance)
    if (a.target < 0) {
        j = 0;
        for (int q = warp; q < c; q += nwarp) {
            double s = 0.0;
            for (int r = lane; r < nR; r += 32) { double v = GT[(int64_t)q * a.ldg + r]; s += v * v; }
#pragma unroll
            for (int off = 16; off; off >>= 1) s += __shfl_down_sync(0xffffffffu, s, off);
            if (lane == 0) { norms[q] = s; used[q] = 0; }
        }
    } else {
        j = a.rank[z];
    }
    __syncthreads();
    double tail = 0.0;
    while (true) {
        double part = 0.0;
        for (int q = threadIdx.x; q < c; q += blockDim.x)
            if (!used[q]) part += norms[q];
        tail = sqrt(block_sum(part, redv));
        if (full) {
            // no early stop
        } else if (a.target < 0) {
            if (tail <= a.tol[z]) break;
        } else if (j >= a.target) {
            break;
        }
        if (j >= kmax) break;
        const int p = block_argmax_unused(norms, used, c, redv, redi);
        double *x = GT + (int64_t)p * a.ldg;
        double part2 = 0.0;
        for (int r = j + 1 + threadIdx.x; r < nR; r += blockDim.x) part2 += x[r] * x[r];
        const double xn2 = block_sum(part2, redv);
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
            tau[j] = s_tau;
            piv[j] = p;
            used[p] = 1;
        }
        __syncthreads();
        const double tj = s_tau;
        for (int r = j + 1 + threadIdx.x; r < nR; r += blockDim.x) x[r] *= s_scale;
        __syncthreads();
        if (threadIdx.x == 0) x[j] = s_beta;
        // apply H_j = I - tau v v^T (v = [1, x[j+1:]]) to the remaining columns
        for (int q = warp; q < c; q += nwarp) {
            if (used[q]) continue;
            double *y = GT + (int64_t)q * a.ldg;
            double s = (lane == 0) ? y[j] : 0.0;
            for (int r = j + 1 + lane; r < nR; r += 32) s += x[r] * y[r];
#pragma unroll
            for (int off = 16; off; off >>= 1) s += __shfl_xor_sync(0xffffffffu, s, off);
            const double f = tj * s;
            if (lane == 0) y[j] -= f;
            double nn = 0.0;
            for (int r = j + 1 + lane; r < nR; r += 32) {
                double v = y[r] - f * x[r];
                y[r] = v;
                nn += v * v;
            }
#pragma unroll
            for (int off = 16; off; off >>= 1) nn += __shfl_down_sync(0xffffffffu, nn, off);
            if (lane == 0) norms[q] = nn;
        }
        __syncthreads();
        ++j;
    }
    if (threadIdx.x == 0 && !full) {
        a.rank[z] = j;
        if (a.target < 0) a.dropped[z] = tail;
    }
}

// Tr rows: [U_r^T (nR - t rows) ; U_s^T (t rows)], U = H_0 ... H_{t-1}.
__global__ void __launch_bounds__(QR_THREADS) form_tr_kernel(const double *GT, int64_t gstride,
                                                             int ldg, const double *tau,
                                                             const int *piv, int64_t vstride,
                                                             int nR, int t, double *Tr,
                                                             int64_t tstride, const int *active) {
    const int z = blockIdx.x;
    double *T = Tr + z * tstride;
    const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5, nwarp = blockDim.x >> 5;
    // QT row q lives at Tr row map(q)
    auto row = [&](int q) { return q >= t ? q - t : nR - t + q; };
    for (int64_t e = threadIdx.x; e < (int64_t)nR * nR; e += blockDim.x) {
        const int q = (int)(e / nR), r = (int)(e % nR);
        T[(int64_t)row(q) * nR + r] = (q == r) ? 1.0 : 0.0;
    }
    if (active && !active[z]) return;
    __syncthreads();
    const double *G = GT + z * gstride;
    const double *tz = tau + z * vstride;
    const int *pz = piv + z * vstride;
    for (int j = t - 1; j >= 0; --j) {
        const double *x = G + (int64_t)pz[j] * ldg;  // v = [1, x[j+1:]]
        const double tj = tz[j];
        for (int q = j + warp; q < nR; q += nwarp) {
            double *y = T + (int64_t)row(q) * nR;
            double s = (lane == 0) ? y[j] : 0.0;
            for (int r = j + 1 + lane; r < nR; r += 32) s += x[r] * y[r];
#pragma unroll
            for (int off = 16; off; off >>= 1) s += __shfl_xor_sync(0xffffffffu, s, off);
            const double f = tj * s;
            if (lane == 0) y[j] -= f;
            for (int r = j + 1 + lane; r < nR; r += 32) y[r] -= f * x[r];
        }
        __syncthreads();
    }
}

}  // namespace

cudaError_t launch_pqr(double *GT, int64_t gstride, int c, int nR, int ldg, double *tau, int *piv,
                       int *used, double *norms, int64_t vstride, int64_t cstride,
                       const double *tol, int *rank, double *dropped, const int *active,
                       int target, int nshift, cudaStream_t st) {
    if (nshift <= 0) return cudaSuccess;
    QrArgs a{GT, gstride, c, nR, ldg, tau, piv, used, norms, vstride, cstride,
             tol, rank, dropped, active, target};
    pqr_kernel<<<nshift, QR_THREADS, 0, st>>>(a);
    return cudaGetLastError();
}

cudaError_t launch_form_tr(const double *GT, int64_t gstride, int ldg, const double *tau,
                           const int *piv, int64_t vstride, int nR, int t, double *Tr,
                           int64_t tstride, const int *active, int nshift, cudaStream_t st) {
    if (nshift <= 0 || nR <= 0) return cudaSuccess;
    form_tr_kernel<<<nshift, QR_THREADS, 0, st>>>(GT, gstride, ldg, tau, piv, vstride, nR, t, Tr,
                                                  tstride, active);
    return cudaGetLastError();
}

}  // namespace h2l
