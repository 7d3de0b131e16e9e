// Recompression ordering (K7): column-pivoted Householder QR of the n x n Gram
// matrix M = G G^T of a cluster's fill rows (engine.cu recompress; the rank is
// then taken from exact energies in k_rrqr.cu).
//
// Reference: gldl.py:67-79 runs scipy.linalg.qr(G, mode="full", pivoting=True)
// on G itself (n_R x c, c up to ~10^5) and keeps the first t directions whose
// Frobenius tail exceeds drop_tol.  Here the ordering comes from the Gram
// matrix (n_R x n_R):
//   * pqr_cluster_kernel: M in the distributed shared memory of a thread-block
//     cluster, one cluster barrier per column (primary path, n up to ~900);
//   * form_q_rows_kernel: Q^T from the reflectors, rows in parallel;
//   * pqr_kernel / form_tr_kernel: single-CTA fallback on M in global memory
//     (larger n), also usable with the reference's tolerance stop directly on
//     G^T (target -1) or continued to a common rank (target >= 0).
// Column norms are recomputed exactly after every step (no downdating), ties
// pick the lowest column.  Storage: GT = G^T row-major (a column of G is a
// contiguous row); M is symmetric, so its rows are its columns.
#include "common.cuh"

#include <cooperative_groups.h>

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


// ---------------------------------------------------------------------------
// Cluster-parallel full column-pivoted QR of the n x n Gram matrix M (the
// recompression's ordering step, engine.cu recompress).  One thread-block
// cluster of CS CTAs per shift; CTA c keeps columns q = c, c+CS, ... of M in
// its shared memory (the whole matrix lives in the cluster's distributed
// shared memory), so a step costs two cluster barriers instead of passes over
// L2: (1) every CTA publishes the arg-max of its unused column norms and all
// CTAs reduce the CS candidates (lowest index on ties); (2) the owner of the
// pivot builds the Householder vector, the others copy it through DSMEM, and
// every CTA applies it to its own columns and recomputes their trailing norms
// exactly.  Reflector j is written to row j of M (global; M is dead once
// staged) as v = [1, x[j+1:]] with tau[j], piv[j] -- the input of form_q_rows.
namespace cg = cooperative_groups;

constexpr int PQRC_THREADS = 256;

template <int CS>
__device__ __forceinline__ void pqr_cluster_body(double *Mg, int64_t mstride, int n, double *tau,
                                                 int *piv, int64_t vstride, const int *active,
                                                 int kmax) {
    // One cluster barrier per column: every CTA proposes its best unused column
    // together with that column's Householder vector (double-buffered by step
    // parity), then all CTAs take the same winner, copy its vector through
    // DSMEM and apply it.  A CTA can run at most one step ahead of the slowest
    // (it must pass the next barrier), so the two buffers never race.
    cg::cluster_group cluster = cg::this_cluster();
    const int crank = (int)cluster.block_rank();
    const int z = blockIdx.y;
    if (active && !active[z]) return;  // uniform over the cluster: no barrier is reached
    extern __shared__ __align__(16) double qsm[];
    const int nloc = (n + CS - 1) / CS;
    double *col = qsm;                          // [nloc][n]
    double *vb = col + (size_t)nloc * n;        // [2][n] candidate vectors
    double *vcur = vb + 2 * (size_t)n;          // [n] the step's reflector
    double *nrm = vcur + n;                     // [nloc]
    double *slot = nrm + nloc;                  // [2][4]: norm, tau, beta, (index as double)
    double *red = slot + 8;                     // [32]: 16 values, then 16 ints
    int *usedl = (int *)(red + 32);             // [nloc]
    const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5, nwarp = blockDim.x >> 5;
    double *M = Mg + z * mstride;
    double *tz = tau + z * vstride;
    int *pz = piv + z * vstride;
    for (int lc = warp; lc < nloc; lc += nwarp) {
        const int q = lc * CS + crank;
        double s2 = 0.0;
        if (q < n) {
            for (int r = lane; r < n; r += 32) {
                const double v = M[(int64_t)q * n + r];
                col[(size_t)lc * n + r] = v;
                s2 += v * v;
            }
        }
#pragma unroll
        for (int off = 16; off; off >>= 1) s2 += __shfl_down_sync(0xffffffffu, s2, off);
        if (lane == 0) { nrm[lc] = s2; usedl[lc] = q < n ? 0 : 1; }
    }
    cluster.sync();  // every CTA has read M before any reflector overwrites it
    __shared__ int s_lc, s_win[2];
    __shared__ double s_tau;
    // kmax < n: only the leading kmax pivots are ordered (the recompression keeps a
    // few dozen directions); Q = H_0 ... H_{kmax-1} still spans R^n, its trailing
    // columns an unordered orthonormal complement
    for (int j = 0; j < kmax; ++j) {
        const int par = j & 1;
        double *myv = vb + (size_t)par * n;
        double *mys = slot + 4 * par;
        // ---- local candidate: arg-max of the unused trailing norms (lowest index on ties)
        double bv = -1.0;
        int bi = 0x7fffffff;
        for (int lc = tid; lc < nloc; lc += blockDim.x) {
            if (usedl[lc]) continue;
            const double v = nrm[lc];
            const int q = lc * CS + crank;
            if (v > bv || (v == bv && q < bi)) { bv = v; bi = q; }
        }
#pragma unroll
        for (int off = 16; off; off >>= 1) {
            const double ov = __shfl_down_sync(0xffffffffu, bv, off);
            const int oi = __shfl_down_sync(0xffffffffu, bi, off);
            if (ov > bv || (ov == bv && oi < bi)) { bv = ov; bi = oi; }
        }
        if (lane == 0) { red[warp] = bv; ((int *)(red + 16))[warp] = bi; }
        __syncthreads();
        if (tid == 0) {
            double xv = red[0];
            int xi = ((int *)(red + 16))[0];
            for (int w = 1; w < nwarp; ++w) {
                const double ov = red[w];
                const int oi = ((int *)(red + 16))[w];
                if (ov > xv || (ov == xv && oi < xi)) { xv = ov; xi = oi; }
            }
            mys[0] = xv;
            mys[3] = (double)xi;
            s_lc = xi < n ? xi / CS : -1;
        }
        __syncthreads();
        const int clc = s_lc;
        // ---- its Householder vector (not applied unless it wins)
        if (clc >= 0) {
            const double *x = col + (size_t)clc * n;
            double part = 0.0;
            for (int r = j + 1 + tid; r < n; r += blockDim.x) part += x[r] * x[r];
#pragma unroll
            for (int off = 16; off; off >>= 1) part += __shfl_down_sync(0xffffffffu, part, off);
            if (lane == 0) red[warp] = part;
            __syncthreads();
            double xn2 = 0.0;
            for (int w = 0; w < nwarp; ++w) xn2 += red[w];
            const double alpha = x[j];
            double t_, sc, be;
            if (xn2 == 0.0) { t_ = 0.0; be = alpha; sc = 0.0; }
            else {
                be = -copysign(sqrt(alpha * alpha + xn2), alpha);
                t_ = (be - alpha) / be;
                sc = 1.0 / (alpha - be);
            }
            for (int r = j + 1 + tid; r < n; r += blockDim.x) myv[r] = x[r] * sc;
            if (tid == 0) { myv[j] = 1.0; mys[1] = t_; mys[2] = be; }
        }
        cluster.sync();
        // ---- the winner (every CTA computes the same one): lane c of warp 0 reads
        // CTA c's proposal, one DSMEM round trip, then a warp arg-max
        if (warp == 0) {
            double ov = -1.0, ot = 0.0;
            int oi = 0x7fffffff, oc = lane;
            if (lane < CS) {
                const double *os = cluster.map_shared_rank(slot, lane) + 4 * par;
                ov = os[0];
                ot = os[1];
                oi = (int)os[3];
            }
#pragma unroll
            for (int off = 16; off; off >>= 1) {
                const double v2 = __shfl_xor_sync(0xffffffffu, ov, off);
                const int i2 = __shfl_xor_sync(0xffffffffu, oi, off);
                const int c2 = __shfl_xor_sync(0xffffffffu, oc, off);
                const double t2 = __shfl_xor_sync(0xffffffffu, ot, off);
                if (v2 > ov || (v2 == ov && i2 < oi)) { ov = v2; oi = i2; oc = c2; ot = t2; }
            }
            if (lane == 0) { s_win[0] = oi; s_win[1] = oc; s_tau = ot; }
        }
        __syncthreads();
        const int p = s_win[0], wc = s_win[1];
        const double tj = s_tau;
        if (wc == crank) {
            double *x = col + (size_t)(p / CS) * n;
            double *vrow = M + (int64_t)j * n;
            for (int r = j + tid; r < n; r += blockDim.x) {
                const double v = myv[r];
                vcur[r] = v;
                vrow[r] = v;
                if (r > j) x[r] = v;
            }
            if (tid == 0) {
                x[j] = mys[2];
                tz[j] = tj;
                pz[j] = p;
                usedl[p / CS] = 1;
            }
        } else {
            const double *ov = cluster.map_shared_rank(vb, wc) + (size_t)par * n;
            for (int r = j + tid; r < n; r += blockDim.x) vcur[r] = ov[r];
        }
        __syncthreads();
        // ---- apply H_j = I - tau v v^T to the own unused columns; exact trailing norms.
        // A warp takes up to 4 columns at once: their dot products, reductions and
        // updates are independent, so the shuffle latencies overlap
        for (int lc0 = warp; lc0 < nloc; lc0 += 4 * nwarp) {
            double sd[4] = {0.0, 0.0, 0.0, 0.0};
            bool on[4];
#pragma unroll
            for (int u = 0; u < 4; ++u) {
                const int lc = lc0 + u * nwarp;
                on[u] = lc < nloc && !usedl[lc];
            }
            for (int r = j + lane; r < n; r += 32) {
                const double vr = vcur[r];
#pragma unroll
                for (int u = 0; u < 4; ++u)
                    if (on[u]) sd[u] += vr * col[(size_t)(lc0 + u * nwarp) * n + r];
            }
#pragma unroll
            for (int off = 16; off; off >>= 1)
#pragma unroll
                for (int u = 0; u < 4; ++u) sd[u] += __shfl_xor_sync(0xffffffffu, sd[u], off);
            double nn[4] = {0.0, 0.0, 0.0, 0.0};
            for (int r = j + lane; r < n; r += 32) {
                const double vr = vcur[r];
#pragma unroll
                for (int u = 0; u < 4; ++u)
                    if (on[u]) {
                        double *y = col + (size_t)(lc0 + u * nwarp) * n;
                        const double v = y[r] - (tj * sd[u]) * vr;
                        y[r] = v;
                        if (r > j) nn[u] += v * v;
                    }
            }
#pragma unroll
            for (int off = 16; off; off >>= 1)
#pragma unroll
                for (int u = 0; u < 4; ++u) nn[u] += __shfl_down_sync(0xffffffffu, nn[u], off);
            if (lane == 0)
#pragma unroll
                for (int u = 0; u < 4; ++u)
                    if (on[u]) nrm[lc0 + u * nwarp] = nn[u];
        }
        __syncthreads();
    }
    cluster.sync();  // no CTA exits while its shared memory may still be read
}

template <int CS>
__global__ void __launch_bounds__(PQRC_THREADS) pqr_cluster_kernel(double *Mg, int64_t mstride, int n,
                                                                   double *tau, int *piv,
                                                                   int64_t vstride,
                                                                   const int *active, int kmax) {
    pqr_cluster_body<CS>(Mg, mstride, n, tau, piv, vstride, active, kmax);
}

// a group of clusters' Gram matrices in one launch: thread-block cluster c of the
// grid row serves job c (all CTAs of a cluster read the same job: uniform exits)
template <int CS>
__global__ void __launch_bounds__(PQRC_THREADS) pqr_cluster_multi_kernel(const PqrJob *jobs,
                                                                         const int *active) {
    const PqrJob jb = jobs[blockIdx.x / CS];
    if (jb.n <= 0) return;
    pqr_cluster_body<CS>(jb.M, jb.mstride, jb.n, jb.tau, jb.piv, jb.vstride, active,
                         jb.kmax <= 0 ? jb.n : min(jb.kmax, jb.n));
}

// Q^T of the reflectors in rows of V (row j: v_j = [1 at j, V[j][r] for r > j]):
// row q of Q^T = (H_0 ... H_{n-1} e_q)^T, built by one warp from e_q with
// H_j for j = min(q, n-1) .. 0 (H_j e_q = e_q for j > q).  Rows are independent,
// so the grid spreads them over many CTAs and no barrier is needed.
constexpr int FQ_WARPS = 8;

__device__ __forceinline__ void form_q_rows_body(const double *V, int64_t vstr, int n,
                                                 const double *tau, int64_t tstr, double *QT,
                                                 int64_t qstr, const int *active, int kref) {
    extern __shared__ __align__(16) double ybuf[];
    const int z = blockIdx.y;
    const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
    const int q = blockIdx.x * FQ_WARPS + warp;
    if (q >= n) return;
    double *out = QT + z * qstr + (int64_t)q * n;
    if (active && !active[z]) {
        for (int r = lane; r < n; r += 32) out[r] = (r == q) ? 1.0 : 0.0;
        return;
    }
    double *y = ybuf + (size_t)warp * n;
    for (int r = lane; r < n; r += 32) y[r] = (r == q) ? 1.0 : 0.0;
    __syncwarp();
    const double *Vz = V + z * vstr;
    const double *tzz = tau + z * tstr;
    for (int j = min(q, kref - 1); j >= 0; --j) {
        const double *v = Vz + (int64_t)j * n;
        double sdot = (lane == 0) ? y[j] : 0.0;
        for (int r = j + 1 + lane; r < n; r += 32) sdot += v[r] * y[r];
#pragma unroll
        for (int off = 16; off; off >>= 1) sdot += __shfl_xor_sync(0xffffffffu, sdot, off);
        const double f = tzz[j] * sdot;
        if (lane == 0) y[j] -= f;
        for (int r = j + 1 + lane; r < n; r += 32) y[r] -= f * v[r];
        __syncwarp();
    }
    for (int r = lane; r < n; r += 32) out[r] = y[r];
}

__global__ void __launch_bounds__(FQ_WARPS * 32) form_q_rows_kernel(const double *V, int64_t vstr,
                                                                   int n, const double *tau,
                                                                   int64_t tstr, double *QT,
                                                                   int64_t qstr,
                                                                   const int *active, int kref) {
    form_q_rows_body(V, vstr, n, tau, tstr, QT, qstr, active, kref);
}

__global__ void __launch_bounds__(FQ_WARPS * 32) form_q_rows_multi_kernel(const PqrJob *jobs,
                                                                         const int *active) {
    const PqrJob jb = jobs[blockIdx.z];
    if (blockIdx.x * FQ_WARPS >= jb.n) return;
    form_q_rows_body(jb.M, jb.mstride, jb.n, jb.tau, jb.vstride, jb.QT, jb.qstride, active,
                     jb.kmax <= 0 ? jb.n : min(jb.kmax, jb.n));
}

size_t pqr_cluster_smem(int n, int cs) {
    const int nloc = (n + cs - 1) / cs;
    return sizeof(double) * ((size_t)nloc * n + 3 * (size_t)n + nloc + 8 + 32) + sizeof(int) * (nloc + 2);
}

template <int CS>
cudaError_t launch_pqr_cluster_cs(double *M, int64_t mstride, int n, double *tau, int *piv,
                                  int64_t vstride, const int *active, int nshift, cudaStream_t st,
                                  int kmax) {
    const size_t smem = pqr_cluster_smem(n, CS);
    cudaError_t e = smem_optin(pqr_cluster_kernel<CS>);
    if (e != cudaSuccess) return e;
    if (CS > 8) {
        static std::once_flag once;
        std::call_once(once, [] {
            cudaFuncSetAttribute(pqr_cluster_kernel<CS>, cudaFuncAttributeNonPortableClusterSizeAllowed, 1);
        });
    }
    cudaLaunchConfig_t cfg = {};
    cfg.gridDim = dim3(CS, nshift, 1);
    cfg.blockDim = dim3(PQRC_THREADS, 1, 1);
    cfg.dynamicSmemBytes = smem;
    cfg.stream = st;
    cudaLaunchAttribute at[1];
    at[0].id = cudaLaunchAttributeClusterDimension;
    at[0].val.clusterDim.x = CS;
    at[0].val.clusterDim.y = 1;
    at[0].val.clusterDim.z = 1;
    cfg.attrs = at;
    cfg.numAttrs = 1;
    return cudaLaunchKernelEx(&cfg, pqr_cluster_kernel<CS>, M, mstride, n, tau, piv, vstride, active,
                              kmax);
}

template <int CS>
cudaError_t launch_pqr_cluster_multi_cs(const PqrJob *jobs, int njobs, int nmax, const int *active,
                                        int nshift, cudaStream_t st) {
    const size_t smem = pqr_cluster_smem(nmax, CS);
    cudaError_t e = smem_optin(pqr_cluster_multi_kernel<CS>);
    if (e != cudaSuccess) return e;
    if (CS > 8) {
        static std::once_flag once;
        std::call_once(once, [] {
            cudaFuncSetAttribute(pqr_cluster_multi_kernel<CS>,
                                 cudaFuncAttributeNonPortableClusterSizeAllowed, 1);
        });
    }
    cudaLaunchConfig_t cfg = {};
    cfg.gridDim = dim3(CS * njobs, nshift, 1);
    cfg.blockDim = dim3(PQRC_THREADS, 1, 1);
    cfg.dynamicSmemBytes = smem;
    cfg.stream = st;
    cudaLaunchAttribute at[1];
    at[0].id = cudaLaunchAttributeClusterDimension;
    at[0].val.clusterDim.x = CS;
    at[0].val.clusterDim.y = 1;
    at[0].val.clusterDim.z = 1;
    cfg.attrs = at;
    cfg.numAttrs = 1;
    return cudaLaunchKernelEx(&cfg, pqr_cluster_multi_kernel<CS>, jobs, active);
}

}  // namespace

// cluster size for an n x n Gram matrix (0: too large for distributed shared memory)
int pqr_cluster_size(int n) {
    const size_t cap = 220 * 1024;
    if (pqr_cluster_smem(n, 8) <= cap) return 8;
    if (pqr_cluster_smem(n, 16) <= cap) return 16;
    return 0;
}

cudaError_t launch_pqr_cluster(double *M, int64_t mstride, int n, double *tau, int *piv,
                               int64_t vstride, const int *active, int nshift, cudaStream_t st,
                               int kmax) {
    if (nshift <= 0 || n <= 0) return cudaSuccess;
    kmax = kmax <= 0 ? n : std::min(kmax, n);
    const int cs = pqr_cluster_size(n);
    if (cs == 8) return launch_pqr_cluster_cs<8>(M, mstride, n, tau, piv, vstride, active, nshift, st, kmax);
    if (cs == 16) return launch_pqr_cluster_cs<16>(M, mstride, n, tau, piv, vstride, active, nshift, st, kmax);
    return cudaErrorInvalidValue;
}

cudaError_t launch_form_q_rows(const double *V, int64_t vstride, int n, const double *tau,
                               int64_t tstride, double *QT, int64_t qstride, const int *active,
                               int nshift, cudaStream_t st, int kref) {
    if (nshift <= 0 || n <= 0) return cudaSuccess;
    kref = kref <= 0 ? n : std::min(kref, n);
    const size_t smem = sizeof(double) * FQ_WARPS * (size_t)n;
    cudaError_t e = smem_optin(form_q_rows_kernel);
    if (e != cudaSuccess) return e;
    dim3 grid((n + FQ_WARPS - 1) / FQ_WARPS, nshift);
    form_q_rows_kernel<<<grid, FQ_WARPS * 32, smem, st>>>(V, vstride, n, tau, tstride, QT, qstride,
                                                         active, kref);
    return cudaGetLastError();
}

cudaError_t launch_pqr_cluster_multi(const PqrJob *jobs, int njobs, int nmax, const int *active,
                                     int nshift, cudaStream_t st) {
    if (njobs <= 0 || nshift <= 0 || nmax <= 0) return cudaSuccess;
    const int cs = pqr_cluster_size(nmax);
    if (cs == 8) return launch_pqr_cluster_multi_cs<8>(jobs, njobs, nmax, active, nshift, st);
    if (cs == 16) return launch_pqr_cluster_multi_cs<16>(jobs, njobs, nmax, active, nshift, st);
    return cudaErrorInvalidValue;
}

cudaError_t launch_form_q_rows_multi(const PqrJob *jobs, int njobs, int nmax, const int *active,
                                     int nshift, cudaStream_t st) {
    if (njobs <= 0 || nshift <= 0 || nmax <= 0) return cudaSuccess;
    const size_t smem = sizeof(double) * FQ_WARPS * (size_t)nmax;
    cudaError_t e = smem_optin(form_q_rows_multi_kernel);
    if (e != cudaSuccess) return e;
    dim3 grid((nmax + FQ_WARPS - 1) / FQ_WARPS, nshift, njobs);
    form_q_rows_multi_kernel<<<grid, FQ_WARPS * 32, smem, st>>>(jobs, active);
    return cudaGetLastError();
}

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
