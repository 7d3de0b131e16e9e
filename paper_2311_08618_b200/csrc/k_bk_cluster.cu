// Bunch-Kaufman LDL^T of one large redundant block (n > BK_SMEM_MAX) on a
// thread-block cluster (K2 + K3 for the big fronts of configs 2-5).
//
// Same algorithm, operation order and rounding as bk_core in k_bk.cu (the
// reference kernel `_core.bk_factor`, _kernels.pyx:21-125, and `inertia_of`,
// dense.py:127-168): every element update is the same expression on the same
// operands, pivot tests read the same values and max-reductions are
// order-free, so the factor is bit-identical to the single-CTA kernel.  What
// changes is where the matrix lives: the packed lower triangle is spread over
// the cluster's shared memory by columns (column j on CTA j % CS), so a step
// no longer streams the trailing matrix through L2 from one SM.  One step:
//   finish the previous pivot (deferred scaling / 2x2 write-back, owners)
//   decision: column arg-max (look-ahead of the owner), row-max of row imax
//             across the cluster when the 1x1 test fails           | sync
//   interchange kk <-> kp (owner of column kk, DSMEM)               | sync
//   copy the pivot column(s) into every CTA; rank-1 / rank-2 update of the
//   own columns; the owner of the next pivot column reduces its arg-max | sync
#include <cfloat>
#include <cooperative_groups.h>
#include "common.cuh"

namespace h2l {

namespace {

namespace cg = cooperative_groups;
constexpr int BKC_THREADS = 256;

struct Am {
    double v;
    int i;
};
__device__ __forceinline__ Am am_better(Am a, Am b) {
    return (b.v > a.v || (b.v == a.v && b.i < a.i)) ? b : a;
}
__device__ __forceinline__ Am am_warp(Am x) {
#pragma unroll
    for (int off = 16; off; off >>= 1) {
        Am o{__shfl_xor_sync(0xffffffffu, x.v, off), __shfl_xor_sync(0xffffffffu, x.i, off)};
        x = am_better(x, o);
    }
    return x;
}

struct BkcShared {
    Am red_a[8];
    double red_d[8];
    Am next;        // look-ahead arg-max of the next pivot column (valid at its owner)
    double part;    // row-max / tolerance partial of this CTA
    int kp, kstep, info, pad;
};

template <int CS>
struct Dist {
    double *col;  // own packed columns
    int n, crank;
    // offset of column j inside its owner's packed store
    __device__ __forceinline__ int64_t off(int j) const {
        const int64_t lc = j / CS, c = j % CS;
        return lc * n - (int64_t)CS * lc * (lc - 1) / 2 - c * lc;
    }
    __device__ __forceinline__ bool mine(int j) const { return j % CS == crank; }
    __device__ __forceinline__ double *loc(int i, int j) const { return col + off(j) + (i - j); }
    __device__ __forceinline__ double *rem(cg::cluster_group &cl, int i, int j) const {
        double *base = cl.map_shared_rank(col, j % CS);
        return base + off(j) + (i - j);
    }
};

__device__ double cta_max(double v, double *red) {
    const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
#pragma unroll
    for (int off = 16; off; off >>= 1) v = fmax(v, __shfl_xor_sync(0xffffffffu, v, off));
    if (lane == 0) red[warp] = v;
    __syncthreads();
    double x = 0.0;
    for (int w = 0; w < (int)(blockDim.x >> 5); ++w) x = fmax(x, red[w]);
    __syncthreads();
    return x;
}

template <int CS>
__global__ void __launch_bounds__(BKC_THREADS) bk_cluster_kernel(const BkJob *jobs,
                                                                 long long *counts, int *status) {
    cg::cluster_group cl = cg::this_cluster();
    const int crank = (int)cl.block_rank();
    const BkJob jb = jobs[blockIdx.x / CS];
    const int z = blockIdx.y;
    const int n = jb.n;
    if (n <= 0) return;  // uniform over the cluster
    extern __shared__ __align__(16) double bsm[];
    __shared__ BkcShared sh;
    const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5, nthr = blockDim.x;
    const int nwarp = nthr >> 5;
    const int nloc = (n - crank + CS - 1) / CS;  // own columns: crank, crank+CS, ...
    Dist<CS> A{bsm, n, crank};
    // the per-CTA buffers sit at the same offset in every CTA (remote w0/w1 reads):
    // after the largest packed share, rank 0's
    const int64_t l0 = (n + CS - 1) / CS - 1;
    const int64_t own = l0 * n - (int64_t)CS * l0 * (l0 - 1) / 2 + (n - l0 * CS);
    double *pk = bsm + own;   // pivot column k (rows k..n-1 at index i)
    double *pk1 = pk + n;     // pivot column k+1
    double *w0 = pk1 + n;     // 2x2 L columns for own j
    double *w1 = w0 + n;
    int *swaps = (int *)(w1 + n);
    double *a = jb.a + z * jb.astride;
    int *perm = jb.perm + z * jb.pstride;
    double *dinfo = jb.dinfo + 3 * z * jb.pstride;
    const double alpha = (1.0 + sqrt(17.0)) / 8.0;

    // ---- load own columns, tolerance over the full n x n block (dense.py:50-53)
    for (int lcn = warp; lcn < nloc; lcn += nwarp) {
        const int j = crank + lcn * CS;
        double *c = A.loc(j, j);
        for (int i = j + lane; i < n; i += 32) c[i - j] = a[(int64_t)i * jb.ld + j];
    }
    double m = 0.0;
    for (int i = crank + CS * warp; i < n; i += CS * nwarp)
        for (int j = lane; j < n; j += 32) m = fmax(m, fabs(a[(int64_t)i * jb.ld + j]));
    m = cta_max(m, sh.red_d);
    if (tid == 0) sh.part = m;
    for (int i = tid; i < 2 * n; i += nthr) swaps[i] = -1;
    if (crank == 0)
        for (int i = tid; i < n; i += nthr) perm[i] = i;
    __syncthreads();
    // column 0 arg-max at its owner (CTA 0)
    if (crank == 0) {
        Am mine{0.0, 0x7fffffff};
        for (int i = 1 + tid; i < n; i += nthr) {
            const double v = fabs(*A.loc(i, 0));
            if (v > mine.v) { mine.v = v; mine.i = i; }
        }
        mine = am_warp(mine);
        if (lane == 0) sh.red_a[warp] = mine;
        __syncthreads();
        if (tid == 0) {
            Am x{0.0, 0x7fffffff};
            for (int w = 0; w < nwarp; ++w) x = am_better(x, sh.red_a[w]);
            sh.next = x;
        }
    }
    cl.sync();
    double amax = 0.0;
    for (int c = 0; c < CS; ++c) amax = fmax(amax, cl.map_shared_rank(&sh, c)->part);
    const double tol = 1e3 * DBL_EPSILON * amax;
    cl.sync();  // partials read before they are reused

    int prev = -1, prev_step = 0;
    double prev_r1 = 0.0;
    int k = 0, info = 0;
    while (k < n) {
        // ---- finish the previous pivot (owners; nobody reads these columns until the end)
        if (prev_step == 1 && A.mine(prev)) {
            double *c = A.loc(prev, prev);
            for (int i = prev + 1 + tid; i < n; i += nthr) c[i - prev] = __dmul_rn(c[i - prev], prev_r1);
        } else if (prev_step == 2) {
            if (A.mine(prev))
                for (int j = prev + 2 + tid; j < n; j += nthr)
                    *A.loc(j, prev) = cl.map_shared_rank(w0, j % CS)[j];
            if (A.mine(prev + 1))
                for (int j = prev + 2 + tid; j < n; j += nthr)
                    *A.loc(j, prev + 1) = cl.map_shared_rank(w1, j % CS)[j];
        }
        // ---- pivot decision (uniform: every CTA reads the same values)
        const Am cm = cl.map_shared_rank(&sh, k % CS)->next;
        const double colmax = cm.v;
        const int imax = cm.v > 0.0 ? cm.i : k;
        const double absakk = fabs(*A.rem(cl, k, k));
        int kp = k, kstep = 1;
        if (!(absakk >= __dmul_rn(alpha, colmax))) {
            const double aii = fabs(*A.rem(cl, imax, imax));
            double r = 0.0;
            for (int j = k + tid; j < imax; j += nthr)
                if (A.mine(j)) r = fmax(r, fabs(*A.loc(imax, j)));
            if (A.mine(imax))
                for (int i = imax + 1 + tid; i < n; i += nthr) r = fmax(r, fabs(*A.loc(i, imax)));
            r = cta_max(r, sh.red_d);
            if (tid == 0) sh.part = r;
            cl.sync();
            double rowmax = 0.0;
            for (int c = 0; c < CS; ++c) rowmax = fmax(rowmax, cl.map_shared_rank(&sh, c)->part);
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
        if (tid == 0) { swaps[2 * k] = kk; swaps[2 * k + 1] = kp; }
        // without an interchange nothing the other CTAs may still read (column k,
        // the owner's arg-max slot) is written before the end-of-step barrier, so
        // the two interchange barriers are skipped (kp, kk are cluster-uniform)
        if (kp != kk) cl.sync();  // every decision input has been read
        // ---- interchange kk <-> kp on the lower triangle (owner of column kk)
        if (kp != kk && A.mine(kk)) {
            for (int i = kp + 1 + tid; i < n; i += nthr) {
                double *x = A.loc(i, kk), *y = A.rem(cl, i, kp);
                const double t = *x; *x = *y; *y = t;
            }
            for (int j = kk + 1 + tid; j < kp; j += nthr) {
                double *x = A.loc(j, kk), *y = A.rem(cl, kp, j);
                const double t = *x; *x = *y; *y = t;
            }
            if (tid == 0) {
                double *x = A.loc(kk, kk), *y = A.rem(cl, kp, kp);
                double t = *x; *x = *y; *y = t;
                if (kstep == 2) {
                    double *u = A.rem(cl, kk, k), *v = A.rem(cl, kp, k);
                    t = *u; *u = *v; *v = t;
                }
            }
        }
        if (kp != kk && crank == 0 && tid == 0) { const int q = perm[kk]; perm[kk] = perm[kp]; perm[kp] = q; }
        if (kp != kk) cl.sync();
        // ---- pivot columns into every CTA
        {
            const double *src = A.rem(cl, k, k);
            for (int i = k + tid; i < n; i += nthr) pk[i] = src[i - k];
            if (kstep == 2 && k + 1 < n) {
                const double *s1 = A.rem(cl, k + 1, k + 1);
                for (int i = k + 1 + tid; i < n; i += nthr) pk1[i] = s1[i - k - 1];
            }
        }
        __syncthreads();
        Am nx{0.0, 0x7fffffff};
        if (kstep == 1) {
            const double d = pk[k];
            if (fabs(d) <= tol) { info = k + 1; break; }
            const double r1 = 1.0 / d;
            for (int j = k + 1 + warp * CS + ((crank - (k + 1) % CS + CS) % CS); j < n; j += nwarp * CS) {
                // own columns j > k, one warp per column
                const double wj = __dmul_rn(r1, pk[j]);
                double *c = A.loc(j, j);
                const bool look = (j == k + 1);
                for (int i = j + lane; i < n; i += 32) {
                    const double v = __dsub_rn(c[i - j], __dmul_rn(pk[i], wj));
                    c[i - j] = v;
                    if (look && i > j && fabs(v) > nx.v) { nx.v = fabs(v); nx.i = i; }
                }
                if (look) {
                    nx = am_warp(nx);
                    if (lane == 0) sh.next = nx;
                }
            }
            if (crank == 0 && tid == 0) { dinfo[3 * k] = d; dinfo[3 * k + 1] = 0.0; dinfo[3 * k + 2] = 1.0; }
            prev_r1 = r1;
        } else {
            const double a11 = pk[k], a22 = pk1[k + 1];
            double d21 = pk[k + 1];
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
                for (int j = k + 2 + warp * CS + ((crank - (k + 2) % CS + CS) % CS); j < n; j += nwarp * CS) {
                    const double ajk = pk[j], ajk1 = pk1[j];
                    const double wk = __dmul_rn(d21, __dsub_rn(__dmul_rn(d11, ajk), ajk1));
                    const double wk1 = __dmul_rn(d21, __dsub_rn(__dmul_rn(d22, ajk1), ajk));
                    double *c = A.loc(j, j);
                    const bool look = (j == k + 2);
                    for (int i = j + lane; i < n; i += 32) {
                        const double s = __dadd_rn(__dmul_rn(pk[i], wk), __dmul_rn(pk1[i], wk1));
                        const double v = __dsub_rn(c[i - j], s);
                        c[i - j] = v;
                        if (look && i > j && fabs(v) > nx.v) { nx.v = fabs(v); nx.i = i; }
                    }
                    if (lane == 0) { w0[j] = wk; w1[j] = wk1; }
                    if (look) {
                        nx = am_warp(nx);
                        if (lane == 0) sh.next = nx;
                    }
                }
            }
            if (crank == 0 && tid == 0) {
                dinfo[3 * k] = a11; dinfo[3 * k + 1] = pk[k + 1]; dinfo[3 * k + 2] = 2.0;
                dinfo[3 * k + 3] = a22; dinfo[3 * k + 4] = 0.0; dinfo[3 * k + 5] = 0.0;
            }
        }
        cl.sync();
        prev = k;
        prev_step = kstep;
        k += kstep;
    }
    // ---- finish the last pivot
    if (!info) {
        if (prev_step == 1 && A.mine(prev)) {
            double *c = A.loc(prev, prev);
            for (int i = prev + 1 + tid; i < n; i += nthr) c[i - prev] = __dmul_rn(c[i - prev], prev_r1);
        } else if (prev_step == 2) {
            if (A.mine(prev))
                for (int j = prev + 2 + tid; j < n; j += nthr)
                    *A.loc(j, prev) = cl.map_shared_rank(w0, j % CS)[j];
            if (A.mine(prev + 1))
                for (int j = prev + 2 + tid; j < n; j += nthr)
                    *A.loc(j, prev + 1) = cl.map_shared_rank(w1, j % CS)[j];
        }
    }
    cl.sync();
    // ---- engine mode: replay the interchanges on the finished L columns (own columns)
    if (!info) {
        for (int lcn = warp; lcn < nloc; lcn += nwarp) {
            const int c = crank + lcn * CS;
            if (lane == 0)
                for (int s = c + 1; s < n; ++s) {
                    const int kk = swaps[2 * s], kp = swaps[2 * s + 1];
                    if (kk < 0 || kp == kk) continue;
                    double *x = A.loc(kk, c), *y = A.loc(kp, c);
                    const double t = *x; *x = *y; *y = t;
                }
        }
        __syncthreads();
    }
    for (int lcn = warp; lcn < nloc; lcn += nwarp) {
        const int j = crank + lcn * CS;
        const double *c = A.loc(j, j);
        for (int i = j + lane; i < n; i += 32) a[(int64_t)i * jb.ld + j] = c[i - j];
    }
    cl.sync();  // remote reads done; dinfo complete
    if (info) {
        if (crank == 0 && tid == 0) atomicOr(status + z, 1);
        return;
    }
    if (crank != 0) return;
    double dm = 0.0;
    for (int q = tid; q < n; q += nthr) dm = fmax(dm, fmax(fabs(dinfo[3 * q]), fabs(dinfo[3 * q + 1])));
    const double dmax = cta_max(dm, sh.red_d);
    if (tid == 0) {
        const double zt = 1e3 * DBL_EPSILON * dmax;
        long long neg = 0, zero = 0, pos = 0;
        for (int q = 0; q < n;) {
            if (dinfo[3 * q + 2] < 1.5) {
                const double d = dinfo[3 * q];
                if (fabs(d) <= zt) ++zero; else if (d < 0.0) ++neg; else ++pos;
                q += 1;
            } else {
                const double x = dinfo[3 * q], y = dinfo[3 * q + 3], e = dinfo[3 * q + 1];
                const double det = __dsub_rn(__dmul_rn(x, y), __dmul_rn(e, e));
                const double tr = __dadd_rn(x, y);
                const double zt2 = __dmul_rn(zt, zt);
                if (det < -zt2) { ++neg; ++pos; }
                else if (det > zt2) { if (tr < 0.0) neg += 2; else pos += 2; }
                else {
                    ++zero;
                    if (tr < -zt) ++neg; else if (tr > zt) ++pos; else ++zero;
                }
                q += 2;
            }
        }
        atomicAdd((unsigned long long *)(counts + 3 * z + 0), (unsigned long long)neg);
        atomicAdd((unsigned long long *)(counts + 3 * z + 1), (unsigned long long)zero);
        atomicAdd((unsigned long long *)(counts + 3 * z + 2), (unsigned long long)pos);
    }
}

size_t bkc_smem(int n, int cs) {
    // the largest own share belongs to rank 0 (columns 0, cs, 2cs, ...)
    const int64_t nloc = (n + cs - 1) / cs;
    const int64_t lc = nloc - 1;
    const int64_t own = lc * n - (int64_t)cs * lc * (lc - 1) / 2 + (n - lc * cs);
    return sizeof(double) * (size_t)(own + 4 * (int64_t)n) + sizeof(int) * 2 * (size_t)n;
}

template <int CS>
cudaError_t launch_cs(const BkJob *jobs, int njobs, int nshift, int n, int64_t *counts, int *status,
                      cudaStream_t st) {
    cudaError_t e = smem_optin(bk_cluster_kernel<CS>);
    if (e != cudaSuccess) return e;
    if (CS > 8) {
        static std::once_flag once;
        std::call_once(once, [] {
            cudaFuncSetAttribute(bk_cluster_kernel<CS>, cudaFuncAttributeNonPortableClusterSizeAllowed, 1);
        });
    }
    cudaLaunchConfig_t cfg = {};
    cfg.gridDim = dim3(CS * njobs, nshift, 1);
    cfg.blockDim = dim3(BKC_THREADS, 1, 1);
    cfg.dynamicSmemBytes = bkc_smem(n, CS);
    cfg.stream = st;
    cudaLaunchAttribute at[1];
    at[0].id = cudaLaunchAttributeClusterDimension;
    at[0].val.clusterDim.x = CS;
    at[0].val.clusterDim.y = 1;
    at[0].val.clusterDim.z = 1;
    cfg.attrs = at;
    cfg.numAttrs = 1;
    return cudaLaunchKernelEx(&cfg, bk_cluster_kernel<CS>, jobs, (long long *)counts, status);
}

}  // namespace

int bk_cluster_size(int n) {
    const size_t cap = 200 * 1024;
    if (bkc_smem(n, 8) <= cap) return 8;
    if (bkc_smem(n, 16) <= cap) return 16;
    return 0;
}

cudaError_t launch_bk_cluster(const BkJob *dev_jobs, int njobs, int nshift, int n, int64_t *counts,
                              int *status, cudaStream_t st) {
    if (njobs <= 0 || nshift <= 0 || n <= 0) return cudaSuccess;
    const int cs = bk_cluster_size(n);
    if (cs == 8) return launch_cs<8>(dev_jobs, njobs, nshift, n, counts, status, st);
    if (cs == 16) return launch_cs<16>(dev_jobs, njobs, nshift, n, counts, status, st);
    return cudaErrorInvalidValue;
}

}  // namespace h2l
