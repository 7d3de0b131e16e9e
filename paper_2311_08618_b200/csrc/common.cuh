// Shared declarations of the sm_100a kernels behind libh2ldl.so.
//
// Every kernel is "batched twice": over a host-built task list (the blocks
// of one elimination step / merge) and over shifts (gridDim.y = s).  A task
// stores the pointers of shift 0 plus a per-operand shift stride, so one
// launch advances every shift of the wave (shift batching).
// All matrices are row-major float64.
#pragma once

#include <cstdint>
#include <mutex>
#include <set>
#include <utility>
#include <vector>
#include <cuda_runtime.h>

namespace h2l {

// dst = (acc ? dst : 0) + alpha * op(src) - [shift_diag] mu[z] * I   (rows x cols)
// src == nullptr -> zero fill (identity when ident != 0).
struct CopyTask {
    const double *src;
    double *dst;
    int64_t sstride, dstride;  // per-shift strides (elements)
    int rows, cols;
    int lds, ldd;
    int trans;                 // element (r, c) = src[c*lds + r]
    int acc;
    int ident;
    int shift_diag;
    double alpha;
};

// C = alpha * opA(MxK) * opB(KxN) + beta * C
//   opA: tA=0 A[m*lda+k], tA=1 A[k*lda+m];  opB: tB=0 B[k*ldb+n], tB=1 B[n*ldb+k]
struct GemmTask {
    const double *A;
    const double *B;
    double *C;
    int64_t sA, sB, sC;
    int M, N, K;
    int lda, ldb, ldc;
    int tA, tB;
    double alpha, beta;
};

constexpr int PANEL_ROWS = 32;

// one <= 32-row tile of the elimination panel (k_panel.cu)
struct PanelTile {
    const double *src;
    int64_t sstride;
    int lds;
    int trans;       // panel row r = column (src_row0 + r) of src
    int row0;        // first panel row of the tile
    int nrows;
    int src_row0;
    int job;         // PanelJob of the tile (multi-cluster launches)
};

// one cluster's factor + outputs of a panel launch (a group of independent
// clusters goes out in one launch: tiles carry their job index)
struct PanelJob {
    const double *L;   // BK factor (shift 0), row-major, ld = ldl
    int64_t lstride;
    const int *perm;   // [shift][pstride]
    const double *dinfo;
    int64_t pstride;
    double *W, *X;     // outputs (shift 0), ld = ldw
    int64_t wstride;
    int ldl, n, ldw, lcw;
};

// one cluster of a multi-cluster symmetric Schur update (k_gemm.cu)
struct SchurTarget;
struct SchurJob {
    const double *X, *Bg;
    int64_t sx;
    int ld, R, K, nseg;
    const int *seg_of, *seg_start;
    const struct SchurTarget *tbl;
    int tile0;         // first grid tile of the job
    int pad;
};

// recompression jobs (k_qr.cu / k_rrqr.cu / k_copy.cu): one cluster each
struct PqrJob {
    double *M;          // Gram matrix (shift 0); reflectors overwrite its rows
    int64_t mstride;
    double *tau;
    int *piv;
    int64_t vstride;
    double *QT;         // Q^T output (form_q_rows)
    int64_t qstride;
    int n, kmax;        // kmax: leading pivots to order (<= n)
};
struct RankJob {
    const double *DT;   // c x n (shift 0)
    int64_t dstride;
    double *part;       // [shift][nchunk][n]
    int *rank, *r1;     // [shift] each (r1 may be null)
    double *dropped;    // [shift]
    int c, n;
};
struct SumJob {
    const double *in;
    int64_t zin, pstride;
    double *out;
    int64_t zout, count;
    int nparts, pad;
};
// zero, per shift z, rows (orient 0) or columns (orient 1) [base + rank[z], base + t)
// of a block: the directions a shift's own rank drops although the wave keeps them
struct TailZeroJob {
    double *p;
    int64_t bs;
    const int *rank;    // [shift]
    int ld, other, base, t, orient, pad;  // other: extent of the untouched dimension
};

// Engine-mode BK job: factor the leading n x n block of a (row-major, ld).
struct BkJob {
    double *a;
    int64_t astride;
    int ld;
    int n;
    int *perm;       // [shift][pstride]
    double *dinfo;   // [shift][3*pstride]: d, e (2x2 off-diagonal), block size
    int64_t pstride;
};

// Opt a kernel into the largest dynamic shared memory once per (kernel, device),
// before its first launch.  Setting function attributes while another host
// thread launches the same kernel is avoided entirely (waves run concurrently).
template <class F>
inline cudaError_t smem_optin(F *f) {
    static std::mutex mu;
    static std::set<std::pair<const void *, int>> done;
    int dev = 0;
    cudaError_t e = cudaGetDevice(&dev);
    if (e != cudaSuccess) return e;
    std::lock_guard<std::mutex> g(mu);
    const auto key = std::make_pair((const void *)f, dev);
    if (done.count(key)) return cudaSuccess;
    int optin = 0;
    e = cudaDeviceGetAttribute(&optin, cudaDevAttrMaxSharedMemoryPerBlockOptin, dev);
    if (e != cudaSuccess) return e;
    cudaFuncAttributes fa;
    e = cudaFuncGetAttributes(&fa, f);
    if (e != cudaSuccess) return e;
    e = cudaFuncSetAttribute(f, cudaFuncAttributeMaxDynamicSharedMemorySize,
                             optin - (int)fa.sharedSizeBytes);
    if (e == cudaSuccess) done.insert(key);
    return e;
}

// ---- launchers (stream-ordered; return the launch error)
int copy_tiles(int rows, int cols);
void launch_copy_prefixed(const CopyTask *dev_tasks, const int *dev_prefix, int ntasks,
                          int total_tiles, int nshift, const double *mu, cudaStream_t st);

// target of one segment pair (a <= b) of the symmetric Schur update: element
// (ra, cb) lives at base + z*bs + (trans ? cb*ldc + ra : ra*ldc + cb)
struct SchurTarget {
    double *base;
    int64_t bs;
    int ldc, trans;
};
int schur_sym_tiles(int R);

// fire-and-forget global fp64 add (RED.E.ADD.F64 in L2)
__device__ __forceinline__ void red_add_f64(double *p, double v) {
    asm volatile("red.global.add.f64 [%0], %1;" ::"l"(__cvta_generic_to_global(p)), "d"(v) : "memory");
}

// one cluster of the INT8-tensor-core (Ozaki) Schur update (k_schur_oz.cu): its
// X / Bg rows are packed at rows [row0, row0 + round_up(R, 128)) of the slice buffers
struct OzJob {
    const double *X, *Bg;
    int64_t sx;
    int ld, R, K, nseg;
    const int *seg_of, *seg_start;
    const SchurTarget *tbl;
    int row0;          // first packed row
    int tile0;         // first grid tile
};
int schur_oz_tiles(int R);
void schur_oz_tile_order(int R, int job, std::vector<int2> &out);
size_t schur_oz_scratch_bytes(int rows_total, int kpad, int nshift);
cudaError_t launch_schur_oz(const OzJob *jobs, const int *row_job, const int2 *tile_ij,
                            int rows_total, int kpad, int total_tiles, int nshift, void *scratch,
                            cudaStream_t st, int probe = 0);
void oz_prof_fetch(unsigned long long *out, bool reset);  // probe 8 phase counters (16 values)
void launch_schur_sym(const double *X, const double *Bg, int64_t sx, int ld, int R, int K,
                      const int *seg_of, const int *seg_start, int nseg, const SchurTarget *tbl,
                      int nshift, cudaStream_t st, int variant = 0);
// several independent clusters in one launch: tile_job[t] = job of grid tile t
void launch_schur_sym_multi(const SchurJob *jobs, const int *tile_job, int total_tiles,
                            int nshift, cudaStream_t st);
void launch_sum_partials_multi(const SumJob *jobs, int njobs, int64_t max_count, int nshift,
                               cudaStream_t st);
cudaError_t launch_tail_zero(const TailZeroJob *jobs, int njobs, int nshift, cudaStream_t st);
void launch_sum_partials(const double *in, int64_t zin, int64_t pstride, int nparts, double *out,
                         int64_t zout, int64_t count, int nshift, cudaStream_t st);
int gemm_tiles(int M, int N);
void launch_gemm(const GemmTask *dev_tasks, const int *dev_tile_prefix, int ntasks,
                 int total_tiles, int nshift, cudaStream_t st, bool schur = false,
                 const int *dev_tile_task = nullptr);

// cluster BK for fronts above the single-CTA shared-memory size (k_bk_cluster.cu)
int bk_cluster_size(int n);
cudaError_t launch_bk_cluster(const BkJob *dev_jobs, int njobs, int nshift, int n, int64_t *counts,
                              int *status, cudaStream_t st);
int64_t bk_scratch_doubles(int n);
cudaError_t launch_bk_engine(const BkJob *dev_jobs, int njobs, int nshift, int nmax,
                             int64_t *counts, int *status, double *scratch,
                             int64_t scratch_stride, cudaStream_t st);
cudaError_t launch_bk_kat(double *a, int n, int count, const double *tol, int64_t *ipiv,
                          int64_t *info, double *scratch, cudaStream_t st);
cudaError_t launch_bk_inertia(const double *a, int n, int count, const int64_t *ipiv,
                              const double *zero_tol, int64_t *counts, cudaStream_t st);

cudaError_t launch_panel(const PanelTile *dev_tiles, int ntiles, int nshift, const double *L,
                         int64_t lstride, int ldl, int n, const int *perm, const double *dinfo,
                         int64_t pstride, double *W, double *X, int64_t wstride, int ldw,
                         cudaStream_t st);
// multi-cluster panel: tiles index `jobs`; smem_bytes = max panel_smem_bytes(n) over jobs
size_t panel_smem_bytes(int n);
int panel_lcw(int n);
cudaError_t launch_panel_multi(const PanelTile *dev_tiles, int ntiles, int nshift,
                               const PanelJob *dev_jobs, size_t smem_bytes, cudaStream_t st);

cudaError_t launch_pqr(double *GT, int64_t gstride, int c, int nR, int ldg, double *tau, int *piv,
                       int *used, double *norms, int64_t vstride, int64_t cstride,
                       const double *tol, int *rank, double *dropped, const int *active,
                       int target, int nshift, cudaStream_t st);
cudaError_t launch_tail_rank(const double *DT, int64_t dstride, int c, int n, double *part,
                             const double *tol, int *rank, double *dropped, int *r1out,
                             const int *active, int nshift, cudaStream_t st);
int64_t tail_rank_part_doubles(int c, int n);
// cluster-parallel full pivoted QR of an n x n Gram matrix (reflectors to rows of M)
int pqr_cluster_size(int n);
// kmax / kref <= 0: all n pivots / reflectors
cudaError_t launch_pqr_cluster(double *M, int64_t mstride, int n, double *tau, int *piv,
                               int64_t vstride, const int *active, int nshift, cudaStream_t st,
                               int kmax = 0);
cudaError_t launch_form_q_rows(const double *V, int64_t vstride, int n, const double *tau,
                               int64_t tstride, double *QT, int64_t qstride, const int *active,
                               int nshift, cudaStream_t st, int kref = 0);
// multi-cluster versions: nmax = largest n over the jobs (sizes shared memory / grid)
cudaError_t launch_pqr_cluster_multi(const PqrJob *jobs, int njobs, int nmax, const int *active,
                                     int nshift, cudaStream_t st);
cudaError_t launch_form_q_rows_multi(const PqrJob *jobs, int njobs, int nmax, const int *active,
                                     int nshift, cudaStream_t st);
cudaError_t launch_tail_rank_multi(const RankJob *jobs, int njobs, int cmax, int nmax,
                                   const double *tol, const int *active, int nshift,
                                   cudaStream_t st);
cudaError_t launch_form_tr(const double *GT, int64_t gstride, int ldg, const double *tau,
                           const int *piv, int64_t vstride, int nR, int t, double *Tr,
                           int64_t tstride, const int *active, int nshift, cudaStream_t st);

}  // namespace h2l
