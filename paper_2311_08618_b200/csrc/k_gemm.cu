// Grouped + shift-batched fp64 GEMM on the FP64 tensor pipe (DMMA).
//
// Blackwell has no fp64 tcgen05 kind (SURVEY.md finding 7: ptxas rejects
// .kind::f64), so the double-precision tensor path on sm_100a is
// mma.sync.m8n8k4.f64 -> DMMA.8x8x4 SASS.  This kernel serves every dense
// product of the elimination: the Schur-complement updates
// (target -= X_a W_b^T, gldl.py:388-409), the recompression rotations
// (gldl.py:313-331), the merge congruences Q^T R Q (gldl.py:523-545) and the
// skeleton prologue Q^T A Q (compress.py:99-127).
//
// Tiling: one CTA computes a 64x64 tile of one task for one shift with 4
// warps (2x2), each warp a 32x32 sub-tile = 4x4 DMMA fragments (32 fp64
// accumulators / thread).  K advances in chunks of 16 through a register-
// staged double buffer in shared memory (row stride 20 doubles: conflict-free
// fragment reads).  Tasks are flattened into one grid through a tile prefix
// array, so thousands of small blocks of one elimination step go out in a
// single launch; gridDim.y enumerates shifts.
#include "common.cuh"

namespace h2l {

namespace {

constexpr int BM = 64, BN = 64, BK = 16, SK = BK + 4;

__device__ __forceinline__ int find_task(const int *prefix, int ntasks, int tile) {
    int lo = 0, hi = ntasks - 1;
    while (lo < hi) {
        int mid = (lo + hi + 1) >> 1;
        if (prefix[mid] <= tile) lo = mid; else hi = mid - 1;
    }
    return lo;
}

__device__ __forceinline__ void dmma(double &c0, double &c1, double a, double b) {
    asm volatile("mma.sync.aligned.m8n8k4.row.col.f64.f64.f64.f64 {%0,%1}, {%2}, {%3}, {%0,%1};\n"
                 : "+d"(c0), "+d"(c1)
                 : "d"(a), "d"(b));
}

// Load the 64x16 chunk of op(X) starting at (row0, k0) into registers.
// op: element (r, k) = trans ? X[k*ld + r] : X[r*ld + k]
__device__ __forceinline__ void load_chunk(double (&reg)[8], const double *X, int ld, int trans,
                                           int rows, int K, int row0, int k0, int tid) {
    if (!trans) {
        const int k = k0 + (tid & 15);
#pragma unroll
        for (int i = 0; i < 8; ++i) {
            const int r = row0 + (tid >> 4) + 8 * i;
            reg[i] = (r < rows && k < K) ? __ldg(X + (int64_t)r * ld + k) : 0.0;
        }
    } else {
        const int r = row0 + (tid & 63);
#pragma unroll
        for (int i = 0; i < 8; ++i) {
            const int k = k0 + (tid >> 6) + 2 * i;
            reg[i] = (r < rows && k < K) ? __ldg(X + (int64_t)k * ld + r) : 0.0;
        }
    }
}

__device__ __forceinline__ void store_chunk(double (*S)[SK], const double (&reg)[8], int trans,
                                            int tid) {
    if (!trans) {
#pragma unroll
        for (int i = 0; i < 8; ++i) S[(tid >> 4) + 8 * i][tid & 15] = reg[i];
    } else {
#pragma unroll
        for (int i = 0; i < 8; ++i) S[tid & 63][(tid >> 6) + 2 * i] = reg[i];
    }
}

__global__ void __launch_bounds__(128) gemm_kernel(const GemmTask *tasks, const int *prefix,
                                                   int ntasks) {
    __shared__ __align__(16) double As[2][BM][SK];
    __shared__ __align__(16) double Bs[2][BN][SK];

    const int t = find_task(prefix, ntasks, blockIdx.x);
    const GemmTask tk = tasks[t];
    const int local = blockIdx.x - prefix[t];
    const int tiles_n = (tk.N + BN - 1) / BN;
    const int m0 = (local / tiles_n) * BM;
    const int n0 = (local % tiles_n) * BN;
    const int z = blockIdx.y;
    const double *A = tk.A + z * tk.sA;
    const double *B = tk.B + z * tk.sB;
    double *C = tk.C + z * tk.sC;

    const int tid = threadIdx.x;
    const int lane = tid & 31, warp = tid >> 5;
    const int wm = (warp >> 1) * 32, wn = (warp & 1) * 32;
    // opB element (k, n): tB=1 -> B[n*ldb+k] (rows of B are n) ; tB=0 -> B[k*ldb+n]
    const int b_trans = tk.tB ? 0 : 1;

    double acc[4][4][2];
#pragma unroll
    for (int i = 0; i < 4; ++i)
#pragma unroll
        for (int j = 0; j < 4; ++j) acc[i][j][0] = acc[i][j][1] = 0.0;

    double ra[8], rb[8];
    const int nk = (tk.K + BK - 1) / BK;
    if (nk > 0) {
        load_chunk(ra, A, tk.lda, tk.tA, tk.M, tk.K, m0, 0, tid);
        load_chunk(rb, B, tk.ldb, b_trans, tk.N, tk.K, n0, 0, tid);
        store_chunk(As[0], ra, tk.tA, tid);
        store_chunk(Bs[0], rb, b_trans, tid);
    }
    __syncthreads();
    for (int kc = 0; kc < nk; ++kc) {
        const int cur = kc & 1;
        if (kc + 1 < nk) {
            load_chunk(ra, A, tk.lda, tk.tA, tk.M, tk.K, m0, (kc + 1) * BK, tid);
            load_chunk(rb, B, tk.ldb, b_trans, tk.N, tk.K, n0, (kc + 1) * BK, tid);
        }
#pragma unroll
        for (int kk = 0; kk < BK; kk += 4) {
            double af[4], bf[4];
#pragma unroll
            for (int i = 0; i < 4; ++i) af[i] = As[cur][wm + i * 8 + (lane >> 2)][kk + (lane & 3)];
#pragma unroll
            for (int j = 0; j < 4; ++j) bf[j] = Bs[cur][wn + j * 8 + (lane >> 2)][kk + (lane & 3)];
#pragma unroll
            for (int i = 0; i < 4; ++i)
#pragma unroll
                for (int j = 0; j < 4; ++j) dmma(acc[i][j][0], acc[i][j][1], af[i], bf[j]);
        }
        if (kc + 1 < nk) {
            store_chunk(As[cur ^ 1], ra, tk.tA, tid);
            store_chunk(Bs[cur ^ 1], rb, b_trans, tid);
        }
        __syncthreads();
    }

    // epilogue: C = alpha*acc + beta*C
#pragma unroll
    for (int i = 0; i < 4; ++i) {
        const int r = m0 + wm + i * 8 + (lane >> 2);
        if (r >= tk.M) continue;
#pragma unroll
        for (int j = 0; j < 4; ++j) {
            const int c = n0 + wn + j * 8 + 2 * (lane & 3);
            double *p = C + (int64_t)r * tk.ldc + c;
            if (c < tk.N) p[0] = tk.alpha * acc[i][j][0] + (tk.beta != 0.0 ? tk.beta * p[0] : 0.0);
            if (c + 1 < tk.N) p[1] = tk.alpha * acc[i][j][1] + (tk.beta != 0.0 ? tk.beta * p[1] : 0.0);
        }
    }
}

}  // namespace

int gemm_tiles(int M, int N) {
    if (M <= 0 || N <= 0) return 0;
    return ((M + BM - 1) / BM) * ((N + BN - 1) / BN);
}

void launch_gemm(const GemmTask *dev_tasks, const int *dev_tile_prefix, int ntasks,
                 int total_tiles, int nshift, cudaStream_t st) {
    if (ntasks <= 0 || total_tiles <= 0 || nshift <= 0) return;
    dim3 grid(total_tiles, nshift);
    gemm_kernel<<<grid, 128, 0, st>>>(dev_tasks, dev_tile_prefix, ntasks);
}

}  // namespace h2l
