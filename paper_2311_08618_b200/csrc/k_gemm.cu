// Grouped + shift-batched fp64 GEMM on the FP64 tensor pipe (DMMA).
//
// Blackwell has no fp64 tcgen05 kind (SURVEY.md finding 7: ptxas rejects
// .kind::f64), so the double-precision tensor path on sm_100a is
// mma.sync.m8n8k4.f64 -> DMMA.8x8x4 SASS.  This kernel serves every dense
// product of the elimination: the Schur-complement updates
// (target -= X_a W_b^T, gldl.py:388-409), the panel products, the
// recompression rotations (gldl.py:313-331), the merge congruences Q^T R Q
// (gldl.py:523-545) and the skeleton prologue Q^T A Q (compress.py:99-127).
//
// Tiling: one CTA computes a 64x64 tile of one task for one shift with 4
// warps (2x2), each warp a 32x32 sub-tile = 4x4 DMMA fragments.  The C
// fragments of the read-modify-write target are prefetched into registers
// before the K loop (the K extent of a Schur update is only n_R ~ 100-400,
// so an exposed epilogue load would dominate).  K advances in chunks of 16 through a 3-stage cp.async
// pipeline (global -> shared without register staging; out-of-range
// elements zero-filled by the copy), shared rows padded to 20 doubles so
// fragment reads are conflict-free.  Tasks are flattened into one grid
// through a tile prefix array: thousands of small blocks of one elimination
// step go out in a single launch; gridDim.y enumerates shifts.
#include "common.cuh"

namespace h2l {

namespace {

constexpr int BM = 64, BN = 64, BK = 16, SK = BK + 4, STAGES = 3;
constexpr int FM = BM / 16;  // DMMA fragments per warp along M (warp tile (BM/2) x 32)

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

__device__ __forceinline__ void cp_async8(void *smem, const void *gmem, bool pred) {
    const unsigned s = (unsigned)__cvta_generic_to_shared(smem);
    const int bytes = pred ? 8 : 0;
    asm volatile("cp.async.ca.shared.global [%0], [%1], 8, %2;\n" ::"r"(s), "l"(gmem), "r"(bytes));
}
__device__ __forceinline__ void cp_commit() { asm volatile("cp.async.commit_group;\n" ::); }
template <int N>
__device__ __forceinline__ void cp_wait() { asm volatile("cp.async.wait_group %0;\n" ::"n"(N)); }

// Stage the ROWS x 16 chunk of op(X) starting at (row0, k0) into S[ROWS][SK].
// op: element (r, k) = trans ? X[k*ld + r] : X[r*ld + k]
template <int ROWS>
__device__ __forceinline__ void load_chunk(double (*S)[SK], const double *X, int ld, int trans,
                                           int rows, int K, int row0, int k0, int tid) {
    constexpr int PER = ROWS * BK / 128;
    if (!trans) {
        const int k = k0 + (tid & 15);
#pragma unroll
        for (int i = 0; i < PER; ++i) {
            const int rl = (tid >> 4) + 8 * i;
            const int r = row0 + rl;
            const bool ok = r < rows && k < K;
            cp_async8(&S[rl][tid & 15], ok ? X + (int64_t)r * ld + k : X, ok);
        }
    } else {
        constexpr int RSTEP = 128 / ROWS;  // k rows covered per pass
#pragma unroll
        for (int i = 0; i < PER; ++i) {
            const int rl = tid % ROWS;
            const int kl = tid / ROWS + RSTEP * i;
            const int r = row0 + rl, k = k0 + kl;
            const bool ok = r < rows && k < K;
            cp_async8(&S[rl][kl], ok ? X + (int64_t)k * ld + r : X, ok);
        }
    }
}

__global__ void __launch_bounds__(128) gemm_kernel(const GemmTask *tasks, const int *prefix,
                                                   int ntasks) {
    extern __shared__ __align__(16) double gsm[];
    double (*As)[BM][SK] = reinterpret_cast<double (*)[BM][SK]>(gsm);
    double (*Bs)[BN][SK] = reinterpret_cast<double (*)[BN][SK]>(gsm + STAGES * BM * SK);

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
    const int wm = (warp >> 1) * (BM / 2), wn = (warp & 1) * 32;
    // opB element (k, n): tB=1 -> B[n*ldb+k] (rows of B are n) ; tB=0 -> B[k*ldb+n]
    const int b_trans = tk.tB ? 0 : 1;

    double acc[FM][4][2];
#pragma unroll
    for (int i = 0; i < FM; ++i)
#pragma unroll
        for (int j = 0; j < 4; ++j) acc[i][j][0] = acc[i][j][1] = 0.0;
    // prefetch the C fragments (beta != 0): the loads overlap the whole K loop
    const bool rd = tk.beta != 0.0;
    double cpre[FM][4][2];
#pragma unroll
    for (int i = 0; i < FM; ++i) {
        const int r = m0 + wm + i * 8 + (lane >> 2);
#pragma unroll
        for (int j = 0; j < 4; ++j) {
            const int c = n0 + wn + j * 8 + 2 * (lane & 3);
            const double *p = C + (int64_t)r * tk.ldc + c;
            cpre[i][j][0] = (rd && r < tk.M && c < tk.N) ? p[0] : 0.0;
            cpre[i][j][1] = (rd && r < tk.M && c + 1 < tk.N) ? p[1] : 0.0;
        }
    }

    const int nk = (tk.K + BK - 1) / BK;
#pragma unroll
    for (int s = 0; s < STAGES - 1; ++s) {
        if (s < nk) {
            load_chunk<BM>(As[s], A, tk.lda, tk.tA, tk.M, tk.K, m0, s * BK, tid);
            load_chunk<BN>(Bs[s], B, tk.ldb, b_trans, tk.N, tk.K, n0, s * BK, tid);
        }
        cp_commit();
    }
    for (int kc = 0; kc < nk; ++kc) {
        cp_wait<STAGES - 2>();
        __syncthreads();
        const int nxt = kc + STAGES - 1;
        if (nxt < nk) {
            const int sl = nxt % STAGES;
            load_chunk<BM>(As[sl], A, tk.lda, tk.tA, tk.M, tk.K, m0, nxt * BK, tid);
            load_chunk<BN>(Bs[sl], B, tk.ldb, b_trans, tk.N, tk.K, n0, nxt * BK, tid);
        }
        cp_commit();
        const int cur = kc % STAGES;
#pragma unroll
        for (int kk = 0; kk < BK; kk += 4) {
            double af[FM], bf[4];
#pragma unroll
            for (int i = 0; i < FM; ++i) af[i] = As[cur][wm + i * 8 + (lane >> 2)][kk + (lane & 3)];
#pragma unroll
            for (int j = 0; j < 4; ++j) bf[j] = Bs[cur][wn + j * 8 + (lane >> 2)][kk + (lane & 3)];
#pragma unroll
            for (int i = 0; i < FM; ++i)
#pragma unroll
                for (int j = 0; j < 4; ++j) dmma(acc[i][j][0], acc[i][j][1], af[i], bf[j]);
        }
    }
    cp_wait<0>();

    // epilogue: C = alpha*acc + beta*C (C already in registers)
#pragma unroll
    for (int i = 0; i < FM; ++i) {
        const int r = m0 + wm + i * 8 + (lane >> 2);
        if (r >= tk.M) continue;
        double *crow = C + (int64_t)r * tk.ldc;
#pragma unroll
        for (int j = 0; j < 4; ++j) {
            const int c = n0 + wn + j * 8 + 2 * (lane & 3);
            if (c < tk.N) crow[c] = tk.alpha * acc[i][j][0] + tk.beta * cpre[i][j][0];
            if (c + 1 < tk.N) crow[c + 1] = tk.alpha * acc[i][j][1] + tk.beta * cpre[i][j][1];
        }
    }
}

constexpr size_t GEMM_SMEM = sizeof(double) * STAGES * (BM + BN) * SK;

}  // namespace

int gemm_tiles(int M, int N) {
    if (M <= 0 || N <= 0) return 0;
    return ((M + BM - 1) / BM) * ((N + BN - 1) / BN);
}

void launch_gemm(const GemmTask *dev_tasks, const int *dev_tile_prefix, int ntasks,
                 int total_tiles, int nshift, cudaStream_t st) {
    if (ntasks <= 0 || total_tiles <= 0 || nshift <= 0) return;
    cudaFuncSetAttribute(gemm_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)GEMM_SMEM);
    dim3 grid(total_tiles, nshift);
    gemm_kernel<<<grid, 128, GEMM_SMEM, st>>>(dev_tasks, dev_tile_prefix, ntasks);
}

}  // namespace h2l
