// DMMA GEMM tile machinery shared by k_gemm.cu (the product kernels) and
// k_gemm_variants.cu (tile variants of the benchmarking library).  Everything
// here has internal linkage: each translation unit instantiates what it launches.
#pragma once

#include "common.cuh"

namespace h2l {

namespace {


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

template <int BM_, int BN_, int WM_, int WN_, int STAGES_, bool CSTAGE_ = true, int MINB_ = 1,
          int BK_ = 16, bool KP_ = false>
struct GemmCfg {
    static constexpr int BM = BM_, BN = BN_, WM = WM_, WN = WN_, STAGES = STAGES_;
    // KP: k permuted inside a 16-chunk (position (k % 4) * 4 + k / 4) so a lane's
    // fragments of the 4 DMMA k-steps are contiguous: 2 LDS.128 instead of 4
    // LDS.64 per fragment; row stride 18 keeps the 128-bit loads conflict-free
    static constexpr bool KP = KP_;
    static_assert(!KP_ || BK_ == 16, "k permutation defined for 16-chunks");
    static constexpr int BK = BK_, SK = KP_ ? BK_ + 2 : BK_ + 4;  // K chunk; padded shared row
    static constexpr bool CSTAGE = CSTAGE_;  // prefetch C into shared memory
    static constexpr int MINB = MINB_;       // min resident CTAs per SM (register cap)
    static constexpr int WARPS = (BM / WM) * (BN / WN);
    static constexpr int THREADS = WARPS * 32;
    static constexpr int FM = WM / 8, FN = WN / 8;
    static constexpr int CS = BN + 1;  // padded row stride of the staged C tile
    static constexpr size_t SMEM =
        sizeof(double) * ((size_t)STAGES * (BM + BN) * SK + (CSTAGE ? (size_t)BM * CS : 0));
};

// Per-thread staging plan of the ROWS x 16 chunks of op(X), element (r, k) =
// trans ? X[k*ld + r] : X[r*ld + k].  Thread tid copies the elements
// e = tid + q*THREADS (q < ROWS*16/THREADS) of every chunk; their global and
// shared addresses differ by fixed strides, so the pointers, row predicates
// and shared offsets are computed once per tile and each chunk costs one add.
template <int ROWS, int THREADS, int BK, int SK, bool KP = false>
struct Loader {
    static __device__ __forceinline__ int kpos(int k) { return KP ? (k & 3) * 4 + (k >> 2) : k; }
    static_assert(THREADS % ROWS == 0 && THREADS % BK == 0, "loader layout");
    static constexpr int NQ = ROWS * BK / THREADS;
    const double *p;        // element q = 0 of chunk 0
    int64_t dq, dk;         // pointer strides per q and per chunk (doubles)
    unsigned soff, sdq;     // shared byte offset of q = 0 and per-q stride
    unsigned rowok;         // bit q: row in range
    int kl0, kstep;         // k within the chunk of element q: kl0 + q * kstep
    __device__ __forceinline__ Loader(const double *X, int ld, int trans, int rows, int row0,
                                      int tid) {
        int rl0, rstep;
        if (!trans) {  // rows contiguous in k: consecutive threads walk k
            rl0 = tid / BK; rstep = THREADS / BK; kl0 = tid % BK; kstep = 0;
            p = X + (int64_t)(row0 + rl0) * ld + kl0;
            dq = (int64_t)rstep * ld; dk = BK;
        } else {       // columns contiguous in r: consecutive threads walk r
            rl0 = tid % ROWS; rstep = 0; kl0 = tid / ROWS; kstep = THREADS / ROWS;
            p = X + (int64_t)kl0 * ld + row0 + rl0;
            dq = (int64_t)kstep * ld; dk = (int64_t)BK * ld;
        }
        soff = (unsigned)((rl0 * SK + kpos(kl0)) * sizeof(double));
        sdq = (unsigned)((rstep * SK + kstep) * sizeof(double));  // KP: trans uses kpos per q
        rowok = 0;
#pragma unroll
        for (int q = 0; q < NQ; ++q) rowok |= (row0 + rl0 + q * rstep < rows) ? (1u << q) : 0u;
    }
    // stage chunk c (k0 = c*BK) into the shared buffer at byte address sbase
    __device__ __forceinline__ void load(unsigned sbase, int c, int K) const {
        const double *pc = p + c * dk;
        const int krem = K - c * BK;
#pragma unroll
        for (int q = 0; q < NQ; ++q) {
            const bool ok = ((rowok >> q) & 1u) && (kl0 + q * kstep < krem);
            const unsigned so = (KP && kstep)
                ? soff + (unsigned)((kpos(kl0 + q * kstep) - kpos(kl0)) * sizeof(double))
                : soff + q * sdq;
            // src-size 0 (zero fill) reads nothing, so the address needs no clamp
            asm volatile("cp.async.ca.shared.global.L2::128B [%0], [%1], 8, %2;\n"
                         ::"r"(sbase + so), "l"(pc + q * dq), "r"(ok ? 8 : 0));
        }
    }
};

// K loop of one BM x BN tile: acc += op(A)[m0:, :] op(B)[:, n0:] (cp.async
// pipeline, DMMA.8x8x4).  Shared by the grouped GEMM and the Schur kernel.
template <class Cfg>
__device__ __forceinline__ void tile_mainloop(const double *A, int lda, int tA, int M,
                                              const double *B, int ldb, int b_trans, int N, int K,
                                              int m0, int n0, int wm, int wn,
                                              double (&acc)[Cfg::FM][Cfg::FN][2]) {
    constexpr int BM = Cfg::BM, BN = Cfg::BN, STAGES = Cfg::STAGES, FM = Cfg::FM, FN = Cfg::FN;
    constexpr int BK = Cfg::BK, SK = Cfg::SK, THREADS = Cfg::THREADS;
    extern __shared__ __align__(16) double gsm[];
    double (*As)[BM][SK] = reinterpret_cast<double (*)[BM][SK]>(gsm);
    double (*Bs)[BN][SK] = reinterpret_cast<double (*)[BN][SK]>(gsm + STAGES * BM * SK);
    const int tid = threadIdx.x, lane = tid & 31;
#pragma unroll
    for (int i = 0; i < FM; ++i)
#pragma unroll
        for (int j = 0; j < FN; ++j) acc[i][j][0] = acc[i][j][1] = 0.0;
    const int nk = (K + BK - 1) / BK;
    const Loader<BM, THREADS, BK, SK, Cfg::KP> la(A, lda, tA, M, m0, tid);
    const Loader<BN, THREADS, BK, SK, Cfg::KP> lb(B, ldb, b_trans, N, n0, tid);
    const unsigned sA = (unsigned)__cvta_generic_to_shared(&As[0][0][0]);
    const unsigned sB = (unsigned)__cvta_generic_to_shared(&Bs[0][0][0]);
    constexpr unsigned SA_STAGE = BM * SK * sizeof(double), SB_STAGE = BN * SK * sizeof(double);
#pragma unroll
    for (int s = 0; s < STAGES - 1; ++s) {
        if (s < nk) {
            la.load(sA + s * SA_STAGE, s, K);
            lb.load(sB + s * SB_STAGE, s, K);
        }
        cp_commit();
    }
    for (int kc = 0; kc < nk; ++kc) {
        cp_wait<STAGES - 2>();
        __syncthreads();
        const int nxt = kc + STAGES - 1;
        if (nxt < nk) {
            const int sl = nxt % STAGES;
            la.load(sA + sl * SA_STAGE, nxt, K);
            lb.load(sB + sl * SB_STAGE, nxt, K);
        }
        cp_commit();
        const int cur = kc % STAGES;
        if constexpr (Cfg::KP) {
            // same accumulation order as below (k-steps 0, 4, 8, 12): bitwise identical
#pragma unroll
            for (int hp = 0; hp < 2; ++hp) {
                double2 af[FM], bf[FN];
#pragma unroll
                for (int i = 0; i < FM; ++i)
                    af[i] = *reinterpret_cast<const double2 *>(
                        &As[cur][wm + i * 8 + (lane >> 2)][(lane & 3) * 4 + 2 * hp]);
#pragma unroll
                for (int j = 0; j < FN; ++j)
                    bf[j] = *reinterpret_cast<const double2 *>(
                        &Bs[cur][wn + j * 8 + (lane >> 2)][(lane & 3) * 4 + 2 * hp]);
#pragma unroll
                for (int i = 0; i < FM; ++i)
#pragma unroll
                    for (int j = 0; j < FN; ++j) dmma(acc[i][j][0], acc[i][j][1], af[i].x, bf[j].x);
#pragma unroll
                for (int i = 0; i < FM; ++i)
#pragma unroll
                    for (int j = 0; j < FN; ++j) dmma(acc[i][j][0], acc[i][j][1], af[i].y, bf[j].y);
            }
        } else {
#pragma unroll
        for (int kk = 0; kk < BK; kk += 4) {
            double af[FM], bf[FN];
#pragma unroll
            for (int i = 0; i < FM; ++i) af[i] = As[cur][wm + i * 8 + (lane >> 2)][kk + (lane & 3)];
#pragma unroll
            for (int j = 0; j < FN; ++j) bf[j] = Bs[cur][wn + j * 8 + (lane >> 2)][kk + (lane & 3)];
#pragma unroll
            for (int i = 0; i < FM; ++i)
#pragma unroll
                for (int j = 0; j < FN; ++j) dmma(acc[i][j][0], acc[i][j][1], af[i], bf[j]);
        }
        }
    }
    cp_wait<0>();
    __syncthreads();
}

template <class Cfg>
__device__ __forceinline__ void gemm_body(const GemmTask *tasks, const int *prefix, int ntasks,
                                          const int *tile_task) {
    constexpr int BM = Cfg::BM, BN = Cfg::BN, STAGES = Cfg::STAGES, FM = Cfg::FM, FN = Cfg::FN;
    constexpr int SK = Cfg::SK;
    constexpr int THREADS = Cfg::THREADS, CS = Cfg::CS;
    extern __shared__ __align__(16) double gsm[];
    double *Cs = gsm + STAGES * (BM + BN) * SK;

    // tile -> task: one load from the staged map (large launches) or a binary
    // search of the tile prefix (small ones)
    const int t = tile_task ? tile_task[blockIdx.x] : find_task(prefix, ntasks, blockIdx.x);
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
    constexpr int WCOLS = BN / Cfg::WN;
    const int wm = (warp / WCOLS) * Cfg::WM, wn = (warp % WCOLS) * Cfg::WN;
    const int b_trans = tk.tB ? 0 : 1;
    const bool rd = tk.beta != 0.0;

    // C prefetch (own cp.async group, completes with the first K stage)
    if (Cfg::CSTAGE && rd) {
        for (int e = tid; e < BM * BN; e += THREADS) {
            const int rl = e / BN, cl = e % BN;
            const int r = m0 + rl, c = n0 + cl;
            const bool ok = r < tk.M && c < tk.N;
            cp_async8(&Cs[rl * CS + cl], ok ? C + (int64_t)r * tk.ldc + c : C, ok);
        }
    }
    cp_commit();

    double acc[FM][FN][2];
    tile_mainloop<Cfg>(A, tk.lda, tk.tA, tk.M, B, tk.ldb, b_trans, tk.N, tk.K, m0, n0, wm, wn, acc);

    // epilogue: C = alpha*acc + beta*C
    if (Cfg::CSTAGE) {
#pragma unroll
        for (int i = 0; i < FM; ++i) {
            const int rl = wm + i * 8 + (lane >> 2);
            const int r = m0 + rl;
            if (r >= tk.M) continue;
            double *crow = C + (int64_t)r * tk.ldc;
#pragma unroll
            for (int j = 0; j < FN; ++j) {
                const int cl = wn + j * 8 + 2 * (lane & 3);
                const int c = n0 + cl;
                if (c < tk.N)
                    crow[c] = tk.alpha * acc[i][j][0] + (rd ? tk.beta * Cs[rl * CS + cl] : 0.0);
                if (c + 1 < tk.N)
                    crow[c + 1] = tk.alpha * acc[i][j][1] + (rd ? tk.beta * Cs[rl * CS + cl + 1] : 0.0);
            }
        }
    } else {
        // all loads of a fragment row group before its stores (no aliasing stalls)
#pragma unroll
        for (int i = 0; i < FM; ++i) {
            const int r = m0 + wm + i * 8 + (lane >> 2);
            if (r >= tk.M) continue;
            double *crow = C + (int64_t)r * tk.ldc;
            double cv[FN][2];
#pragma unroll
            for (int j = 0; j < FN; ++j) {
                const int c = n0 + wn + j * 8 + 2 * (lane & 3);
                cv[j][0] = (rd && c < tk.N) ? crow[c] : 0.0;
                cv[j][1] = (rd && c + 1 < tk.N) ? crow[c + 1] : 0.0;
            }
#pragma unroll
            for (int j = 0; j < FN; ++j) {
                const int c = n0 + wn + j * 8 + 2 * (lane & 3);
                if (c < tk.N) crow[c] = tk.alpha * acc[i][j][0] + tk.beta * cv[j][0];
                if (c + 1 < tk.N) crow[c + 1] = tk.alpha * acc[i][j][1] + tk.beta * cv[j][1];
            }
        }
    }
}

// K6 as one symmetric update per elimination step (engine.cu eliminate):
// C_big -= X Bg^T over the upper triangle of the R x R panel space, where X
// (R x K) and Bg (R x K) are the panel's rows stacked segment by segment.
// Tiles never straddle tasks, so no tile is padded except at the end of R (the
// per-pair task list padded every segment to a multiple of 64); the epilogue
// scatters element (r, c), r <= c, to its target block through the
// segment-pair table (diagonal segments also write the mirrored element).
// upper-triangular tile index -> (I <= J)
__device__ __forceinline__ void tri_tile(int t, int &I, int &J) {
    J = (int)((sqrt(8.0 * t + 1.0) - 1.0) * 0.5);
    while ((J + 1) * (J + 2) / 2 <= t) ++J;
    while (J * (J + 1) / 2 > t) --J;
    I = t - J * (J + 1) / 2;
}

template <class Cfg, bool ATOM = false>
__device__ __forceinline__ void schur_sym_epilogue(double (&acc)[Cfg::FM][Cfg::FN][2], int m0,
                                                   int n0, int z, int R, const int *seg_of,
                                                   const int *seg_start, int nseg,
                                                   const SchurTarget *tbl);
template <class Cfg>
__device__ __forceinline__ void schur_target_prefetch(int m0, int n0, int z, int R,
                                                      const int *seg_of, const int *seg_start,
                                                      const SchurTarget *tbl, int nseg);

template <class Cfg, int PF>
__device__ __forceinline__ void schur_sym_body(const double *X, const double *Bg, int64_t sx,
                                               int ld, int R, int K, const int *seg_of,
                                               const int *seg_start, int nseg,
                                               const SchurTarget *tbl) {
    constexpr int BM = Cfg::BM, BN = Cfg::BN, FM = Cfg::FM, FN = Cfg::FN;
    static_assert(BM == BN, "square tiles");
    const int tid = threadIdx.x, warp = tid >> 5;
    constexpr int WCOLS = BN / Cfg::WN;
    const int wm = (warp / WCOLS) * Cfg::WM, wn = (warp % WCOLS) * Cfg::WN;
    int I, J;
    tri_tile(blockIdx.x, I, J);
    const int z = blockIdx.y;
    if (PF & 1) schur_target_prefetch<Cfg>(I * BM, J * BN, z, R, seg_of, seg_start, tbl, nseg);
    double acc[FM][FN][2];
    tile_mainloop<Cfg>(X + z * sx, ld, 0, R, Bg + z * sx, ld, 0, R, K, I * BM, J * BN, wm, wn, acc);
    schur_sym_epilogue<Cfg, (PF & 2) != 0>(acc, I * BM, J * BN, z, R, seg_of, seg_start, nseg, tbl);
}

// L2 prefetch of a tile's target rows (variant 1): thread t covers row t / 2,
// columns (t % 2) * 32 .. +32, one prefetch per 8 columns, each address taken
// from its own segment pair (always inside the target block)
template <class Cfg>
__device__ __forceinline__ void schur_target_prefetch(int m0, int n0, int z, int R,
                                                      const int *seg_of, const int *seg_start,
                                                      const SchurTarget *tbl, int nseg) {
    const int tid = threadIdx.x;
    if (tid >= 2 * Cfg::BM) return;
    const int rl = tid >> 1, c0 = (tid & 1) * 32;
    const int r = m0 + rl;
    if (r >= R) return;
    const int a = seg_of[r], ra = r - seg_start[a];
    for (int c = c0; c < c0 + 32; c += 8) {
        const int cc = n0 + c;
        if (cc >= R || cc < r) continue;
        const int b = seg_of[cc];
        const SchurTarget e = tbl[(size_t)a * nseg + b];
        if (!e.base || e.trans) continue;
        const double *pp = e.base + z * e.bs + (int64_t)ra * e.ldc + (cc - seg_start[b]);
        asm volatile("prefetch.global.L2 [%0];" ::"l"(pp));
    }
}

template <class Cfg, bool ATOM>
__device__ __forceinline__ void schur_sym_epilogue(double (&acc)[Cfg::FM][Cfg::FN][2], int m0,
                                                   int n0, int z, int R, const int *seg_of,
                                                   const int *seg_start, int nseg,
                                                   const SchurTarget *tbl) {
    constexpr int BM = Cfg::BM, BN = Cfg::BN, FM = Cfg::FM, FN = Cfg::FN;
    const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
    constexpr int WCOLS = BN / Cfg::WN;
    const int wm = (warp / WCOLS) * Cfg::WM, wn = (warp % WCOLS) * Cfg::WN;
    // epilogue: the tile's row / column segments and the few segment-pair targets
    // it touches are resolved once into shared memory; then, like the grouped
    // GEMM, all target loads of a fragment row are issued before its stores
    constexpr int MAXT = 64;
    __shared__ int s_rseg[BM], s_roff[BM], s_cseg[BN], s_coff[BN], s_box[4];
    __shared__ SchurTarget s_tbl[MAXT];

    for (int q = tid; q < BM + BN; q += Cfg::THREADS) {
        const int x = q < BM ? m0 + q : n0 + (q - BM);
        const int sg = x < R ? seg_of[x] : -1;
        const int off = sg >= 0 ? x - seg_start[sg] : 0;
        if (q < BM) { s_rseg[q] = sg; s_roff[q] = off; }
        else { s_cseg[q - BM] = sg; s_coff[q - BM] = off; }
    }
    __syncthreads();
    if (tid == 0) {
        const int rl = min(BM, R - m0) - 1, cl = min(BN, R - n0) - 1;
        s_box[0] = s_rseg[0];
        s_box[1] = s_rseg[rl] - s_rseg[0] + 1;
        s_box[2] = s_cseg[0];
        s_box[3] = s_cseg[cl] - s_cseg[0] + 1;
    }
    __syncthreads();
    const int alo = s_box[0], na = s_box[1], blo = s_box[2], nb = s_box[3];
    const bool in_smem = na * nb <= MAXT;
    if (in_smem)
        for (int q = tid; q < na * nb; q += Cfg::THREADS)
            s_tbl[q] = tbl[(size_t)(alo + q / nb) * nseg + blo + q % nb];
    __syncthreads();
    auto entry = [&](int a, int b) -> SchurTarget {
        return in_smem ? s_tbl[(a - alo) * nb + (b - blo)] : tbl[(size_t)a * nseg + b];
    };
    if constexpr (ATOM) {
        // each target element receives exactly one update per launch, so a
        // fire-and-forget reduction in L2 (RED.ADD.F64) gives the same IEEE result
        // as load / subtract / store without a round trip in the epilogue
#pragma unroll
        for (int i = 0; i < FM; ++i) {
            const int rl = wm + i * 8 + (lane >> 2);
            const int r = m0 + rl, a = s_rseg[rl], ra = s_roff[rl];
            if (a < 0) continue;
#pragma unroll
            for (int j = 0; j < FN; ++j)
#pragma unroll
                for (int h = 0; h < 2; ++h) {
                    const int cl = wn + j * 8 + 2 * (lane & 3) + h;
                    const int b = s_cseg[cl], cb = s_coff[cl];
                    if (b < 0 || n0 + cl < r) continue;
                    const SchurTarget e = entry(a, b);
                    if (!e.base) continue;
                    double *p = e.base + z * e.bs + (e.trans ? (int64_t)cb * e.ldc + ra
                                                              : (int64_t)ra * e.ldc + cb);
                    red_add_f64(p, -acc[i][j][h]);
                    if (a == b && cb != ra) red_add_f64(e.base + z * e.bs + (int64_t)cb * e.ldc + ra,
                                                        -acc[i][j][h]);
                }
        }
    } else {
#pragma unroll
    for (int i = 0; i < FM; ++i) {
        const int rl = wm + i * 8 + (lane >> 2);
        const int r = m0 + rl, a = s_rseg[rl], ra = s_roff[rl];
        if (a < 0) continue;
        double *ptr[FN][2];
        double cv[FN][2];
#pragma unroll
        for (int j = 0; j < FN; ++j)
#pragma unroll
            for (int h = 0; h < 2; ++h) {
                const int cl = wn + j * 8 + 2 * (lane & 3) + h;
                const int b = s_cseg[cl], cb = s_coff[cl];
                ptr[j][h] = nullptr;
                cv[j][h] = 0.0;
                if (b < 0 || n0 + cl < r) continue;
                const SchurTarget e = entry(a, b);
                if (!e.base) continue;
                double *p = e.base + z * e.bs + (e.trans ? (int64_t)cb * e.ldc + ra
                                                          : (int64_t)ra * e.ldc + cb);
                ptr[j][h] = p;
                cv[j][h] = *p;
            }
#pragma unroll
        for (int j = 0; j < FN; ++j)
#pragma unroll
            for (int h = 0; h < 2; ++h)
                if (ptr[j][h]) *ptr[j][h] = cv[j][h] - acc[i][j][h];
    }
    // diagonal segment pairs: the mirrored element (a separate, rare pass)
#pragma unroll
    for (int i = 0; i < FM; ++i) {
        const int rl = wm + i * 8 + (lane >> 2);
        const int r = m0 + rl, a = s_rseg[rl], ra = s_roff[rl];
        if (a < 0) continue;
#pragma unroll
        for (int j = 0; j < FN; ++j)
#pragma unroll
            for (int h = 0; h < 2; ++h) {
                const int cl = wn + j * 8 + 2 * (lane & 3) + h;
                const int b = s_cseg[cl], cb = s_coff[cl];
                if (b != a || cb == ra || n0 + cl < r) continue;
                const SchurTarget e = entry(a, b);
                if (!e.base) continue;
                e.base[z * e.bs + (int64_t)cb * e.ldc + ra] -= acc[i][j][h];
            }
    }
    }
}

template <class Cfg>
__global__ void __launch_bounds__(Cfg::THREADS, Cfg::MINB) gemm_kernel(const GemmTask *tasks,
                                                            const int *prefix, int ntasks,
                                                            const int *tile_task) {
    gemm_body<Cfg>(tasks, prefix, ntasks, tile_task);
}
// same code under its own name so profiles separate the Schur updates (K6)
template <class Cfg>
__global__ void __launch_bounds__(Cfg::THREADS, Cfg::MINB) schur_gemm_kernel(const GemmTask *tasks,
                                                                  const int *prefix, int ntasks,
                                                            const int *tile_task) {
    gemm_body<Cfg>(tasks, prefix, ntasks, tile_task);
}

template <class Cfg, int PF>
__global__ void __launch_bounds__(Cfg::THREADS, Cfg::MINB) schur_sym_kernel(
    const double *X, const double *Bg, int64_t sx, int ld, int R, int K, const int *seg_of,
    const int *seg_start, int nseg, const SchurTarget *tbl) {
    schur_sym_body<Cfg, PF>(X, Bg, sx, ld, R, K, seg_of, seg_start, nseg, tbl);
}

// production configuration (chosen with tools/gemm_bench.py)
using Prod = GemmCfg<64, 64, 32, 32, 2, false, 4>;

// a group of independent clusters (disjoint Schur targets) in one launch: grid
// tile t belongs to job tile_job[t] and is its (t - tile0)-th upper-triangle tile
template <class Cfg>
__global__ void __launch_bounds__(Cfg::THREADS, Cfg::MINB) schur_sym_multi_kernel(
    const SchurJob *jobs, const int *tile_job) {
    constexpr int BM = Cfg::BM, BN = Cfg::BN, FM = Cfg::FM, FN = Cfg::FN;
    const SchurJob jb = jobs[tile_job[blockIdx.x]];
    const int tid = threadIdx.x, warp = tid >> 5;
    constexpr int WCOLS = BN / Cfg::WN;
    const int wm = (warp / WCOLS) * Cfg::WM, wn = (warp % WCOLS) * Cfg::WN;
    int I, J;
    tri_tile(blockIdx.x - jb.tile0, I, J);
    const int z = blockIdx.y;
    double acc[FM][FN][2];
    tile_mainloop<Cfg>(jb.X + z * jb.sx, jb.ld, 0, jb.R, jb.Bg + z * jb.sx, jb.ld, 0, jb.R, jb.K,
                       I * BM, J * BN, wm, wn, acc);
    schur_sym_epilogue<Cfg, true>(acc, I * BM, J * BN, z, jb.R, jb.seg_of, jb.seg_start, jb.nseg,
                                  jb.tbl);
}

template <class Cfg>
void launch_cfg(const GemmTask *dev_tasks, const int *dev_tile_prefix, int ntasks,
                int total_tiles, int nshift, cudaStream_t st) {
    smem_optin(gemm_kernel<Cfg>);
    dim3 grid(total_tiles, nshift);
    gemm_kernel<Cfg><<<grid, Cfg::THREADS, Cfg::SMEM, st>>>(dev_tasks, dev_tile_prefix, ntasks,
                                                             nullptr);
}

}  // namespace

}  // namespace h2l
