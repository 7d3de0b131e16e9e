// K6 Schur update  C_big -= X Bg^T  on the INT8 tensor cores (tcgen05.mma.kind::i8),
// fp64-accurate by exact integer slicing (the Ozaki scheme).
//
// Blackwell has no fp64 tcgen05 kind; the fp64 path is DMMA through mma.sync at
// ~37 TF/s (k_gemm.cu schur_sym_kernel).  The INT8 tensor pipe is 4.5 POPS dense nominal (cuBLASLt measures 3.0-3.1).
// Every row r of X (and of Bg) is written exactly as
//     x_rk = 2^e_r * sum_{p<8} 2^{-7(p+1)} s_rkp ,   s_rkp in [-127, 127]
// (e_r = exponent of the row's largest entry; each slice peels 7 bits; the residual
// after 8 slices is < 2^-56 of the row maximum, below fp64's 53-bit mantissa).
// Then (X Bg^T)_rc = 2^(e_r + e_c) sum_{i,j} 2^{-7(i+j+2)} (S_i T_j^T)_rc, each slice
// product exact in int32 (|sum| <= 127^2 K < 2^31 for K <= 2^17).  Pairs with
// i + j <= 7 are kept (36 of 64; the dropped tail is < 2^-63 of the row/column
// maxima), and all pairs of one i + j = g share one int32 accumulator in tensor
// memory: 8 groups x 64 columns = the SM's 512 TMEM columns.  The epilogue merges
// the 8 group totals exactly in int64, three at a time, sums the three fp64 terms
// (smallest first) and applies the row/column exponents; the only roundings are
// those of that final three-term sum -- fewer than the K-term fp64 dot product of
// the DMMA kernel.
//
// Kernel structure (persistent: one CTA of 10 warps per SM walks (shift, tile) items;
// tile = 128 x 64 of a cluster's upper triangle, fixed by the 512 TMEM columns):
//   warp 0      TMA producer: per 32-byte K block the 8 slices of 128 X rows and of 64 Bg
//               rows (8 x 4 KB + 8 x 2 KB = 48 KB, SWIZZLE_32B), 3 stages, running ahead
//               across items; the slice planes are stored [K block][row][32 bytes], so
//               a box is one contiguous run;
//   warp 1      TMEM allocation + MMA issue (one thread): slice i of X against the
//               stacked slices [T_0 .. T_{7-i}] of Bg -- 12 wide MMAs (N <= 256) per K
//               step land all 36 pairs in the accumulators of their groups;
//               tcgen05.commit frees the stage;
//   warps 2..9  eight independent epilogue warps (no barrier between them): warp (q, h)
//               owns the 32 x 32 patch at TMEM lane quadrant q, column half h -- tcgen05.ld
//               of its 8 group totals, exact int64 merge, fp64 sum, release of tensor
//               memory, transpose through its own shared-memory slab, scatter to the
//               target blocks as fire-and-forget RED.ADD.F64 (one writer per element per
//               launch), row-contiguous.  Segment data live in registers, fetched one
//               item ahead; power-of-two scales are applied on the integer pipe.
// Reference: the Schur update of the elimination, gldl.py:388-409.
#include <cuda.h>
#include <cstdio>
#include <cstring>
#include <algorithm>
#include <mutex>
#include <vector>

#include "common.cuh"
#include "tcgen05.cuh"

namespace h2l {

namespace oz {
using namespace tc;

constexpr int SLICES = 8;
constexpr int BM = 128, BN = 64, BKB = 32;           // tile rows, tile cols, K bytes per stage
constexpr int A_SLICE = BM * BKB, B_SLICE = BN * BKB;  // 4 KB, 2 KB
constexpr int STAGE = SLICES * (A_SLICE + B_SLICE);    // 48 KB
constexpr int NSTAGE = 3;
constexpr int EPI_WARPS = 8;
constexpr int THREADS = 64 + 32 * EPI_WARPS;           // 320
constexpr int PATCH_LD = 33;                           // staged 32 x 32 patch row stride (doubles)
constexpr int CT_BYTES = EPI_WARPS * 32 * PATCH_LD * 8;  // one patch per epilogue warp
constexpr int SMEM = NSTAGE * STAGE + CT_BYTES + 1024 /*align*/ + 256 /*barriers*/;

// K-major operand tile with 32-byte swizzle: rows of 32 bytes (one K step), 8-row
// groups 256 B apart
__device__ __forceinline__ uint64_t sdesc(uint32_t saddr) {
    uint64_t d = 0;
    d |= (uint64_t)((saddr >> 4) & 0x3FFF);          // start address
    d |= (uint64_t)1 << 16;                          // leading byte offset (unused: swizzled K-major)
    d |= (uint64_t)(8 * BKB >> 4) << 32;             // stride byte offset: next 8-row group
    d |= (uint64_t)1 << 46;                          // descriptor version (sm_100)
    d |= (uint64_t)6 << 61;                          // SWIZZLE_32B
    return d;
}
// instruction descriptor: kind::i8, s32 accumulate, signed A/B, both K-major, M=128, N=n
__host__ __device__ constexpr uint32_t idesc_n(int n) {
    return (2u << 4) | (1u << 7) | (1u << 10) | ((uint32_t)(n >> 3) << 17) | ((uint32_t)(BM >> 4) << 24);
}

}  // namespace oz

int schur_oz_tiles(int R) {
    if (R <= 0) return 0;
    const int NI = (R + oz::BM - 1) / oz::BM, NJ = (R + oz::BN - 1) / oz::BN;
    int n = 0;
    for (int I = 0; I < NI; ++I) n += NJ - 2 * I > 0 ? NJ - 2 * I : 0;
    return n;
}

// --------------------------------------------------------------------- slicing
// rows of X (which = 0) / Bg (which = 1) of every job -> 8 int8 slices + row exponent.
// One warp per row; grid (row blocks of 8 rows over the packed rows, shifts, 2).
__global__ void __launch_bounds__(256) oz_split_kernel(const OzJob *jobs, const int *row_job,
                                                       int rows_total, int kpad, int8_t *sx_out,
                                                       int8_t *sb_out, int *ex_out, int *eb_out) {
    const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
    const int row = blockIdx.x * 8 + warp;
    if (row >= rows_total) return;
    const int z = blockIdx.y, which = blockIdx.z;
    const OzJob jb = jobs[row_job[row / oz::BM]];
    const int r = row - jb.row0;
    // slice plane layout [K block of 32 bytes][row][32]: the 128 (64) rows of one K block
    // of a tile are one contiguous 4 KB (2 KB) run, so the TMA fetches whole 128-byte lines
    // instead of one 32-byte sector per row
    const size_t plane = (size_t)rows_total * kpad;
    int8_t *out = (which ? sb_out : sx_out) + (size_t)z * oz::SLICES * plane + (size_t)row * oz::BKB;
    const size_t kbs = (size_t)rows_total * oz::BKB;   // bytes between K blocks
    int *eo = (which ? eb_out : ex_out) + (size_t)z * rows_total + row;
    if (r >= jb.R) {
        for (int p = 0; p < oz::SLICES; ++p)
            for (int k = lane * 4; k < kpad; k += 128)
                *(int *)(out + p * plane + (k / oz::BKB) * kbs + (k % oz::BKB)) = 0;
        if (lane == 0) *eo = 0;
        return;
    }
    const double *src = (which ? jb.Bg : jb.X) + z * jb.sx + (int64_t)r * jb.ld;
    double mx = 0.0;
    for (int k = lane; k < jb.K; k += 32) mx = fmax(mx, fabs(src[k]));
#pragma unroll
    for (int o = 16; o; o >>= 1) mx = fmax(mx, __shfl_xor_sync(0xffffffffu, mx, o));
    // e: 2^(e-1) <= max < 2^e, so |x| 2^-e < 1 and each slice digit |s| <= 127
    const int e = mx > 0.0 ? ilogb(mx) + 1 : 0;
    if (lane == 0) *eo = e;
    for (int k0 = lane * 4; k0 < kpad; k0 += 128) {
        double v[4];
#pragma unroll
        for (int q = 0; q < 4; ++q) v[q] = k0 + q < jb.K ? scalbn(src[k0 + q], -e) : 0.0;
#pragma unroll
        for (int p = 0; p < oz::SLICES; ++p) {
            uint32_t packed = 0;
#pragma unroll
            for (int q = 0; q < 4; ++q) {
                const double t = v[q] * 128.0;       // exact (power of two)
                const double d = trunc(t);           // |d| <= 127
                v[q] = t - d;                        // exact: the remaining bits
                packed |= ((uint32_t)(uint8_t)(int8_t)(int)d) << (8 * q);
            }
            *(uint32_t *)(out + p * plane + (k0 / oz::BKB) * kbs + (k0 % oz::BKB)) = packed;
        }
    }
}

// ------------------------------------------------------------------ the GEMM
// exact int32 -> fp64 without the XU pipe: the bits of 2^52 + 2^51 + v, minus 2^52 + 2^51
__device__ __forceinline__ double i2d_exact(int v) {
    return __hiloint2double(0x43380000 + (v >> 31), v) - 6755399441055744.0;
}
// exact int64 -> fp64 for |v| < 2^51, same trick in 64 bits
__device__ __forceinline__ double i2d_exact64(long long v) {
    return __longlong_as_double(0x4338000000000000LL + v) - 6755399441055744.0;
}
// -v 2^e on the integer pipe (v normal or zero; a result below the normal range is flushed
// to zero: it is < 2^-1022 against targets of order one)
__device__ __forceinline__ double neg_scale_pow2(double v, int e) {
    const int hi = __double2hiint(v), lo = __double2loint(v);
    const int ex = (hi >> 20) & 0x7ff;
    const bool zero = ex == 0 || ex + e <= 0;
    return __hiloint2double(zero ? 0 : (hi + (e << 20)) ^ 0x80000000, zero ? 0 : lo);
}
// 2^e (exact; fast path for the normal range)
__device__ __forceinline__ double pow2i(int e) {
    return (e >= -1022 && e <= 1023) ? __longlong_as_double((long long)(e + 1023) << 52)
                                     : scalbn(1.0, e);
}

// probe 8 (diagnostic): cycles per phase, summed over CTAs.  0 items, 1 epilogue: segment
// tables, 2 epilogue: wait for the MMAs, 3 TMEM read + group sum, 4 tile staging,
// 5 scatter, 8 issuer: wait for the epilogue, 9 issuer: wait for TMA, 10 issuer: issue
__device__ unsigned long long g_oz_prof[16];

// Persistent: one CTA per SM walks the (shift, tile) items; the TMA producer and the
// MMA issuer run ahead across items, the epilogue of item i overlaps the MMAs of
// item i + 1 (it releases tensor memory right after reading the 8 group totals).
__global__ void __launch_bounds__(oz::THREADS, 1)
    schur_oz_kernel(const __grid_constant__ CUtensorMap map_x,
                    const __grid_constant__ CUtensorMap map_b, const OzJob *jobs,
                    const int2 *tile_ij, int total_tiles, int nshift, int rows_total,
                    const int *ex_all, const int *eb_all, int probe) {
    using namespace oz;
    extern __shared__ __align__(1024) unsigned char smem_raw[];
    // aligned by an offset (not a cast) so the compiler keeps the shared address space
    unsigned char *smem = smem_raw + ((1024u - (su32(smem_raw) & 1023u)) & 1023u);
    double *ct = (double *)(smem + NSTAGE * STAGE);           // staged output tile
    uint64_t *full = (uint64_t *)(smem + NSTAGE * STAGE + CT_BYTES);
    uint64_t *empty = full + NSTAGE;
    uint64_t *tfull = empty + NSTAGE;
    uint64_t *tempty = tfull + 1;
    uint32_t *tmem_slot = (uint32_t *)(tempty + 1);

    const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
    const int items = total_tiles * nshift;
    const bool prof = probe == 8;

    if (warp == 0 && lane == 0) {
        for (int s = 0; s < NSTAGE; ++s) {
            mbar_init(&full[s], 1);
            mbar_init(&empty[s], 1);
        }
        mbar_init(tfull, 1);
        mbar_init(tempty, EPI_WARPS);
        asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
        asm volatile("prefetch.tensormap [%0];" ::"l"(&map_x) : "memory");
        asm volatile("prefetch.tensormap [%0];" ::"l"(&map_b) : "memory");
    }
    if (warp == 1) {
        asm volatile("tcgen05.alloc.cta_group::1.sync.aligned.shared::cta.b32 [%0], 512;" ::"r"(
                         su32(tmem_slot))
                     : "memory");
        asm volatile("tcgen05.relinquish_alloc_permit.cta_group::1.sync.aligned;" ::: "memory");
    }
    tc_fence_before();
    __syncthreads();
    tc_fence_after();
    const uint32_t tmem = *tmem_slot;

    auto locate = [&](int item, OzJob &jb, int &z, int &m0, int &n0) {
        z = item / total_tiles;
        const int2 tj = tile_ij[item - z * total_tiles];
        jb = jobs[tj.x];
        m0 = (tj.y >> 16) * BM;
        n0 = (tj.y & 0xFFFF) * BN;
    };

    if (warp == 0) {
        if (lane == 0) {
            int kstep = 0;
            for (int item = blockIdx.x; item < items; item += gridDim.x) {
                OzJob jb;
                int z, m0, n0;
                locate(item, jb, z, m0, n0);
                const int nkb = (jb.K + BKB - 1) / BKB;
                for (int kb = 0; kb < nkb; ++kb, ++kstep) {
                    const int s = kstep % NSTAGE;
                    mbar_wait(&empty[s], ((kstep / NSTAGE) & 1) ^ 1);
                    mbar_expect_tx(&full[s], STAGE);
                    unsigned char *a = smem + s * STAGE, *b = a + SLICES * A_SLICE;
                    for (int p = 0; p < SLICES; ++p) {
                        tma_load_4d(a + p * A_SLICE, &map_x, &full[s], 0, jb.row0 + m0, kb,
                                    z * SLICES + p);
                        tma_load_4d(b + p * B_SLICE, &map_b, &full[s], 0, jb.row0 + n0, kb,
                                    z * SLICES + p);
                    }
                }
            }
        }
    } else if (warp == 1) {
        if (lane == 0) {
            int kstep = 0, it = 0;
            long long pm[3] = {0, 0, 0};
            for (int item = blockIdx.x; item < items; item += gridDim.x, ++it) {
                OzJob jb;
                int z, m0, n0;
                locate(item, jb, z, m0, n0);
                const int nkb = (jb.K + BKB - 1) / BKB;
                long long c0 = prof ? clock64() : 0;
                mbar_wait(tempty, (it & 1) ^ 1);     // the epilogue has read the previous totals
                tc_fence_after();
                if (prof) { const long long c1 = clock64(); pm[0] += c1 - c0; c0 = c1; }
                for (int kb = 0; kb < nkb; ++kb, ++kstep) {
                    const int s = kstep % NSTAGE;
                    // probe (benchmarking only): 1 = MMAs without waiting for the loads,
                    // 2 = loads without MMAs
                    if (probe != 1) mbar_wait(&full[s], (kstep / NSTAGE) & 1);
                    tc_fence_after();
                    if (prof) { const long long c1 = clock64(); pm[1] += c1 - c0; c0 = c1; }
                    if (probe == 2) {
                        asm volatile("mbarrier.arrive.shared::cta.b64 _, [%0];" ::"r"(su32(&empty[s])) : "memory");
                        continue;
                    }
                    const uint32_t a = su32(smem + s * STAGE), b = a + SLICES * A_SLICE;
                    // slice i of X against the stacked slices [T_0; T_1; ...; T_{7-i}] of
                    // Bg (contiguous in shared memory): one wide MMA lands every pair
                    // (i, j) in the accumulator of its group g = i + j (columns g * 64).
                    // An MMA costs the same for any N <= 256, so 12 wide instructions
                    // per K step replace 36 of N = 64.
#pragma unroll
                    for (int i = 0; i < SLICES; ++i) {
                        const int cols = (SLICES - i) * BN;
#pragma unroll
                        for (int off = 0; off < cols; off += 256) {
                            const int n = cols - off < 256 ? cols - off : 256;
                            mma_i8(tmem + i * BN + off, sdesc(a + i * A_SLICE),
                                   sdesc(b + (off / BN) * B_SLICE), idesc_n(n), (kb | i) != 0);
                        }
                    }
                    tc_commit(&empty[s]);
                    if (prof) { const long long c1 = clock64(); pm[2] += c1 - c0; c0 = c1; }
                }
                tc_commit(tfull);
            }
            if (prof) {
                atomicAdd(&g_oz_prof[8], (unsigned long long)pm[0]);
                atomicAdd(&g_oz_prof[9], (unsigned long long)pm[1]);
                atomicAdd(&g_oz_prof[10], (unsigned long long)pm[2]);
                atomicAdd(&g_oz_prof[0], (unsigned long long)it);
            }
        }
    } else {
        // ---------------------------------------------------------- epilogue
        // Eight independent warps, no barrier between them: warp (q, h) owns the 32 x 32
        // patch of the tile at rows 32 q (its TMEM lane quadrant), columns 32 h.  Per item:
        // the 8 group totals of its patch are read from tensor memory and summed (C), the
        // patch is transposed through the warp's own shared-memory slab (D: row = TMEM
        // lane -> row-contiguous lanes) and scattered to the target blocks as
        // fire-and-forget L2 reductions, one writer per element per launch (E).  The
        // segment data of the warp's rows / columns live in registers (lane = row, and
        // lane = column) and are fetched one item ahead; since the warps drift apart,
        // one warp's reductions drain while another converts.
        // (tools/micro/scatter_bench.cu: reductions, load/add/store and TMA bulk reduce all
        // run at the same HBM-bound rate for this traffic; only the reductions need no
        // loads in flight.)
        const int q = warp & 3, h = (warp - 2) >> 2;       // TMEM lane quadrant, column half
        const int ew = warp - 2;
        double *patch = ct + ew * (32 * PATCH_LD);
        int it = 0;
        long long pe[5] = {0, 0, 0, 0, 0}, c0 = prof ? clock64() : 0;
        auto tick = [&](int k) {
            if (prof) { const long long c1 = clock64(); pe[k] += c1 - c0; c0 = c1; }
        };
        struct Seg {              // lane = row (r*) and lane = column (c*) of the patch
            int rseg, roff, cseg, coff;
            int er, ec;           // row / column scale exponents
            SchurTarget e0;       // target of (first row segment, this lane's column segment)
        };
        auto fetch = [&](int item, Seg &sg) {
            OzJob jb;
            int z, m0, n0;
            locate(item, jb, z, m0, n0);
            const int gr = m0 + 32 * q + lane, gc = n0 + 32 * h + lane;
            sg.rseg = gr < jb.R ? __ldg(jb.seg_of + gr) : -1;
            sg.cseg = gc < jb.R ? __ldg(jb.seg_of + gc) : -1;
            sg.roff = sg.rseg >= 0 ? gr - __ldg(jb.seg_start + sg.rseg) : 0;
            sg.coff = sg.cseg >= 0 ? gc - __ldg(jb.seg_start + sg.cseg) : 0;
            sg.er = __ldg(ex_all + (size_t)z * rows_total + jb.row0 + gr);
            sg.ec = __ldg(eb_all + (size_t)z * rows_total + jb.row0 + gc);
            const int a0 = __shfl_sync(0xffffffffu, sg.rseg, 0);
            sg.e0 = SchurTarget{nullptr, 0, 0, 0};
            if (a0 >= 0 && sg.cseg >= 0) sg.e0 = jb.tbl[(size_t)a0 * jb.nseg + sg.cseg];
        };
        Seg cur, nxt;
        if ((int)blockIdx.x < items) fetch(blockIdx.x, cur);
        for (int item = blockIdx.x; item < items; item += gridDim.x, ++it) {
            OzJob jb;
            int z, m0, n0;
            locate(item, jb, z, m0, n0);
            // the next item's segment data: the loads fly during this item's work
            if (item + (int)gridDim.x < items) fetch(item + gridDim.x, nxt);
            tick(0);
            // ---- (C) group totals
            mbar_wait(tfull, it & 1);
            tc_fence_after();
            tick(1);
            // the 8 group totals are merged exactly in 64-bit integers three at a time
            // (|total| < 2^31, so v0 2^14 + v1 2^7 + v2 < 2^46) before the fp64 sum: 3
            // conversions and 3 fp64 terms per element instead of 8
            double acc[32];
#pragma unroll
            for (int half = 0; half < 2; ++half) {
                const uint32_t tcol = tmem + ((uint32_t)(q * 32) << 16) + h * 32 + half * 16;
                uint32_t va[16], vb[16], vc[16];
                tmem_ld16_nowait(tcol + 6 * BN, va);
                tmem_ld16_nowait(tcol + 7 * BN, vb);
                tmem_ld_wait();
#pragma unroll
                for (int c = 0; c < 16; ++c)
                    acc[half * 16 + c] =
                        i2d_exact64(((long long)(int)va[c] << 7) + (int)vb[c]) * 0x1p-63;
                tmem_ld16_nowait(tcol + 3 * BN, va);
                tmem_ld16_nowait(tcol + 4 * BN, vb);
                tmem_ld16_nowait(tcol + 5 * BN, vc);
                tmem_ld_wait();
#pragma unroll
                for (int c = 0; c < 16; ++c)
                    acc[half * 16 + c] = fma(i2d_exact64(((long long)(int)va[c] << 14) +
                                                         ((long long)(int)vb[c] << 7) + (int)vc[c]),
                                             0x1p-49, acc[half * 16 + c]);
                tmem_ld16_nowait(tcol + 0 * BN, va);
                tmem_ld16_nowait(tcol + 1 * BN, vb);
                tmem_ld16_nowait(tcol + 2 * BN, vc);
                tmem_ld_wait();
#pragma unroll
                for (int c = 0; c < 16; ++c)
                    acc[half * 16 + c] = fma(i2d_exact64(((long long)(int)va[c] << 14) +
                                                         ((long long)(int)vb[c] << 7) + (int)vc[c]),
                                             0x1p-28, acc[half * 16 + c]);
            }
            tc_fence_before();
            __syncwarp();
            if (lane == 0) asm volatile("mbarrier.arrive.shared::cta.b64 _, [%0];" ::"r"(su32(tempty)) : "memory");
            tick(2);
            // ---- (D) transpose through the warp's slab
            {
                double *row = patch + lane * PATCH_LD;
#pragma unroll
                for (int c = 0; c < 32; ++c) row[c] = acc[c];
            }
            __syncwarp();
            tick(3);
            // ---- (E) row j of the patch -> one row-contiguous reduction per lane
            if (probe != 4) {
                const bool live = cur.cseg >= 0;
                const int gc = n0 + 32 * h + lane, cb = cur.coff, b = cur.cseg;
                int a_cur = __shfl_sync(0xffffffffu, cur.rseg, 0);
                SchurTarget e = cur.e0;
#pragma unroll 4
                for (int j = 0; j < 32; ++j) {
                    const int a = __shfl_sync(0xffffffffu, cur.rseg, j);
                    const int ra = __shfl_sync(0xffffffffu, cur.roff, j);
                    const int er = __shfl_sync(0xffffffffu, cur.er, j);
                    if (a < 0) break;
                    if (a != a_cur) {
                        a_cur = a;
                        if (live) e = jb.tbl[(size_t)a * jb.nseg + b];
                    }
                    if (!live || !e.base || gc < m0 + 32 * q + j) continue;
                    const double val = neg_scale_pow2(patch[j * PATCH_LD + lane], er + cur.ec);
                    double *tb = e.base + z * e.bs;
                    const int64_t tld = e.ldc;
                    red_add_f64(tb + (e.trans ? (int64_t)cb * tld + ra : (int64_t)ra * tld + cb), val);
                    if (a == b && cb != ra && probe != 3) red_add_f64(tb + (int64_t)cb * tld + ra, val);
                }
            }
            __syncwarp();
            cur = nxt;
            tick(4);
        }
        if (prof && ew == 0 && lane == 0)
            for (int k = 0; k < 5; ++k) atomicAdd(&g_oz_prof[1 + k], (unsigned long long)pe[k]);
    }
    tc_fence_before();
    __syncthreads();
    if (warp == 1) {
        tc_fence_after();
        asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, 512;" ::"r"(tmem) : "memory");
    }
}

// ------------------------------------------------------------------- host side
namespace {
typedef CUresult (*EncodeTiled)(CUtensorMap *, CUtensorMapDataType, cuuint32_t, void *,
                                const cuuint64_t *, const cuuint64_t *, const cuuint32_t *,
                                const cuuint32_t *, CUtensorMapInterleave, CUtensorMapSwizzle,
                                CUtensorMapL2promotion, CUtensorMapFloatOOBfill);
EncodeTiled encode_fn() {
    static EncodeTiled fn = nullptr;
    static std::once_flag once;
    std::call_once(once, [] {
        void *p = nullptr;
        cudaDriverEntryPointQueryResult q;
        if (cudaGetDriverEntryPoint("cuTensorMapEncodeTiled", &p, cudaEnableDefault, &q) ==
                cudaSuccess &&
            q == cudaDriverEntryPointSuccess)
            fn = (EncodeTiled)p;
    });
    return fn;
}
cudaError_t make_map(CUtensorMap *m, const int8_t *base, int kpad, int rows, int planes,
                     int box_rows) {
    EncodeTiled fn = encode_fn();
    if (!fn) return cudaErrorNotSupported;
    // [plane][K block][row][32 bytes]
    cuuint64_t dims[4] = {(cuuint64_t)oz::BKB, (cuuint64_t)rows, (cuuint64_t)(kpad / oz::BKB),
                          (cuuint64_t)planes};
    cuuint64_t strides[3] = {(cuuint64_t)oz::BKB, (cuuint64_t)oz::BKB * rows, (cuuint64_t)kpad * rows};
    cuuint32_t box[4] = {(cuuint32_t)oz::BKB, (cuuint32_t)box_rows, 1, 1};
    cuuint32_t es[4] = {1, 1, 1, 1};
    CUresult r = fn(m, CU_TENSOR_MAP_DATA_TYPE_UINT8, 4, (void *)base, dims, strides, box, es,
                    CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_32B,
                    CU_TENSOR_MAP_L2_PROMOTION_L2_256B, CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
    return r == CUDA_SUCCESS ? cudaSuccess : cudaErrorInvalidValue;
}
}  // namespace

void oz_prof_fetch(unsigned long long *out, bool reset) {
    cudaMemcpyFromSymbol(out, g_oz_prof, sizeof(g_oz_prof));
    if (reset) {
        unsigned long long z[16] = {};
        cudaMemcpyToSymbol(g_oz_prof, z, sizeof(z));
    }
}

size_t schur_oz_scratch_bytes(int rows_total, int kpad, int nshift) {
    const size_t sl = (size_t)oz::SLICES * rows_total * kpad * nshift;
    const size_t ex = (size_t)rows_total * nshift * sizeof(int);
    return 2 * sl + 2 * ((ex + 255) / 256 * 256);
}

// Grid tiles of one job in the launch order: column blocks of OZ_JB column tiles
// (64 rows of Bg each); within a block, row tiles ascending, then the block's column
// tiles.  Concurrent CTAs then share one block of Bg slices (L2-resident) and stream
// the X slices once per block, instead of re-reading every Bg tile once per row tile
// (the panels reach 60k rows: their slices are GBs, far above L2).
constexpr int OZ_JB = 64;
void schur_oz_tile_order(int R, int job, std::vector<int2> &out) {
    const int NJ = (R + oz::BN - 1) / oz::BN;
    for (int j0 = 0; j0 < NJ; j0 += OZ_JB) {
        const int j1 = std::min(NJ, j0 + OZ_JB);
        for (int I = 0; 2 * I < j1; ++I)
            for (int J = std::max(j0, 2 * I); J < j1; ++J) out.push_back(make_int2(job, (I << 16) | J));
    }
}

// jobs / row_job / tile_ij are device arrays (row_job: one entry per 128 packed rows,
// tile_ij: (job, I << 16 | J) per grid tile in launch order, schur_oz_tile_order);
// scratch holds schur_oz_scratch_bytes(rows_total, kpad, nshift) bytes.
cudaError_t launch_schur_oz(const OzJob *jobs, const int *row_job, const int2 *tile_ij,
                            int rows_total, int kpad, int total_tiles, int nshift, void *scratch,
                            cudaStream_t st, int probe) {
    if (total_tiles <= 0 || nshift <= 0 || rows_total <= 0) return cudaSuccess;
    if (kpad % 64 || rows_total % oz::BM) return cudaErrorInvalidValue;
    const size_t sl = (size_t)oz::SLICES * rows_total * kpad * nshift;
    const size_t ex = ((size_t)rows_total * nshift * sizeof(int) + 255) / 256 * 256;
    int8_t *sx = (int8_t *)scratch, *sb = sx + sl;
    int *exr = (int *)(sb + sl), *ebr = (int *)((char *)exr + ex);
    dim3 g1((rows_total + 7) / 8, nshift, 2);
    oz_split_kernel<<<g1, 256, 0, st>>>(jobs, row_job, rows_total, kpad, sx, sb, exr, ebr);
    CUtensorMap mx, mb;
    cudaError_t e = make_map(&mx, sx, kpad, rows_total, oz::SLICES * nshift, oz::BM);
    if (e != cudaSuccess) return e;
    e = make_map(&mb, sb, kpad, rows_total, oz::SLICES * nshift, oz::BN);
    if (e != cudaSuccess) return e;
    static std::once_flag once;
    std::call_once(once, [] {
        cudaFuncSetAttribute(schur_oz_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, oz::SMEM);
    });
    static int nsm = 0;
    if (!nsm) {
        int dev = 0;
        cudaGetDevice(&dev);
        cudaDeviceGetAttribute(&nsm, cudaDevAttrMultiProcessorCount, dev);
    }
    static const int env_probe = getenv("H2L_OZ_PROBE") ? atoi(getenv("H2L_OZ_PROBE")) : 0;
    if (!probe) probe = env_probe;
    const int items = total_tiles * nshift;
    schur_oz_kernel<<<items < nsm ? items : nsm, oz::THREADS, oz::SMEM, st>>>(
        mx, mb, jobs, tile_ij, total_tiles, nshift, rows_total, exr, ebr, probe);
    return cudaGetLastError();
}

}  // namespace h2l
