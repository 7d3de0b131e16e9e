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
// Tiling (template GemmCfg): a CTA computes a BM x BN tile of one task for
// one shift; warps are laid out (BM/WM) x (BN/WN), each warp owns a WM x WN
// sub-tile of (WM/8) x (WN/8) DMMA fragments.  K advances in chunks of 16
// through a STAGES-deep cp.async pipeline (global -> shared without register
// staging; out-of-range elements zero-filled by the copy), shared rows padded
// to 20 doubles so fragment reads are conflict-free.  The production tile
// (64x64, 2x2 warps of 32x32, 2 stages, <= 128 registers so 4 CTAs = 16
// warps share an SM) was picked with tools/gemm_bench.py: on the Schur
// shapes of configs 1-2 (K = n_R = 128-192) occupancy beats deeper
// pipelines and larger warp tiles; the epilogue loads C with all loads of a
// fragment row issued before its stores (other resident CTAs hide the
// latency; staging C in shared memory costs occupancy).  Tasks are flattened
// into one grid through a tile prefix array: thousands of small blocks of one
// elimination step go out in a single launch; gridDim.y enumerates shifts.
#include "gemm_tile.cuh"

namespace h2l {

int schur_sym_tiles(int R) {
    const int nt = (R + Prod::BM - 1) / Prod::BM;
    return nt * (nt + 1) / 2;
}

void launch_schur_sym(const double *X, const double *Bg, int64_t sx, int ld, int R, int K,
                      const int *seg_of, const int *seg_start, int nseg, const SchurTarget *tbl,
                      int nshift, cudaStream_t st, int) {
    const int tiles = schur_sym_tiles(R);
    if (tiles <= 0 || nshift <= 0 || K <= 0) return;
    smem_optin(schur_sym_kernel<Prod, 2>);
    dim3 grid(tiles, nshift);
    schur_sym_kernel<Prod, 2><<<grid, Prod::THREADS, Prod::SMEM, st>>>(X, Bg, sx, ld, R, K, seg_of,
                                                                       seg_start, nseg, tbl);
}

void launch_schur_sym_multi(const SchurJob *jobs, const int *tile_job, int total_tiles,
                            int nshift, cudaStream_t st) {
    if (total_tiles <= 0 || nshift <= 0) return;
    smem_optin(schur_sym_multi_kernel<Prod>);
    dim3 grid(total_tiles, nshift);
    schur_sym_multi_kernel<Prod><<<grid, Prod::THREADS, Prod::SMEM, st>>>(jobs, tile_job);
}

int gemm_tiles(int M, int N) {
    if (M <= 0 || N <= 0) return 0;
    return ((M + Prod::BM - 1) / Prod::BM) * ((N + Prod::BN - 1) / Prod::BN);
}

void launch_gemm(const GemmTask *dev_tasks, const int *dev_tile_prefix, int ntasks,
                 int total_tiles, int nshift, cudaStream_t st, bool schur,
                 const int *dev_tile_task) {
    if (ntasks <= 0 || total_tiles <= 0 || nshift <= 0) return;
    dim3 grid(total_tiles, nshift);
    if (schur) {
        smem_optin(schur_gemm_kernel<Prod>);
        schur_gemm_kernel<Prod><<<grid, Prod::THREADS, Prod::SMEM, st>>>(
            dev_tasks, dev_tile_prefix, ntasks, dev_tile_task);
        return;
    }
    smem_optin(gemm_kernel<Prod>);
    gemm_kernel<Prod><<<grid, Prod::THREADS, Prod::SMEM, st>>>(dev_tasks, dev_tile_prefix, ntasks,
                                                               dev_tile_task);
}

}  // namespace h2l
