// DMMA GEMM tile variants for tools/gemm_bench.py (benchmarking library only;
// not linked into libh2ldl.so).  The tile prefix must use the variant's tiling.
#include "gemm_tile.cuh"

namespace h2l {
namespace {
// ---- variants for tools/gemm_bench.py (the tile prefix must use the variant's tiling)
using V0 = GemmCfg<64, 64, 32, 32, 3>;
using V1 = GemmCfg<64, 128, 32, 64, 3>;
using V2 = GemmCfg<64, 64, 32, 32, 2, false, 5>;
using V3 = GemmCfg<64, 64, 32, 32, 3, false, 3>;
using V4 = GemmCfg<64, 64, 32, 32, 2, false, 4>;
using V5 = GemmCfg<128, 64, 32, 32, 2, false, 2>;
using V6 = GemmCfg<64, 64, 32, 16, 2, false, 6>;
using V7 = GemmCfg<128, 64, 32, 32, 3, false, 2>;
using V8 = GemmCfg<64, 64, 32, 32, 2, false, 3, 32>;
using V9 = GemmCfg<64, 64, 32, 32, 3, false, 2, 32>;
#define H2L_VARIANTS(X) \
    X(0, V0) X(1, V1) X(2, V2) X(3, V3) X(4, V4) X(5, V5) X(6, V6) X(7, V7) X(8, V8) X(9, V9)
}  // namespace

int gemm_variant_tiles(int v, int M, int N) {
    if (M <= 0 || N <= 0) return 0;
#define X(id, C) \
    if (v == id) return ((M + C::BM - 1) / C::BM) * ((N + C::BN - 1) / C::BN);
    H2L_VARIANTS(X)
#undef X
    return 0;
}

void launch_gemm_variant(int v, const GemmTask *dev_tasks, const int *dev_tile_prefix, int ntasks,
                         int total_tiles, int nshift, cudaStream_t st) {
#define X(id, C) \
    if (v == id) launch_cfg<C>(dev_tasks, dev_tile_prefix, ntasks, total_tiles, nshift, st);
    H2L_VARIANTS(X)
#undef X
}

}  // namespace h2l
