// Microbenchmark: ways to add a 128 x 64 fp64 tile (rows `ld` doubles apart) into a large
// HBM-resident matrix, one persistent CTA per SM -- the epilogue traffic of the Schur
// update (k_schur_oz.cu).  Variants: 0 scalar RED.ADD.F64, 1 scalar load / add / store
// (all loads first), 2 cp.reduce.async.bulk .add.f64 per row, 3 cp.async.bulk row loads
// + add + cp.async.bulk row stores.   nvcc -O3 -arch=sm_100a scatter_bench.cu -o scatter_bench
#include <cstdio>
#include <cstdint>
#include <cstdlib>
#include <cuda_runtime.h>

constexpr int BM = 128, BN = 64, LDS_ = 66;
__device__ __forceinline__ uint32_t su32(const void *p) { return (uint32_t)__cvta_generic_to_shared(p); }

__global__ void __launch_bounds__(256, 1) scatter(double *C, int64_t ld, int64_t rows, int tiles, int variant,
                                                  const int2 *pos) {
    extern __shared__ __align__(128) double ct[];   // BM x LDS_
    __shared__ uint64_t bar;
    const int t = threadIdx.x, warp = t >> 5, lane = t & 31;
    for (int i = t; i < BM * LDS_; i += 256) ct[i] = 1.0;
    if (t == 0) {
        asm volatile("mbarrier.init.shared::cta.b64 [%0], 1;" ::"r"(su32(&bar)));
        asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
    }
    __syncthreads();
    int phase = 0;
    for (int tile = blockIdx.x; tile < tiles; tile += gridDim.x) {
        const int2 p = pos[tile];
        double *base = C + (int64_t)p.x * ld + p.y;
        if (variant == 4) {   // the epilogue's pattern: warp (q, h) owns rows 32 q.., columns 32 h..
            const int q = warp & 3, h = warp >> 2;
#pragma unroll 4
            for (int j = 0; j < 32; ++j)
                asm volatile("red.global.add.f64 [%0], %1;" ::"l"(base + (int64_t)(32 * q + j) * ld + h * 32 + lane),
                             "d"(ct[(32 * q + j) * LDS_ + h * 32 + lane]) : "memory");
        } else if (variant == 0) {
            for (int r = warp; r < BM; r += 8)
                for (int h = 0; h < 2; ++h)
                    asm volatile("red.global.add.f64 [%0], %1;" ::"l"(base + (int64_t)r * ld + h * 32 + lane),
                                 "d"(ct[r * LDS_ + h * 32 + lane]) : "memory");
        } else if (variant == 1) {
            double old[16][2];
#pragma unroll
            for (int rr = 0; rr < 16; ++rr)
#pragma unroll
                for (int h = 0; h < 2; ++h) old[rr][h] = __ldcs(base + (int64_t)(warp + 8 * rr) * ld + h * 32 + lane);
#pragma unroll
            for (int rr = 0; rr < 16; ++rr)
#pragma unroll
                for (int h = 0; h < 2; ++h)
                    __stcs(base + (int64_t)(warp + 8 * rr) * ld + h * 32 + lane,
                           old[rr][h] + ct[(warp + 8 * rr) * LDS_ + h * 32 + lane]);
        } else if (variant == 2) {
            asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
            __syncthreads();
            if (t < BM) {
                asm volatile("cp.reduce.async.bulk.global.shared::cta.bulk_group.add.f64 [%0], [%1], %2;" ::"l"(
                                 base + (int64_t)t * ld), "r"(su32(ct + t * LDS_)), "r"(BN * 8) : "memory");
                asm volatile("cp.async.bulk.commit_group;" ::: "memory");
                asm volatile("cp.async.bulk.wait_group.read 0;" ::: "memory");
            }
            __syncthreads();
        } else {
            if (t == 0)
                asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(su32(&bar)), "r"(BM * BN * 8) : "memory");
            __syncthreads();
            if (t < BM)
                asm volatile("cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];" ::"r"(
                                 su32(ct + t * LDS_)), "l"(base + (int64_t)t * ld), "r"(BN * 8), "r"(su32(&bar)) : "memory");
            asm volatile("{\n\t.reg .pred P1;\nW_%=:\n\tmbarrier.try_wait.parity.shared::cta.b64 P1, [%0], %1;\n\t@P1 bra D_%=;\n\tbra W_%=;\nD_%=:\n\t}" ::"r"(su32(&bar)), "r"(phase) : "memory");
            phase ^= 1;
            for (int r = warp; r < BM; r += 8)
                for (int h = 0; h < 2; ++h) ct[r * LDS_ + h * 32 + lane] += 1.0;
            asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
            __syncthreads();
            if (t < BM) {
                asm volatile("cp.async.bulk.global.shared::cta.bulk_group [%0], [%1], %2;" ::"l"(base + (int64_t)t * ld),
                             "r"(su32(ct + t * LDS_)), "r"(BN * 8) : "memory");
                asm volatile("cp.async.bulk.commit_group;" ::: "memory");
                asm volatile("cp.async.bulk.wait_group.read 0;" ::: "memory");
            }
            __syncthreads();
        }
    }
}

int main(int argc, char **argv) {
    const int64_t ld = argc > 1 ? atoll(argv[1]) : 16384;       // doubles per row
    const int64_t rows = argc > 2 ? atoll(argv[2]) : 65536;     // 8 GB at the defaults
    double *C;
    if (cudaMalloc(&C, sizeof(double) * ld * rows) != cudaSuccess) { printf("alloc failed\n"); return 1; }
    cudaMemset(C, 0, sizeof(double) * ld * rows);
    const int tr = rows / BM, tc = (ld - 1) / BN, tiles = tr * tc > 400000 ? 400000 : tr * tc;
    int2 *hp = (int2 *)malloc(sizeof(int2) * tiles), *dp;
    // disjoint tiles in a pseudo-random order (stride permutation)
    const int64_t total = (int64_t)tr * tc;
    for (int i = 0; i < tiles; ++i) {
        const int64_t k = ((int64_t)i * 7919) % total;
        hp[i] = make_int2((int)(k / tc) * BM, (int)(k % tc) * BN + (int)(ld & 1));
    }
    cudaMalloc(&dp, sizeof(int2) * tiles);
    cudaMemcpy(dp, hp, sizeof(int2) * tiles, cudaMemcpyHostToDevice);
    int nsm = 0;
    cudaDeviceGetAttribute(&nsm, cudaDevAttrMultiProcessorCount, 0);
    const int smem = BM * LDS_ * 8;
    cudaFuncSetAttribute(scatter, cudaFuncAttributeMaxDynamicSharedMemorySize, smem);
    for (int v = 0; v < 5; ++v) {
        if ((ld & 1) && (v == 2 || v == 3)) continue;   // bulk copies need 16-byte rows
        cudaEvent_t e0, e1;
        cudaEventCreate(&e0); cudaEventCreate(&e1);
        scatter<<<nsm, 256, smem>>>(C, ld, rows, tiles / 8, v, dp);
        cudaEventRecord(e0);
        scatter<<<nsm, 256, smem>>>(C, ld, rows, tiles, v, dp);
        cudaEventRecord(e1);
        cudaError_t e = cudaDeviceSynchronize();
        float ms = 0;
        cudaEventElapsedTime(&ms, e0, e1);
        const double bytes = (double)tiles * BM * BN * 8;
        printf("variant %d: %s  %.3f ms  payload %.1f GB/s (x2 DRAM r+w)  %.0f cycles/tile/SM @1.9GHz\n", v,
               cudaGetErrorString(e), ms, bytes / ms / 1e6, ms * 1e-3 * 1.9e9 / (tiles / (double)nsm));
    }
    // check: every touched element got 2 adds per variant... (variants 0-3 x (1/8 + 1) passes)
    double h[4];
    cudaMemcpy(h, C + (int64_t)hp[0].x * ld + hp[0].y, sizeof(h), cudaMemcpyDeviceToHost);
    printf("check C[tile0][0..3] = %g %g %g %g (expect 8)\n", h[0], h[1], h[2], h[3]);
    return 0;
}
