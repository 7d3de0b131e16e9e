// cost of cg::this_cluster().sync() and of __syncthreads (one cluster per GPC-ish slot)
#include <cstdio>
#include <cooperative_groups.h>
namespace cg = cooperative_groups;
__global__ void k_cluster(int iters, int *out) {
    cg::cluster_group cl = cg::this_cluster();
    for (int i = 0; i < iters; ++i) cl.sync();
    if (threadIdx.x == 0 && blockIdx.x == 0) out[0] = iters;
}
__global__ void k_block(int iters, int *out) {
    for (int i = 0; i < iters; ++i) __syncthreads();
    if (threadIdx.x == 0 && blockIdx.x == 0) out[0] = iters;
}
__global__ void k_dsmem(int iters, int *out) {
    cg::cluster_group cl = cg::this_cluster();
    __shared__ double v[32];
    if (threadIdx.x < 32) v[threadIdx.x] = threadIdx.x;
    cl.sync();
    double acc = 0;
    const int r = (cl.block_rank() + 1) % cl.num_blocks();
    for (int i = 0; i < iters; ++i) {
        acc += *cl.map_shared_rank(&v[(i + threadIdx.x) & 31], r);
    }
    cl.sync();
    if (acc == -1.0) out[1] = 1;
}
template <class K>
float run(K kern, int cs, int threads, int iters) {
    int *out; cudaMalloc(&out, 16);
    cudaLaunchConfig_t cfg = {};
    cfg.gridDim = dim3(cs, 1, 1); cfg.blockDim = dim3(threads, 1, 1);
    cudaLaunchAttribute at[1];
    at[0].id = cudaLaunchAttributeClusterDimension;
    at[0].val.clusterDim.x = cs; at[0].val.clusterDim.y = 1; at[0].val.clusterDim.z = 1;
    cfg.attrs = at; cfg.numAttrs = 1;
    cudaLaunchKernelEx(&cfg, kern, 10, out);
    cudaDeviceSynchronize();
    cudaEvent_t e0, e1; cudaEventCreate(&e0); cudaEventCreate(&e1);
    cudaEventRecord(e0);
    cudaLaunchKernelEx(&cfg, kern, iters, out);
    cudaEventRecord(e1); cudaEventSynchronize(e1);
    float ms; cudaEventElapsedTime(&ms, e0, e1);
    cudaFree(out);
    return ms * 1e3f / iters;
}
int main() {
    cudaFuncSetAttribute(k_cluster, cudaFuncAttributeNonPortableClusterSizeAllowed, 1);
    for (int cs : {2, 4, 8, 16})
        printf("cluster.sync  cs=%2d 256 thr: %.3f us\n", cs, run(k_cluster, cs, 256, 100000));
    printf("__syncthreads 256 thr: %.3f us\n", run(k_block, 1, 256, 100000));
    printf("__syncthreads 512 thr: %.3f us\n", run(k_block, 1, 512, 100000));
    for (int cs : {2, 8})
        printf("dsmem load latency-bound chain cs=%d: %.3f us per load\n", cs, run(k_dsmem, cs, 32, 100000));
    return 0;
}
