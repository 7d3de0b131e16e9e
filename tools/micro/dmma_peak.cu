// DMMA.8x8x4 pipe peak vs warps per SM (register operands only).
#include <cstdio>
#include <cuda_runtime.h>
__device__ __forceinline__ void dmma(double &c0, double &c1, double a, double b) {
    asm volatile("mma.sync.aligned.m8n8k4.row.col.f64.f64.f64.f64 {%0,%1}, {%2}, {%3}, {%0,%1};\n"
                 : "+d"(c0), "+d"(c1) : "d"(a), "d"(b));
}
template <int NACC>
__global__ void k(double *out, int iters) {
    double c[NACC][2];
    double a = threadIdx.x * 1e-3, b = blockIdx.x * 1e-3;
    for (int i = 0; i < NACC; ++i) c[i][0] = c[i][1] = 0.0;
    for (int it = 0; it < iters; ++it) {
#pragma unroll
        for (int i = 0; i < NACC; ++i) dmma(c[i][0], c[i][1], a, b);
    }
    double s = 0;
    for (int i = 0; i < NACC; ++i) s += c[i][0] + c[i][1];
    if (s == 123.456) out[0] = s;
}
int main() {
    double *out; cudaMalloc(&out, 8);
    int sms; cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, 0);
    cudaEvent_t e0, e1; cudaEventCreate(&e0); cudaEventCreate(&e1);
    for (int wps : {4, 8, 12, 16, 24, 32}) {
        const int iters = 4096;
        const int threads = 128, blocks = sms * wps / 4;
        k<16><<<blocks, threads>>>(out, 16);
        cudaEventRecord(e0);
        k<16><<<blocks, threads>>>(out, iters);
        cudaEventRecord(e1);
        cudaEventSynchronize(e1);
        float ms; cudaEventElapsedTime(&ms, e0, e1);
        double fl = 2.0 * 512 * 16.0 * iters * (blocks * threads / 32);
        printf("NACC=16 warps/SM=%2d: %.2f TF/s\n", wps, fl / (ms / 1e3) / 1e12);
    }
    for (int wps : {8, 16}) {
        const int iters = 4096;
        const int threads = 128, blocks = sms * wps / 4;
        k<4><<<blocks, threads>>>(out, 16);
        cudaEventRecord(e0);
        k<4><<<blocks, threads>>>(out, iters * 4);
        cudaEventRecord(e1);
        cudaEventSynchronize(e1);
        float ms; cudaEventElapsedTime(&ms, e0, e1);
        double fl = 2.0 * 512 * 4.0 * iters * 4 * (blocks * threads / 32);
        printf("NACC=4 warps/SM=%2d: %.2f TF/s\n", wps, fl / (ms / 1e3) / 1e12);
    }
    return 0;
}
