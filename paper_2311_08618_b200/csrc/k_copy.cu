// Batched 2-D block copy / accumulate / zero / identity / diagonal shift.
//
// HBM-bound gather-scatter work of the elimination (Ball gathers, zeroing of
// eliminated rows, merge assembly, per-shift diagonal shift of the skeleton
// arena).  One CTA moves one 32x32 tile of one task for one shift; transposed
// reads are staged through shared memory so both the global read and the
// global write are coalesced (32 consecutive doubles per warp).
#include "common.cuh"

namespace h2l {

namespace {

constexpr int TILE = 32;

__device__ __forceinline__ int find_task(const int *prefix, int ntasks, int tile) {
    int lo = 0, hi = ntasks - 1;
    while (lo < hi) {
        int mid = (lo + hi + 1) >> 1;
        if (prefix[mid] <= tile) lo = mid; else hi = mid - 1;
    }
    return lo;
}

__global__ void __launch_bounds__(256) copy_kernel(const CopyTask *tasks, const int *prefix,
                                                   int ntasks, const double *mu) {
    __shared__ double tile_s[TILE][TILE + 1];
    const int t = find_task(prefix, ntasks, blockIdx.x);
    const CopyTask tk = tasks[t];
    const int local = blockIdx.x - prefix[t];
    const int tiles_c = (tk.cols + TILE - 1) / TILE;
    const int r0 = (local / tiles_c) * TILE;
    const int c0 = (local % tiles_c) * TILE;
    const int z = blockIdx.y;
    double *dst = tk.dst + z * tk.dstride;
    const double *src = tk.src ? tk.src + z * tk.sstride : nullptr;
    const double shift = (tk.shift_diag && mu) ? mu[z] : 0.0;
    const int tx = threadIdx.x & 31, ty = threadIdx.x >> 5;  // 32 x 8

    if (src && tk.trans) {
        // element (r, c) = src[c * lds + r]: read rows of src (= our columns)
        for (int k = ty; k < TILE; k += 8) {
            int c = c0 + k, r = r0 + tx;
            tile_s[k][tx] = (c < tk.cols && r < tk.rows) ? src[(int64_t)c * tk.lds + r] : 0.0;
        }
        __syncthreads();
    }
    for (int k = ty; k < TILE; k += 8) {
        int r = r0 + k, c = c0 + tx;
        if (r >= tk.rows || c >= tk.cols) continue;
        double v;
        if (!src) {
            v = (tk.ident && r == c) ? 1.0 : 0.0;
        } else if (tk.trans) {
            v = tile_s[tx][k];
        } else {
            v = src[(int64_t)r * tk.lds + c];
        }
        v *= tk.alpha;
        if (r == c) v -= shift;
        double *d = dst + (int64_t)r * tk.ldd + c;
        *d = tk.acc ? (*d + v) : v;
    }
}

}  // namespace

// Tile prefix is built on the device-side copy of the task list; to keep the
// launcher self-contained the prefix is computed by the host engine and
// appended after the tasks (see Engine::copy_flush).
void launch_copy_prefixed(const CopyTask *dev_tasks, const int *dev_prefix, int ntasks,
                          int total_tiles, int nshift, const double *mu, cudaStream_t st) {
    if (ntasks <= 0 || total_tiles <= 0 || nshift <= 0) return;
    dim3 grid(total_tiles, nshift);
    copy_kernel<<<grid, 256, 0, st>>>(dev_tasks, dev_prefix, ntasks, mu);
}

int copy_tiles(int rows, int cols) {
    if (rows <= 0 || cols <= 0) return 0;
    return ((rows + TILE - 1) / TILE) * ((cols + TILE - 1) / TILE);
}

}  // namespace h2l

namespace h2l {
namespace {
// out[z][e] = sum_s in[z][s * pstride + e], e < count (split-K partial sums, fixed order)
__global__ void __launch_bounds__(256) sum_partials_kernel(const double *in, int64_t zin,
                                                           int64_t pstride, int nparts,
                                                           double *out, int64_t zout,
                                                           int64_t count) {
    const int z = blockIdx.y;
    const double *src = in + z * zin;
    double *dst = out + z * zout;
    for (int64_t e = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; e < count;
         e += (int64_t)gridDim.x * blockDim.x) {
        double acc = 0.0;
        for (int s = 0; s < nparts; ++s) acc += src[s * pstride + e];
        dst[e] = acc;
    }
}
}  // namespace

void launch_sum_partials(const double *in, int64_t zin, int64_t pstride, int nparts, double *out,
                         int64_t zout, int64_t count, int nshift, cudaStream_t st) {
    if (count <= 0 || nshift <= 0) return;
    const int blocks = (int)std::min<int64_t>(1024, (count + 255) / 256);
    sum_partials_kernel<<<dim3(blocks, nshift), 256, 0, st>>>(in, zin, pstride, nparts, out, zout,
                                                               count);
}
}  // namespace h2l

namespace h2l {
namespace {
// split-K partial sums of several clusters' Gram products (blockIdx.z = job)
__global__ void __launch_bounds__(256) sum_partials_multi_kernel(const SumJob *jobs) {
    const SumJob jb = jobs[blockIdx.z];
    const int z = blockIdx.y;
    const double *src = jb.in + z * jb.zin;
    double *dst = jb.out + z * jb.zout;
    for (int64_t e = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; e < jb.count;
         e += (int64_t)gridDim.x * blockDim.x) {
        double acc = 0.0;
        for (int s = 0; s < jb.nparts; ++s) acc += src[s * jb.pstride + e];
        dst[e] = acc;
    }
}

// per-shift truncation (gldl.py:296-347 with each shift's own rank): zero the
// rows / columns [base + rank[z], base + t) of a block for shift z
__global__ void __launch_bounds__(256) tail_zero_kernel(const TailZeroJob *jobs) {
    const TailZeroJob jb = jobs[blockIdx.x];
    const int z = blockIdx.y;
    const int lo = jb.base + min(jb.rank[z], jb.t), hi = jb.base + jb.t;
    if (hi <= lo) return;
    double *p = jb.p + z * jb.bs;
    const int span = hi - lo;
    const int64_t tot = (int64_t)span * jb.other;
    for (int64_t e = threadIdx.x; e < tot; e += blockDim.x) {
        if (jb.orient == 0) {  // rows lo..hi-1, all `other` columns
            const int r = lo + (int)(e / jb.other), c = (int)(e % jb.other);
            p[(int64_t)r * jb.ld + c] = 0.0;
        } else {               // columns lo..hi-1 of all `other` rows
            const int r = (int)(e / span), c = lo + (int)(e % span);
            p[(int64_t)r * jb.ld + c] = 0.0;
        }
    }
}
}  // namespace

void launch_sum_partials_multi(const SumJob *jobs, int njobs, int64_t max_count, int nshift,
                               cudaStream_t st) {
    if (njobs <= 0 || max_count <= 0 || nshift <= 0) return;
    const int blocks = (int)std::min<int64_t>(256, (max_count + 255) / 256);
    sum_partials_multi_kernel<<<dim3(blocks, nshift, njobs), 256, 0, st>>>(jobs);
}

cudaError_t launch_tail_zero(const TailZeroJob *jobs, int njobs, int nshift, cudaStream_t st) {
    if (njobs <= 0 || nshift <= 0) return cudaSuccess;
    tail_zero_kernel<<<dim3(njobs, nshift), 256, 0, st>>>(jobs);
    return cudaGetLastError();
}
}  // namespace h2l
