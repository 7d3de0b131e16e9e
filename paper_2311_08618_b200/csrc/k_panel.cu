// Elimination panel: gather + permute + unit-lower TRSM + block-diagonal
// D^{-1} scaling, fused (K4 + K5).
//
// Reference: gldl.py:365-378 builds Ball = [D_SR; partner slices] with
// np.vstack, solves W = Ball[:, perm] L^{-T} with scipy solve_triangular
// (dtrsm) and X = W D^{-1} with np.linalg.solve (a full LU of the block
// diagonal D).  The engine runs this kernel on the n x n identity (src ==
// nullptr), giving W_I = P^T L^{-T} and X_I = W_I D^{-1}; the panel of every
// partner block is then one DMMA GEMM with G = X_I W_I^T (engine.cu).  The
// kernel still accepts real source rows (gather folded into the tile load,
// transposed when the partner block is stored (i, j) with i eliminated).
//
// One CTA solves a 32-row tile for one shift: the tile lives in shared
// memory with an odd row stride, L is staged once into shared memory packed
// by columns (n <= PANEL_L_SMEM) so every step reads broadcast operands, and
// the solve runs right-looking, one barrier per column.  D^{-1} is applied
// per 1x1 / 2x2 pivot block (LAPACK dsytrs scaling for 2x2) - mathematically
// the reference's dense solve.
#include "common.cuh"

namespace h2l {

constexpr int PANEL_L_SMEM = 160;
constexpr int PANEL_LC = 16;  // widest L column chunk staged per pass when L does not fit
constexpr size_t PANEL_SMEM_CAP = 226 * 1024;

namespace {

// Register-resident right-looking solve of a 32-row tile: lane = row, warp w
// owns columns w + 8 j (j < NJ) of its row in registers; per column c the
// owning warp publishes T(:, c) through a double-buffered shared vector, one
// barrier per column, and every thread updates its own later columns with L
// read from shared memory.  Result written back to T.
template <int NJ>
__device__ __forceinline__ void solve_regs(double *T, int S, const double *Ls, const int *cs, int n,
                                           double (*colbuf)[PANEL_ROWS]) {
    const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
    double r[NJ];
#pragma unroll
    for (int j = 0; j < NJ; ++j) {
        const int c = warp + 8 * j;
        r[j] = c < n ? T[lane * S + c] : 0.0;
    }
    for (int c = 0; c < n - 1; ++c) {
        if ((c & 7) == warp) {
            const int jc = c >> 3;
            double v = 0.0;
#pragma unroll
            for (int j = 0; j < NJ; ++j)
                if (j == jc) v = r[j];
            colbuf[c & 1][lane] = v;
        }
        __syncthreads();
        const double wc = colbuf[c & 1][lane];
        const double *lc = Ls + cs[c];
#pragma unroll
        for (int j = 0; j < NJ; ++j) {
            const int cc = warp + 8 * j;
            if (cc > c && cc < n) r[j] -= wc * lc[cc];
        }
    }
#pragma unroll
    for (int j = 0; j < NJ; ++j) {
        const int c = warp + 8 * j;
        if (c < n) T[lane * S + c] = r[j];
    }
    __syncthreads();
}

__global__ void __launch_bounds__(256) panel_kernel(const PanelTile *tiles, const PanelJob *jobs) {
    extern __shared__ __align__(16) double sm[];
    __shared__ double colbuf[2][PANEL_ROWS];
    const PanelTile tl = tiles[blockIdx.x];
    const PanelJob jb = jobs[tl.job];
    const double *L = jb.L;
    const int64_t lstride = jb.lstride, pstride = jb.pstride, wstride = jb.wstride;
    const int ldl = jb.ldl, n = jb.n, ldw = jb.ldw, lcw = jb.lcw;
    const int *perm = jb.perm;
    const double *dinfo = jb.dinfo;
    double *W = jb.W, *X = jb.X;
    const int z = blockIdx.y;
    const int S = n + 1 + (n & 1);  // odd row stride -> conflict-free column access
    double *T = sm;                 // PANEL_ROWS x S
    const bool lsm = n <= PANEL_L_SMEM;
    double *Ls = T + PANEL_ROWS * S;  // packed strictly-lower L by columns
    int *cs = (int *)(Ls + (lsm ? (int64_t)n * (n - 1) / 2 : 0));
    const double *src = tl.src ? tl.src + z * tl.sstride : nullptr;
    const double *Lz = L + z * lstride;
    const int *pz = perm + z * pstride;
    const double *dz = dinfo + 3 * z * pstride;
    const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;

    if (lsm) {
        // column c holds rows c+1..n-1 at Ls[cs[c] + row]; cs[c] = c*n - c(c+1)/2 - (c+1)... (row offset)
        for (int c = threadIdx.x; c < n; c += blockDim.x) cs[c] = c * (n - 1) - (c * (c - 1)) / 2 - (c + 1);
        __syncthreads();
        for (int i = warp; i < n; i += 8)
            for (int c = lane; c < i; c += 32) {
                const bool two = dz[3 * c + 2] > 1.5 && i == c + 1;  // 2x2: L(c+1, c) = 0
                Ls[cs[c] + i] = two ? 0.0 : Lz[(int64_t)i * ldl + c];
            }
    }
    // ---- gather + permute (src == nullptr: the identity, i.e. W = P^T L^{-T})
    if (!src) {
        for (int r = warp; r < PANEL_ROWS; r += 8)
            for (int c = lane; c < n; c += 32)
                T[r * S + c] = (r < tl.nrows && pz[c] == tl.src_row0 + r) ? 1.0 : 0.0;
    } else if (tl.trans) {
        for (int c = warp; c < n; c += 8) {
            const int pc = pz[c];
            T[lane * S + c] = lane < tl.nrows ? src[(int64_t)pc * tl.lds + tl.src_row0 + lane] : 0.0;
        }
    } else {
        for (int r = warp; r < PANEL_ROWS; r += 8)
            for (int c = lane; c < n; c += 32)
                T[r * S + c] = r < tl.nrows ? src[(int64_t)(tl.src_row0 + r) * tl.lds + pz[c]] : 0.0;
    }
    __syncthreads();

    // ---- forward substitution with unit-lower L (L(c+1, c) of a 2x2 pivot is D, not L)
    double *trow = T + lane * S;
    if (lsm && n <= 32) solve_regs<4>(T, S, Ls, cs, n, colbuf);
    else if (lsm && n <= 64) solve_regs<8>(T, S, Ls, cs, n, colbuf);
    else if (lsm && n <= 128) solve_regs<16>(T, S, Ls, cs, n, colbuf);
    else if (lsm) solve_regs<20>(T, S, Ls, cs, n, colbuf);
    else {
        // L does not fit: stage it in column chunks of PANEL_LC (rows c0+1..n-1,
        // row-contiguous, coalesced) and run the same column steps from shared memory
        double *Lc = T + PANEL_ROWS * S;  // [n][lcw]
        for (int c0 = 0; c0 < n - 1; c0 += lcw) {
            const int nc = min(lcw, n - 1 - c0);
            __syncthreads();
            for (int e = threadIdx.x; e < (n - c0) * lcw; e += blockDim.x) {
                const int i = c0 + e / lcw, k = e % lcw;
                Lc[(int64_t)i * lcw + k] = (k < nc && i > c0 + k) ? Lz[(int64_t)i * ldl + c0 + k] : 0.0;
            }
            __syncthreads();
            for (int k = 0; k < nc; ++k) {
                const int c = c0 + k;
                const double wc = trow[c];
                const bool two = dz[3 * c + 2] > 1.5;
                for (int cc = c + 1 + warp; cc < n; cc += 8) {
                    const double l = (two && cc == c + 1) ? 0.0 : Lc[(int64_t)cc * lcw + k];
                    trow[cc] -= wc * l;
                }
                __syncthreads();
            }
        }
    }

    // ---- write W, then X = W D^{-1}
    if (lane < tl.nrows) {
        double *wrow = W + z * wstride + (int64_t)(tl.row0 + lane) * ldw;
        double *xrow = X + z * wstride + (int64_t)(tl.row0 + lane) * ldw;
        for (int c = warp; c < n; c += 8) wrow[c] = trow[c];
        for (int c = warp; c < n; c += 8) {
            const double bs = dz[3 * c + 2];
            if (bs > 1.5) {
                const double e = dz[3 * c + 1];
                const double a1 = dz[3 * c] / e, a2 = dz[3 * c + 3] / e;
                const double den = a1 * a2 - 1.0;
                const double b1 = trow[c] / e, b2 = trow[c + 1] / e;
                xrow[c] = (a2 * b1 - b2) / den;
                xrow[c + 1] = (a1 * b2 - b1) / den;
            } else if (bs > 0.5) {
                xrow[c] = trow[c] / dz[3 * c];
            }
        }
    }
}

}  // namespace

// width of the staged L chunk for n > PANEL_L_SMEM (the widest that fits)
int panel_lcw(int n) {
    int w = PANEL_LC;
    while (w > 1 && sizeof(double) * ((size_t)PANEL_ROWS * (n + 2) + (size_t)n * w) > PANEL_SMEM_CAP)
        w >>= 1;
    return w;
}

size_t panel_smem_bytes(int n) {
    size_t b = sizeof(double) * PANEL_ROWS * (size_t)(n + 2);
    if (n <= PANEL_L_SMEM) b += sizeof(double) * (size_t)n * (n - 1) / 2 + sizeof(int) * (size_t)n;
    else b += sizeof(double) * (size_t)n * panel_lcw(n);
    return b;
}

cudaError_t launch_panel_multi(const PanelTile *dev_tiles, int ntiles, int nshift,
                               const PanelJob *dev_jobs, size_t smem_bytes, cudaStream_t st) {
    if (ntiles <= 0 || nshift <= 0) return cudaSuccess;
    cudaError_t e = smem_optin(panel_kernel);
    if (e != cudaSuccess) return e;
    dim3 grid(ntiles, nshift);
    panel_kernel<<<grid, 256, smem_bytes, st>>>(dev_tiles, dev_jobs);
    return cudaGetLastError();
}

}  // namespace h2l
