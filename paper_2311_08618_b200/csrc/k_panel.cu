// Elimination panel: gather + permute + unit-lower TRSM + block-diagonal
// D^{-1} scaling, fused (K4 + K5).
//
// Reference: gldl.py:365-378 builds Ball = [D_SR; partner slices] with
// np.vstack, solves W = Ball[:, perm] L^{-T} with scipy solve_triangular
// (dtrsm) and X = W D^{-1} with np.linalg.solve (a full LU of the block
// diagonal D).  Here the gather is folded into the tile load (each tile reads
// its rows straight from the source block, transposed when the partner block
// is stored (i, j) with i the eliminated cluster), the permutation is applied
// on load, the solve runs right-looking on a 32-row tile held in shared
// memory, and D^{-1} is applied per 1x1 / 2x2 pivot block (LAPACK dsytrs
// scaling for the 2x2 case) - mathematically identical to the reference's
// dense solve and ~100x cheaper.
#include "common.cuh"

namespace h2l {

namespace {

__global__ void __launch_bounds__(256) panel_kernel(const PanelTile *tiles, const double *L,
                                                    int64_t lstride, int ldl, int n,
                                                    const int *perm, const double *dinfo,
                                                    int64_t pstride, double *W, double *X,
                                                    int64_t wstride, int ldw) {
    extern __shared__ __align__(16) double sm[];
    const int S = n + 1 + (n & 1);  // odd row stride -> conflict-free column access
    double *T = sm;       // PANEL_ROWS x S
    const PanelTile tl = tiles[blockIdx.x];
    const int z = blockIdx.y;
    const double *src = tl.src + z * tl.sstride;
    const double *Lz = L + z * lstride;
    const int *pz = perm + z * pstride;
    const double *dz = dinfo + 3 * z * pstride;
    const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;

    // ---- gather + permute
    if (tl.trans) {
        // panel row r = column (src_row0 + r) of src; lanes run along the row of src
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
    for (int c = 0; c < n - 1; ++c) {
        const double wc = T[lane * S + c];
        const bool two = dz[3 * c + 2] > 1.5;
        for (int cc = c + 1 + warp; cc < n; cc += 8) {
            const double l = (two && cc == c + 1) ? 0.0 : __ldg(Lz + (int64_t)cc * ldl + c);
            T[lane * S + cc] -= wc * l;
        }
        __syncthreads();
    }

    // ---- write W, then X = W D^{-1}
    if (lane < tl.nrows) {
        double *wrow = W + z * wstride + (int64_t)(tl.row0 + lane) * ldw;
        double *xrow = X + z * wstride + (int64_t)(tl.row0 + lane) * ldw;
        for (int c = warp; c < n; c += 8) wrow[c] = T[lane * S + c];
        for (int c = warp; c < n; c += 8) {
            const double bs = dz[3 * c + 2];
            if (bs > 1.5) {
                const double e = dz[3 * c + 1];
                const double a1 = dz[3 * c] / e, a2 = dz[3 * c + 3] / e;
                const double den = a1 * a2 - 1.0;
                const double b1 = T[lane * S + c] / e, b2 = T[lane * S + c + 1] / e;
                xrow[c] = (a2 * b1 - b2) / den;
                xrow[c + 1] = (a1 * b2 - b1) / den;
            } else if (bs > 0.5) {
                xrow[c] = T[lane * S + c] / dz[3 * c];
            }
        }
    }
}

}  // namespace

size_t panel_smem_bytes(int n) { return sizeof(double) * PANEL_ROWS * (size_t)(n + 2); }

cudaError_t launch_panel(const PanelTile *dev_tiles, int ntiles, int nshift, const double *L,
                         int64_t lstride, int ldl, int n, const int *perm, const double *dinfo,
                         int64_t pstride, double *W, double *X, int64_t wstride, int ldw,
                         cudaStream_t st) {
    if (ntiles <= 0 || nshift <= 0 || n <= 0) return cudaSuccess;
    size_t sm = panel_smem_bytes(n);
    cudaError_t e =
        cudaFuncSetAttribute(panel_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)sm);
    if (e != cudaSuccess) return e;
    dim3 grid(ntiles, nshift);
    panel_kernel<<<grid, 256, sm, st>>>(dev_tiles, L, lstride, ldl, n, perm, dinfo, pstride, W, X,
                                        wstride, ldw);
    return cudaGetLastError();
}

}  // namespace h2l
