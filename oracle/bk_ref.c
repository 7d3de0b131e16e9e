/*
 * ORACLE — test infrastructure only.  Not part of the product path.
 *
 * Plain-C restatement of the reference's Bunch–Kaufman LDL^T kernel
 * (`/root/reference/pkg/src/h2slice/_core/_kernels.pyx:21-125`, dsytf2 lower
 * variant) and its inertia count (`_kernels.pyx:128-168`, `dense.py:127-168`).
 * Compiled with plain gcc -O2 (no -mfma), so every product and sum rounds
 * exactly as the reference's Cython build does: outputs are bit-identical to
 * `h2slice._core._kernels.bk_factor` (pinned by tests/test_oracle.py against
 * tests/golden/bk_*.npz).
 *
 * Storage: row-major n x n, only the lower triangle is read/written.
 * ipiv: kp >= 0 -> 1x1 pivot with rows k,kp swapped;
 *       ipiv[k] = ipiv[k+1] = -(kp+1) -> 2x2 pivot, rows k+1,kp swapped.
 * Returns 0, or k+1 when column k gives a pivot block at/below tol.
 */
#include <math.h>
#include <stdint.h>

#define AT(i, j) a[(int64_t)(i) * n + (j)]

static void swap_d(double *x, double *y) { double t = *x; *x = *y; *y = t; }

int oracle_bk_factor(double *a, int64_t n, int64_t *ipiv, double tol)
{
    const double alpha = (1.0 + sqrt(17.0)) / 8.0;
    int64_t k = 0;
    while (k < n) {
        int64_t step = 1, piv, imax = k;
        double akk = fabs(AT(k, k)), cmax = 0.0;
        for (int64_t i = k + 1; i < n; ++i) {
            double v = fabs(AT(i, k));
            if (v > cmax) { cmax = v; imax = i; }
        }
        if (akk >= alpha * cmax) {
            piv = k;
        } else {
            double rmax = 0.0;
            for (int64_t j = k; j < imax; ++j) { double v = fabs(AT(imax, j)); if (v > rmax) rmax = v; }
            for (int64_t i = imax + 1; i < n; ++i) { double v = fabs(AT(i, imax)); if (v > rmax) rmax = v; }
            if (akk * rmax >= alpha * cmax * cmax) piv = k;
            else if (fabs(AT(imax, imax)) >= alpha * rmax) piv = imax;
            else { piv = imax; step = 2; }
        }
        int64_t kk = k + step - 1;
        if (piv != kk) {
            for (int64_t i = piv + 1; i < n; ++i) swap_d(&AT(i, kk), &AT(i, piv));
            for (int64_t j = kk + 1; j < piv; ++j) swap_d(&AT(j, kk), &AT(piv, j));
            swap_d(&AT(kk, kk), &AT(piv, piv));
            if (step == 2) swap_d(&AT(kk, k), &AT(piv, k));
        }
        if (step == 1) {
            double d = AT(k, k);
            if (fabs(d) <= tol) return (int)(k + 1);
            double r = 1.0 / d;
            for (int64_t j = k + 1; j < n; ++j) {
                double w = r * AT(j, k);
                for (int64_t i = j; i < n; ++i) AT(i, j) -= AT(i, k) * w;
            }
            for (int64_t i = k + 1; i < n; ++i) AT(i, k) *= r;
            ipiv[k] = piv;
        } else {
            double e = AT(k + 1, k);
            double det = AT(k, k) * AT(k + 1, k + 1) - e * e;
            double bmax = fabs(e);
            if (fabs(AT(k, k)) > bmax) bmax = fabs(AT(k, k));
            if (fabs(AT(k + 1, k + 1)) > bmax) bmax = fabs(AT(k + 1, k + 1));
            if (fabs(det) <= tol * bmax) return (int)(k + 1);
            if (k < n - 2) {
                double p = AT(k + 1, k + 1) / e;
                double q = AT(k, k) / e;
                double t = 1.0 / (p * q - 1.0);
                double s = t / e;
                for (int64_t j = k + 2; j < n; ++j) {
                    double w0 = s * (p * AT(j, k) - AT(j, k + 1));
                    double w1 = s * (q * AT(j, k + 1) - AT(j, k));
                    for (int64_t i = j; i < n; ++i) AT(i, j) -= AT(i, k) * w0 + AT(i, k + 1) * w1;
                    AT(j, k) = w0;
                    AT(j, k + 1) = w1;
                }
            }
            ipiv[k] = -(piv + 1);
            ipiv[k + 1] = -(piv + 1);
        }
        k += step;
    }
    return 0;
}

/* (neg, zero, pos) over the factored block diagonal, zero tolerance zt. */
void oracle_bk_inertia(const double *a, int64_t n, const int64_t *ipiv, double zt, int64_t *out)
{
    int64_t neg = 0, zero = 0, pos = 0, k = 0;
    while (k < n) {
        if (ipiv[k] >= 0) {
            double d = AT(k, k);
            if (fabs(d) <= zt) ++zero; else if (d < 0.0) ++neg; else ++pos;
            k += 1;
        } else {
            double x = AT(k, k), y = AT(k + 1, k + 1), e = AT(k + 1, k);
            double det = x * y - e * e, tr = x + y;
            if (det < -zt * zt) { ++neg; ++pos; }
            else if (det > zt * zt) { if (tr < 0.0) neg += 2; else pos += 2; }
            else {
                ++zero;
                if (tr < -zt) ++neg; else if (tr > zt) ++pos; else ++zero;
            }
            k += 2;
        }
    }
    out[0] = neg; out[1] = zero; out[2] = pos;
}
