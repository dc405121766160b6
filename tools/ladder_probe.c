/* Reading G25: why the GPU fp64 paths sit at e/(kappa eps) ~ 0.06 while the
 * round-1 SURVEY probe (textbook GJ on [A|I], per-element division) showed ~0.015.
 *
 * Runs, on the same Gaussian n x n items (fixed LCG + Box-Muller, seed argv[3]), four fp64
 * Gauss-Jordan variants that differ only in the arithmetic the kernels changed, each
 * against a long-double reference, and prints max over items of e / (kappa_inf eps):
 *   D  textbook: [A | I], pivot row divided element by element, x -= f y  (the probe)
 *   R  pivot row multiplied by the reciprocal 1/p instead of divided
 *   F  R plus fused multiply-add for the elimination (fma(-f, y, x))
 *   G  the kernels' form: compact storage, deferred normalisation (multiplier x_ik * (1/p),
 *      each row scaled by its own pivot's reciprocal at the end), FMA
 * Test tooling only:  gcc -O2 -o /tmp/ladder_probe tools/ladder_probe.c -lm
 *                     /tmp/ladder_probe 32 2000 7
 */
#include <math.h>
#include <stdint.h>
#include <stdio.h>
#include <stdlib.h>
#include <string.h>

static uint64_t st;
static double urand(void) {
    st = st * 6364136223846793005ULL + 1442695040888963407ULL;
    return ((st >> 11) + 0.5) * (1.0 / 9007199254740992.0);
}
static double nrand(void) { return sqrt(-2.0 * log(urand())) * cos(6.283185307179586 * urand()); }

typedef long double ld;

/* reference inverse in long double (textbook, partial pivoting) */
static void inv_ld(int n, const double* A, ld* X) {
    ld* M = calloc((size_t)n * 2 * n, sizeof(ld));
    for (int i = 0; i < n; ++i) {
        for (int j = 0; j < n; ++j) M[i * 2 * n + j] = A[i * n + j];
        M[i * 2 * n + n + i] = 1;
    }
    for (int k = 0; k < n; ++k) {
        int r = k;
        for (int i = k + 1; i < n; ++i)
            if (fabsl(M[i * 2 * n + k]) > fabsl(M[r * 2 * n + k])) r = i;
        if (r != k)
            for (int j = 0; j < 2 * n; ++j) { ld t = M[k * 2 * n + j]; M[k * 2 * n + j] = M[r * 2 * n + j]; M[r * 2 * n + j] = t; }
        ld p = M[k * 2 * n + k];
        for (int j = 0; j < 2 * n; ++j) M[k * 2 * n + j] /= p;
        for (int i = 0; i < n; ++i) {
            if (i == k) continue;
            ld f = M[i * 2 * n + k];
            for (int j = 0; j < 2 * n; ++j) M[i * 2 * n + j] -= f * M[k * 2 * n + j];
        }
    }
    for (int i = 0; i < n; ++i)
        for (int j = 0; j < n; ++j) X[i * n + j] = M[i * 2 * n + n + j];
    free(M);
}

/* variants D / R / F on [A | I] in double */
static void inv_aug(int n, const double* A, double* X, int mode) {
    double* M = calloc((size_t)n * 2 * n, sizeof(double));
    for (int i = 0; i < n; ++i) {
        for (int j = 0; j < n; ++j) M[i * 2 * n + j] = A[i * n + j];
        M[i * 2 * n + n + i] = 1;
    }
    for (int k = 0; k < n; ++k) {
        int r = k;
        for (int i = k + 1; i < n; ++i)
            if (fabs(M[i * 2 * n + k]) > fabs(M[r * 2 * n + k])) r = i;
        if (r != k)
            for (int j = 0; j < 2 * n; ++j) { double t = M[k * 2 * n + j]; M[k * 2 * n + j] = M[r * 2 * n + j]; M[r * 2 * n + j] = t; }
        double p = M[k * 2 * n + k], rp = 1.0 / p;
        for (int j = 0; j < 2 * n; ++j) M[k * 2 * n + j] = mode == 0 ? M[k * 2 * n + j] / p : M[k * 2 * n + j] * rp;
        for (int i = 0; i < n; ++i) {
            if (i == k) continue;
            double f = M[i * 2 * n + k];
            for (int j = 0; j < 2 * n; ++j)
                M[i * 2 * n + j] = mode == 2 ? fma(-f, M[k * 2 * n + j], M[i * 2 * n + j]) : M[i * 2 * n + j] - f * M[k * 2 * n + j];
        }
    }
    for (int i = 0; i < n; ++i)
        for (int j = 0; j < n; ++j) X[i * n + j] = M[i * 2 * n + n + j];
    free(M);
}

/* variant G: compact storage, logical pivoting, deferred normalisation, FMA */
static void inv_kernel_form(int n, const double* A, double* X) {
    double* T = malloc((size_t)n * n * sizeof(double));
    int *pst = malloc(n * sizeof(int)), *row_of = malloc(n * sizeof(int)), *pos = malloc(n * sizeof(int));
    double* piv = malloc(n * sizeof(double));
    memcpy(T, A, (size_t)n * n * sizeof(double));
    for (int i = 0; i < n; ++i) { pst[i] = -1; pos[i] = i; }
    for (int k = 0; k < n; ++k) {
        int r = -1;
        for (int i = 0; i < n; ++i) {
            if (pst[i] >= 0) continue;
            if (r < 0 || fabs(T[i * n + k]) > fabs(T[r * n + k]) ||
                (fabs(T[i * n + k]) == fabs(T[r * n + k]) && pos[i] < pos[r])) r = i;
        }
        int q = pos[r];
        for (int i = 0; i < n; ++i) if (pst[i] < 0 && pos[i] == k) pos[i] = q;
        pos[r] = k;
        pst[r] = k;
        row_of[k] = r;
        double p = T[r * n + k], rp = 1.0 / p;
        piv[k] = p;
        double y[256];
        for (int j = 0; j < n; ++j) y[j] = T[r * n + j];
        for (int i = 0; i < n; ++i) {
            if (i == r) { T[i * n + k] = 1.0; continue; }
            double nf = -(T[i * n + k] * rp);
            for (int j = 0; j < n; ++j) if (j != k) T[i * n + j] = fma(nf, y[j], T[i * n + j]);
            T[i * n + k] = nf;
        }
    }
    /* un-permutation: Ainv[k][row_of[k']] = T[row_of[k]][k'] / p_k */
    for (int k = 0; k < n; ++k) {
        int i = row_of[k];
        double rp = 1.0 / piv[k];
        for (int kp = 0; kp < n; ++kp) X[k * n + row_of[kp]] = T[i * n + kp] * rp;
    }
    free(T); free(pst); free(row_of); free(pos); free(piv);
}

int main(int argc, char** argv) {
    int n = argc > 1 ? atoi(argv[1]) : 32;
    int items = argc > 2 ? atoi(argv[2]) : 2000;
    st = argc > 3 ? strtoull(argv[3], 0, 10) : 7;
    double* A = malloc((size_t)n * n * sizeof(double));
    double* X = malloc((size_t)n * n * sizeof(double));
    ld* R = malloc((size_t)n * n * sizeof(ld));
    double worst[4] = {0, 0, 0, 0};
    const double eps = ldexp(1.0, -52);
    for (int it = 0; it < items; ++it) {
        for (int t = 0; t < n * n; ++t) A[t] = nrand();
        inv_ld(n, A, R);
        ld na = 0, nx = 0, mx = 0;
        for (int i = 0; i < n; ++i) {
            ld sa = 0, sx = 0;
            for (int j = 0; j < n; ++j) { sa += fabsl((ld)A[i * n + j]); sx += fabsl(R[i * n + j]); if (fabsl(R[i * n + j]) > mx) mx = fabsl(R[i * n + j]); }
            if (sa > na) na = sa;
            if (sx > nx) nx = sx;
        }
        double kappa = (double)(na * nx);
        for (int v = 0; v < 4; ++v) {
            if (v < 3) inv_aug(n, A, X, v); else inv_kernel_form(n, A, X);
            ld e = 0;
            for (int t = 0; t < n * n; ++t) { ld d = fabsl((ld)X[t] - R[t]); if (d > e) e = d; }
            double ratio = (double)(e / mx) / (kappa * eps);
            if (ratio > worst[v]) worst[v] = ratio;
        }
    }
    printf("n=%d items=%d  max e/(kappa eps):  D (divide) %.4f   R (reciprocal) %.4f   F (+FMA) %.4f   G (kernel form) %.4f\n",
           n, items, worst[0], worst[1], worst[2], worst[3]);
    return 0;
}
