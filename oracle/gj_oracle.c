/*
 * oracle/gj_oracle.c — CPU ORACLE. TEST INFRASTRUCTURE ONLY.
 *
 * Only tests/, __graft_entry__.smoke() and bench.py's cpu_baseline / --impl reference
 * leg may load this library. The product path (paper_1401_7962_b200/) never links,
 * imports or executes anything under oracle/, and this file shares no code, header,
 * table or helper with it.
 *
 * What it computes: the textbook Gauss–Jordan diagonalisation of the augmented
 * system [A | I] -> [I | A^-1] with max-|a_ik| partial pivoting, in x87 long double,
 * following the paper (arxiv 1401.7962, /root/reference/PAPER.md) step by step:
 *
 *   O1  A^0 = A, D^0 = I, held side by side as one n x 2n array M = [A | D]
 *       ............................................ Eqs. (1)-(2)
 *   O2  s = max |a_ij|, tau = tol * s  (zero threshold "prag de zero prestabilit",
 *       Obs. 2; relative reading G1 of SURVEY.md §8c / DESIGN.md)
 *   O3  for k = 1..n:
 *       a. pivot search: r = first i in k..n attaining max |M[i][k]|
 *          (Obs. 3 "valoare absolut maximă"; strict '>' scan of the
 *          listing, but on |.| — readings G2, G3)
 *       b. |M[r][k]| <= tau  =>  singular at step k (Obs. 2): stop
 *       c. swap rows k and r across all 2n columns (listing PAPER.md)
 *       d. p = M[k][k]; accumulate log|p|, sign, product (Eq. (13), PAPER.md L54,
 *          with the row-swap sign the paper omits — reading G4)
 *       e. M[k][j] /= p for all 2n columns              (Eq. (14))
 *       f. for i != k: M[i][j] -= M[i][k] * M[k][j]     (Eq. (15), PAPER.md L65-L67,
 *          with d_kj^k in the D line — reading G5, consistent with Eq. (8))
 *   O4  A^-1 = right half of M                           (Eq. (12))
 *       No de-pivoting here: the row swaps were applied to D as well, so the right
 *       half already is A^-1 (reading G6). The GPU path (compact storage + logical
 *       swaps + un-permutation) is therefore checked against an independent route.
 *   O5  det = (-1)^swaps * prod p_k, logabsdet = sum log|p_k|, sign.
 *
 * gjo_invert_full: full pivoting (Obs. 2-3, rows AND columns), see F1-F3 below.
 * gjo_solve: the same elimination on [A | B] (multi-RHS solve, Eq. (12) with B for I).
 *
 * Strategy 0 ("none", Eqs. (3)-(10) literally, pivot = a_kk) is kept
 * for tests of "a zero pivot does not imply singularity" (Obs. 2).
 *
 * Diagnostics used by the parity rules (R3/R7): per step the relative gap
 * between the two largest candidates, gap_k = (c1 - c2) / c1, and c1 / s.
 */
#include <math.h>
#include <stdint.h>
#include <stdlib.h>
#include <string.h>
#ifdef _OPENMP
#include <omp.h>
#endif

typedef long double ld;

/* Single matrix.  A: n*n row-major doubles (fp32 inputs are widened exactly by the
 * caller).  All output pointers may be NULL.  Returns 0, or -1 on allocation failure. */
int gjo_invert(int n, const double* A, double tol, int strategy,
               double* Ainv, int32_t* ipiv, double* pivots,
               double* logabsdet, int32_t* sign, double* det, int32_t* info,
               double* gap, double* cmax_rel, int inner_threads)
{
    const int w = 2 * n;
    ld* M = (ld*)malloc(sizeof(ld) * (size_t)n * (size_t)w);
    if (!M && n > 0) return -1;

    /* O1: M = [A | I] */
    ld s = 0.0L;
    for (int i = 0; i < n; ++i) {
        for (int j = 0; j < n; ++j) {
            ld a = (ld)A[(size_t)i * n + j];
            M[(size_t)i * w + j] = a;
            M[(size_t)i * w + n + j] = (i == j) ? 1.0L : 0.0L;
            if (fabsl(a) > s) s = fabsl(a);
        }
    }
    /* O2 */
    const ld tau = (ld)tol * s;

    int swaps = 0, neg = 0, fail = 0;
    ld logabs = 0.0L, prod = 1.0L;
    for (int k = 0; k < n; ++k) {
        /* O3a: candidates |M[i][k]|, i = k..n-1; first maximum wins */
        int r = k;
        ld c1 = fabsl(M[(size_t)k * w + k]), c2 = -1.0L;
        if (strategy == 1) {
            for (int i = k + 1; i < n; ++i) {
                ld c = fabsl(M[(size_t)i * w + k]);
                if (c > c1) { c2 = c1; c1 = c; r = i; }
                else if (c > c2) { c2 = c; }
            }
        }
        if (gap) gap[k] = (c2 < 0.0L) ? INFINITY : (c1 > 0.0L ? (double)((c1 - c2) / c1) : 0.0);
        if (cmax_rel) cmax_rel[k] = (s > 0.0L) ? (double)(c1 / s) : 0.0;
        if (ipiv) ipiv[k] = r + 1;
        /* O3b: zero threshold */
        if (c1 <= tau) { fail = k + 1; break; }
        /* O3c: physical row swap over all 2n columns */
        if (r != k) {
            ld* Rk = M + (size_t)k * w;
            ld* Rr = M + (size_t)r * w;
            for (int j = 0; j < w; ++j) { ld t = Rk[j]; Rk[j] = Rr[j]; Rr[j] = t; }
            swaps ^= 1;
        }
        /* O3d: Eq. (13) */
        ld* Rk = M + (size_t)k * w;
        const ld p = Rk[k];
        if (pivots) pivots[k] = (double)p;
        logabs += logl(fabsl(p));
        if (p < 0.0L) neg ^= 1;
        prod *= p;
        /* O3e: Eq. (14) */
        for (int j = 0; j < w; ++j) Rk[j] = Rk[j] / p;
        /* O3f: Eq. (15) */
#ifdef _OPENMP
#pragma omp parallel for schedule(static) num_threads(inner_threads) if (inner_threads > 1)
#endif
        for (int i = 0; i < n; ++i) {
            if (i == k) continue;
            ld* Ri = M + (size_t)i * w;
            const ld f = Ri[k];
            if (f == 0.0L) continue;   /* row unchanged: M[i][j] - 0*M[k][j] == M[i][j] for finite M */
            for (int j = 0; j < w; ++j) Ri[j] = Ri[j] - f * Rk[j];
        }
    }

    if (info) *info = fail;
    if (fail) {
        if (logabsdet) *logabsdet = -INFINITY;
        if (sign) *sign = 0;
        if (det) *det = 0.0;
        if (Ainv) for (size_t t = 0; t < (size_t)n * n; ++t) Ainv[t] = NAN;
        if (pivots) for (int k = fail - 1; k < n; ++k) pivots[k] = 0.0;
        if (ipiv) for (int k = fail; k < n; ++k) ipiv[k] = 0;
        if (gap) for (int k = fail; k < n; ++k) gap[k] = NAN;
        if (cmax_rel) for (int k = fail; k < n; ++k) cmax_rel[k] = NAN;
    } else {
        /* O4: Eq. (12) */
        if (Ainv)
            for (int i = 0; i < n; ++i)
                for (int j = 0; j < n; ++j)
                    Ainv[(size_t)i * n + j] = (double)M[(size_t)i * w + n + j];
        /* O5 */
        if (logabsdet) *logabsdet = (double)logabs;
        if (sign) *sign = ((swaps ^ neg) ? -1 : 1);
        if (det) *det = (double)(swaps ? -prod : prod);
    }
    free(M);
    return 0;
}

/* Batch of independent matrices, OpenMP over items.  A: batch*n*n doubles.
 * Per-item outputs are laid out item-major ([batch][n][n], [batch][n], [batch]). */
int gjo_invert_batched(int n, int64_t batch, const double* A, double tol, int strategy,
                       double* Ainv, int32_t* ipiv, double* pivots,
                       double* logabsdet, int32_t* sign, double* det, int32_t* info,
                       double* gap, double* cmax_rel, int nthreads)
{
    int err = 0;
    const size_t nn = (size_t)n * n;
#ifdef _OPENMP
#pragma omp parallel for schedule(dynamic, 16) num_threads(nthreads > 0 ? nthreads : omp_get_max_threads()) reduction(|:err)
#endif
    for (int64_t b = 0; b < batch; ++b) {
        err |= gjo_invert(n, A + b * nn, tol, strategy,
                          Ainv ? Ainv + b * nn : NULL,
                          ipiv ? ipiv + b * n : NULL,
                          pivots ? pivots + b * n : NULL,
                          logabsdet ? logabsdet + b : NULL,
                          sign ? sign + b : NULL,
                          det ? det + b : NULL,
                          info ? info + b : NULL,
                          gap ? gap + b * n : NULL,
                          cmax_rel ? cmax_rel + b * n : NULL, 1);
    }
    return err ? -1 : 0;
}

/* Full pivoting: Obs. 2-3 literally — at step k
 * any a_ij, i, j = k..n, may be brought to the pivot position by swapping rows k and i
 * and columns k and j; Obs. 3 takes the one of maximum |a_ij|; "at the end the row and
 * column swaps must be undone".
 *
 *   F1  M = [A | I] (n x 2n), s = max |a_ij|, tau = tol * s            (as O1-O2)
 *   F2  for k = 1..n:
 *       a. (r, c) = first (i, j) in the row-major scan of i = k..n, j = k..n attaining
 *          max |M[i][j]| (strict '>' as the listing's scan, L151-L153; reading G23)
 *       b. |M[r][c]| <= tau => singular at step k (Obs. 2)
 *       c. swap rows k and r over all 2n columns; swap columns k and c of the A half
 *          (the D half's columns are the unknowns' right-hand sides, never swapped)
 *       d. p = M[k][k]; Eq. (13) with the sign of BOTH swaps (det(A Q) = det(A) det(Q))
 *       e. Eq. (14): row k /= p;  f. Eq. (15): rows i != k -= M[i][k] * row k
 *   F3  the right half R = (A Q)^-1 = Q^T A^-1, Q = T_1 ... T_n the column swaps, so
 *       A^-1 = Q R: apply the column swaps in reverse order to the ROWS of R
 *       ("trebuie efectuate din nou schimbarea de linii și coloane", Obs. 3).
 * ipiv[k] = r + 1, jpiv[k] = c + 1 (1-based positions, LAPACK getc2 convention).
 * gap[k] = (c1 - c2) / c1 over all (n-k)^2 candidates of step k. */
int gjo_invert_full(int n, const double* A, double tol, double* Ainv, int32_t* ipiv, int32_t* jpiv,
                    double* pivots, double* logabsdet, int32_t* sign, double* det, int32_t* info, double* gap,
                    double* cmax_rel)
{
    const int w = 2 * n;
    ld* M = (ld*)malloc(sizeof(ld) * (size_t)n * (size_t)w);
    int* cp = (int*)malloc(sizeof(int) * (size_t)(n > 0 ? n : 1));
    if ((!M || !cp) && n > 0) { free(M); free(cp); return -1; }
    /* F1 */
    ld s = 0.0L;
    for (int i = 0; i < n; ++i)
        for (int j = 0; j < n; ++j) {
            ld a = (ld)A[(size_t)i * n + j];
            M[(size_t)i * w + j] = a;
            M[(size_t)i * w + n + j] = (i == j) ? 1.0L : 0.0L;
            if (fabsl(a) > s) s = fabsl(a);
        }
    const ld tau = (ld)tol * s;
    int swaps = 0, neg = 0, fail = 0;
    ld logabs = 0.0L, prod = 1.0L;
    for (int k = 0; k < n; ++k) {
        /* F2a */
        int r = k, c = k;
        ld c1 = -1.0L, c2 = -1.0L;
        for (int i = k; i < n; ++i)
            for (int j = k; j < n; ++j) {
                ld v = fabsl(M[(size_t)i * w + j]);
                if (v > c1) { c2 = c1; c1 = v; r = i; c = j; }
                else if (v > c2) { c2 = v; }
            }
        if (gap) gap[k] = (c2 < 0.0L) ? INFINITY : (c1 > 0.0L ? (double)((c1 - c2) / c1) : 0.0);
        if (cmax_rel) cmax_rel[k] = (s > 0.0L) ? (double)(c1 / s) : 0.0;
        if (ipiv) ipiv[k] = r + 1;
        if (jpiv) jpiv[k] = c + 1;
        cp[k] = c;
        /* F2b */
        if (c1 <= tau) { fail = k + 1; break; }
        /* F2c */
        if (r != k) {
            for (int j = 0; j < w; ++j) {
                ld t = M[(size_t)k * w + j]; M[(size_t)k * w + j] = M[(size_t)r * w + j]; M[(size_t)r * w + j] = t;
            }
            swaps ^= 1;
        }
        if (c != k) {
            for (int i = 0; i < n; ++i) {
                ld t = M[(size_t)i * w + k]; M[(size_t)i * w + k] = M[(size_t)i * w + c]; M[(size_t)i * w + c] = t;
            }
            swaps ^= 1;
        }
        /* F2d */
        ld* Rk = M + (size_t)k * w;
        const ld p = Rk[k];
        if (pivots) pivots[k] = (double)p;
        logabs += logl(fabsl(p));
        if (p < 0.0L) neg ^= 1;
        prod *= p;
        /* F2e */
        for (int j = 0; j < w; ++j) Rk[j] = Rk[j] / p;
        /* F2f */
        for (int i = 0; i < n; ++i) {
            if (i == k) continue;
            ld* Ri = M + (size_t)i * w;
            const ld f = Ri[k];
            if (f == 0.0L) continue;
            for (int j = 0; j < w; ++j) Ri[j] = Ri[j] - f * Rk[j];
        }
    }
    if (info) *info = fail;
    if (fail) {
        if (logabsdet) *logabsdet = -INFINITY;
        if (sign) *sign = 0;
        if (det) *det = 0.0;
        if (Ainv) for (size_t t = 0; t < (size_t)n * n; ++t) Ainv[t] = NAN;
        if (pivots) for (int k = fail - 1; k < n; ++k) pivots[k] = 0.0;
        if (ipiv) for (int k = fail; k < n; ++k) ipiv[k] = 0;
        if (jpiv) for (int k = fail; k < n; ++k) jpiv[k] = 0;
        if (gap) for (int k = fail; k < n; ++k) gap[k] = NAN;
        if (cmax_rel) for (int k = fail; k < n; ++k) cmax_rel[k] = NAN;
    } else {
        /* F3: undo the column swaps on the rows of the right half, last swap first */
        for (int k = n - 1; k >= 0; --k) {
            const int c = cp[k];
            if (c == k) continue;
            for (int j = n; j < w; ++j) {
                ld t = M[(size_t)k * w + j]; M[(size_t)k * w + j] = M[(size_t)c * w + j]; M[(size_t)c * w + j] = t;
            }
        }
        if (Ainv)
            for (int i = 0; i < n; ++i)
                for (int j = 0; j < n; ++j)
                    Ainv[(size_t)i * n + j] = (double)M[(size_t)i * w + n + j];
        if (logabsdet) *logabsdet = (double)logabs;
        if (sign) *sign = ((swaps ^ neg) ? -1 : 1);
        if (det) *det = (double)(swaps ? -prod : prod);
    }
    free(M);
    free(cp);
    return 0;
}

int gjo_invert_full_batched(int n, int64_t batch, const double* A, double tol, double* Ainv, int32_t* ipiv,
                            int32_t* jpiv, double* pivots, double* logabsdet, int32_t* sign, double* det,
                            int32_t* info, double* gap, double* cmax_rel, int nthreads)
{
    int err = 0;
    const size_t nn = (size_t)n * n;
#ifdef _OPENMP
#pragma omp parallel for schedule(dynamic, 16) num_threads(nthreads > 0 ? nthreads : omp_get_max_threads()) reduction(|:err)
#endif
    for (int64_t b = 0; b < batch; ++b)
        err |= gjo_invert_full(n, A + b * nn, tol, Ainv ? Ainv + b * nn : NULL, ipiv ? ipiv + b * n : NULL,
                               jpiv ? jpiv + b * n : NULL, pivots ? pivots + b * n : NULL,
                               logabsdet ? logabsdet + b : NULL, sign ? sign + b : NULL, det ? det + b : NULL,
                               info ? info + b : NULL, gap ? gap + b * n : NULL,
                               cmax_rel ? cmax_rel + b * n : NULL);
    return err ? -1 : 0;
}

/* Multi-RHS solve: the same Gauss–Jordan with the right-hand sides B
 * (n x m) in place of the identity — M = [A | B], Eqs. (14)-(15) on all n + m columns, the
 * listing's partial pivoting (O3a-O3c); at the end M = [I | A^-1 B] (Eq. (12) with B for I).
 * X: n x m row-major.  ipiv / logabsdet / sign / info as gjo_invert. */
int gjo_solve(int n, int m, const double* A, const double* B, double tol, double* X, int32_t* ipiv,
              double* logabsdet, int32_t* sign, int32_t* info, double* gap)
{
    const int w = n + m;
    ld* M = (ld*)malloc(sizeof(ld) * (size_t)n * (size_t)(w > 0 ? w : 1));
    if (!M && n > 0) return -1;
    ld s = 0.0L;
    for (int i = 0; i < n; ++i) {
        for (int j = 0; j < n; ++j) {
            ld a = (ld)A[(size_t)i * n + j];
            M[(size_t)i * w + j] = a;
            if (fabsl(a) > s) s = fabsl(a);
        }
        for (int j = 0; j < m; ++j) M[(size_t)i * w + n + j] = (ld)B[(size_t)i * m + j];
    }
    const ld tau = (ld)tol * s;
    int swaps = 0, neg = 0, fail = 0;
    ld logabs = 0.0L;
    for (int k = 0; k < n; ++k) {
        int r = k;
        ld c1 = fabsl(M[(size_t)k * w + k]), c2 = -1.0L;
        for (int i = k + 1; i < n; ++i) {
            ld c = fabsl(M[(size_t)i * w + k]);
            if (c > c1) { c2 = c1; c1 = c; r = i; }
            else if (c > c2) { c2 = c; }
        }
        if (gap) gap[k] = (c2 < 0.0L) ? INFINITY : (c1 > 0.0L ? (double)((c1 - c2) / c1) : 0.0);
        if (ipiv) ipiv[k] = r + 1;
        if (c1 <= tau) { fail = k + 1; break; }
        if (r != k) {
            for (int j = 0; j < w; ++j) {
                ld t = M[(size_t)k * w + j]; M[(size_t)k * w + j] = M[(size_t)r * w + j]; M[(size_t)r * w + j] = t;
            }
            swaps ^= 1;
        }
        ld* Rk = M + (size_t)k * w;
        const ld p = Rk[k];
        logabs += logl(fabsl(p));
        if (p < 0.0L) neg ^= 1;
        for (int j = 0; j < w; ++j) Rk[j] = Rk[j] / p;
        for (int i = 0; i < n; ++i) {
            if (i == k) continue;
            ld* Ri = M + (size_t)i * w;
            const ld f = Ri[k];
            if (f == 0.0L) continue;
            for (int j = 0; j < w; ++j) Ri[j] = Ri[j] - f * Rk[j];
        }
    }
    if (info) *info = fail;
    if (fail) {
        if (logabsdet) *logabsdet = -INFINITY;
        if (sign) *sign = 0;
        if (X) for (size_t t = 0; t < (size_t)n * m; ++t) X[t] = NAN;
        if (ipiv) for (int k = fail; k < n; ++k) ipiv[k] = 0;
        if (gap) for (int k = fail; k < n; ++k) gap[k] = NAN;
    } else {
        if (X)
            for (int i = 0; i < n; ++i)
                for (int j = 0; j < m; ++j) X[(size_t)i * m + j] = (double)M[(size_t)i * w + n + j];
        if (logabsdet) *logabsdet = (double)logabs;
        if (sign) *sign = ((swaps ^ neg) ? -1 : 1);
    }
    free(M);
    return 0;
}

int gjo_solve_batched(int n, int m, int64_t batch, const double* A, const double* B, double tol, double* X,
                      int32_t* ipiv, double* logabsdet, int32_t* sign, int32_t* info, double* gap, int nthreads)
{
    int err = 0;
#ifdef _OPENMP
#pragma omp parallel for schedule(dynamic, 16) num_threads(nthreads > 0 ? nthreads : omp_get_max_threads()) reduction(|:err)
#endif
    for (int64_t b = 0; b < batch; ++b)
        err |= gjo_solve(n, m, A + b * (size_t)n * n, B + b * (size_t)n * m, tol, X ? X + b * (size_t)n * m : NULL,
                         ipiv ? ipiv + b * n : NULL, logabsdet ? logabsdet + b : NULL, sign ? sign + b : NULL,
                         info ? info + b : NULL, gap ? gap + b * n : NULL);
    return err ? -1 : 0;
}

/* Only the first `nsteps` steps of O3 (no threshold stop, strategy as above);
 * returns the n x 2n working array [A^k | D^k] — for pinning individual steps
 * against the paper's Eqs. (3)-(10) / (14)-(15) on small inputs. */
int gjo_steps(int n, const double* A, int nsteps, int strategy, double* Mout)
{
    const int w = 2 * n;
    ld* M = (ld*)malloc(sizeof(ld) * (size_t)n * (size_t)w);
    if (!M && n > 0) return -1;
    for (int i = 0; i < n; ++i)
        for (int j = 0; j < n; ++j) {
            M[(size_t)i * w + j] = (ld)A[(size_t)i * n + j];
            M[(size_t)i * w + n + j] = (i == j) ? 1.0L : 0.0L;
        }
    for (int k = 0; k < nsteps && k < n; ++k) {
        int r = k;
        ld c1 = fabsl(M[(size_t)k * w + k]);
        if (strategy == 1)
            for (int i = k + 1; i < n; ++i)
                if (fabsl(M[(size_t)i * w + k]) > c1) { c1 = fabsl(M[(size_t)i * w + k]); r = i; }
        if (r != k)
            for (int j = 0; j < w; ++j) {
                ld t = M[(size_t)k * w + j]; M[(size_t)k * w + j] = M[(size_t)r * w + j]; M[(size_t)r * w + j] = t;
            }
        ld* Rk = M + (size_t)k * w;
        const ld p = Rk[k];
        for (int j = 0; j < w; ++j) Rk[j] = Rk[j] / p;
        for (int i = 0; i < n; ++i) {
            if (i == k) continue;
            ld* Ri = M + (size_t)i * w;
            const ld f = Ri[k];
            for (int j = 0; j < w; ++j) Ri[j] = Ri[j] - f * Rk[j];
        }
    }
    for (size_t t = 0; t < (size_t)n * w; ++t) Mout[t] = (double)M[t];
    free(M);
    return 0;
}

/* Residual max_{i in rows, j} |(A X)_ij - delta_ij| in long double.
 * rows == NULL means all rows.  A and X: n*n row-major. */
double gjo_residual_rows(int n, const double* A, const double* X, const int64_t* rows, int64_t nrows,
                         int nthreads)
{
    double worst = 0.0;
    const int64_t R = rows ? nrows : n;
#ifdef _OPENMP
#pragma omp parallel for schedule(dynamic, 1) num_threads(nthreads > 0 ? nthreads : omp_get_max_threads()) reduction(max:worst)
#endif
    for (int64_t t = 0; t < R; ++t) {
        const int64_t i = rows ? rows[t] : t;
        ld* acc = (ld*)calloc((size_t)n, sizeof(ld));
        for (int k = 0; k < n; ++k) {
            const ld a = (ld)A[(size_t)i * n + k];
            const double* Xk = X + (size_t)k * n;
            for (int j = 0; j < n; ++j) acc[j] += a * (ld)Xk[j];
        }
        double m = 0.0;
        for (int j = 0; j < n; ++j) {
            ld d = acc[j] - ((j == i) ? 1.0L : 0.0L);
            double e = (double)fabsl(d);
            if (e > m) m = e;
        }
        free(acc);
        if (m > worst) worst = m;
    }
    return worst;
}

/* Batched residual: out[b] = max |A_b X_b - I| (long double accumulation). */
int gjo_residual_batched(int n, int64_t batch, const double* A, const double* X, double* out, int nthreads)
{
    const size_t nn = (size_t)n * n;
#ifdef _OPENMP
#pragma omp parallel for schedule(static) num_threads(nthreads > 0 ? nthreads : omp_get_max_threads())
#endif
    for (int64_t b = 0; b < batch; ++b)
        out[b] = gjo_residual_rows(n, A + b * nn, X + b * nn, NULL, 0, 1);
    return 0;
}

int gjo_max_threads(void)
{
#ifdef _OPENMP
    return omp_get_max_threads();
#else
    return 1;
#endif
}
