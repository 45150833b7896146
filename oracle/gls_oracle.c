/*
 * gls_oracle.c -- plain, slow, obviously-correct CPU FP64 oracle for the GLS sequence
 *
 *     b_i := (X_i^T M^{-1} X_i)^{-1} X_i^T M^{-1} y,   X_i = (X_L | X_Ri),  1 <= i <= m
 *
 * (§1 eq:probDef; structure X_i = (X_L | X_Ri) PAPER.md:53-54).
 *
 * TEST INFRASTRUCTURE ONLY.  Only tests/, __graft_entry__.smoke() and bench.py's
 * cpu_baseline / --impl reference leg may load this library.  It shares no code,
 * header, table or helper with the CUDA path (paper_1210_7325_b200/), and neither
 * side includes the other.
 *
 * It follows Alg. 4 (seq-gls) with the per-problem steps of
 * Alg. 3 (black-box) written out as scalar loops -- no BLAS, no
 * blocking, no Fig. 1 partition (the hp-gwas partition is what the CUDA path does;
 * the oracle deliberately recomputes L^{-1} X_L for every problem, as Alg. 4 does):
 *
 *   1. L L^T = M                (potrf, Alg. 4 l.1)  -- oracle_cholesky
 *   2. y~ := L^{-1} y           (trsv,  Alg. 4 l.2)  -- oracle_forward
 *   3. for each X_i:
 *        X~_i := L^{-1} X_i     (trsm,  Alg. 4 l.4)  -- oracle_forward per column
 *        S_i  := X~_i^T X~_i    (syrk,  Alg. 4 l.5)  -- dot products
 *        r_i  := X~_i^T y~      (gemv,  Alg. 4 l.6)  -- dot products
 *        b_i  := S_i^{-1} r_i   (posv,  Alg. 4 l.7)  -- oracle_spd_solve (Cholesky of S,
 *                                   justified at PAPER.md:209-212)
 *
 * Readings: NotSPD for M when a pivot d_j <= 2^-52 * max_k M_kk
 * (reading A5); RankDeficient problem when a pivot of S_i satisfies
 * d_j <= 1e-10 * S_jj (original diagonal) -- reading A4; its b row is quiet NaN and
 * status 1, the sequence continues.  Comparisons are written "!(d > thr)" so a NaN
 * pivot is treated as failure.
 *
 * Storage: M, X_L, X_R column-major (element (r, c) at r + c*ld).  The oracle keeps L
 * row-major (L[i*n + k], k <= i) so that row dot products are contiguous.
 *
 * OpenMP is used only across problems (step 3) and across rows of one Cholesky column;
 * every individual sum runs in a fixed sequential order, so results do not depend on
 * the thread count.
 */
#include <math.h>
#include <stdint.h>
#include <stdlib.h>
#include <string.h>

#define ORACLE_OK 0
#define ORACLE_NOT_SPD 3

/* Step 1: L L^T = M (lower).  Crout / dot-product form:
 *   d_j   = M_jj - sum_{k<j} L_jk^2,          L_jj = sqrt(d_j)
 *   L_ij  = (M_ij - sum_{k<j} L_ik L_jk) / L_jj     for i > j
 * Returns ORACLE_NOT_SPD and *fail_pivot = j at the first pivot d_j <= 2^-52 max diag M. */
int oracle_cholesky(int64_t n, const double* M, int64_t ldm, double* L, int64_t* fail_pivot) {
  double maxdiag = 0.0;
  for (int64_t k = 0; k < n; ++k)
    if (M[k + k * ldm] > maxdiag) maxdiag = M[k + k * ldm];
  const double tol = ldexp(1.0, -52) * maxdiag;
  memset(L, 0, (size_t)n * (size_t)n * sizeof(double));
  *fail_pivot = -1;
  for (int64_t j = 0; j < n; ++j) {
    const double* Lj = L + j * n;
    double d = M[j + j * ldm];
    for (int64_t k = 0; k < j; ++k) d -= Lj[k] * Lj[k];
    if (!(d > tol)) {
      *fail_pivot = j;
      return ORACLE_NOT_SPD;
    }
    const double ljj = sqrt(d);
    L[j * n + j] = ljj;
#pragma omp parallel for schedule(static)
    for (int64_t i = j + 1; i < n; ++i) {
      const double* Li = L + i * n;
      double s = M[i + j * ldm];
      for (int64_t k = 0; k < j; ++k) s -= Li[k] * Lj[k];
      L[i * n + j] = s / ljj;
    }
  }
  return ORACLE_OK;
}

/* Forward substitution L x = b (row-major lower L):
 *   x_i = (b_i - sum_{k<i} L_ik x_k) / L_ii. */
void oracle_forward(int64_t n, const double* L, const double* b, double* x) {
  for (int64_t i = 0; i < n; ++i) {
    const double* Li = L + i * n;
    double s = b[i];
    for (int64_t k = 0; k < i; ++k) s -= Li[k] * x[k];
    x[i] = s / Li[i];
  }
}

/* Small SPD solve S b = r (p x p, column-major S, only the lower triangle read):
 * Cholesky S = G G^T with the rank rule, then G w = r and G^T b = w.
 * Returns 0 on success, 1 (RankDeficient) otherwise; b is then all quiet NaN. */
int oracle_spd_solve(int32_t p, const double* S, const double* r, double* b) {
  double G[20 * 20];
  double w[20];
  if (p < 1 || p > 20) return 1;
  for (int32_t j = 0; j < p; ++j) {
    double d = S[j + j * p];
    for (int32_t k = 0; k < j; ++k) d -= G[j * 20 + k] * G[j * 20 + k];
    if (!(d > 1e-10 * S[j + j * p])) {
      for (int32_t k = 0; k < p; ++k) b[k] = NAN;
      return 1;
    }
    const double gjj = sqrt(d);
    G[j * 20 + j] = gjj;
    for (int32_t i = j + 1; i < p; ++i) {
      double s = S[i + j * p];
      for (int32_t k = 0; k < j; ++k) s -= G[i * 20 + k] * G[j * 20 + k];
      G[i * 20 + j] = s / gjj;
    }
  }
  for (int32_t i = 0; i < p; ++i) { /* G w = r */
    double s = r[i];
    for (int32_t k = 0; k < i; ++k) s -= G[i * 20 + k] * w[k];
    w[i] = s / G[i * 20 + i];
  }
  for (int32_t i = p - 1; i >= 0; --i) { /* G^T b = w */
    double s = w[i];
    for (int32_t k = i + 1; k < p; ++k) s -= G[k * 20 + i] * b[k];
    b[i] = s / G[i * 20 + i];
  }
  return 0;
}

/* Steps 2-3 for the selected problems.  sel[t] is the problem index i (0-based); its X_Ri
 * is columns [i*pR, (i+1)*pR) of X_R (ld = ldxr) -- or, when X_R_is_selected != 0, columns
 * [t*pR, (t+1)*pR) (the caller packed only the selected problems).
 * b_out row t (p values, X_L coefficients first -- reading A3) and status[t]. */
void oracle_gls_sequence(int64_t n, int32_t pL, int32_t pR, const double* L,
                         const double* XL, const double* y, const double* XR, int64_t ldxr,
                         int32_t X_R_is_selected, int64_t nsel, const int64_t* sel,
                         double* b_out, int32_t* status) {
  const int32_t p = pL + pR;
  double* yt = (double*)malloc((size_t)n * sizeof(double));
  oracle_forward(n, L, y, yt); /* Alg. 4 l.2 */
#pragma omp parallel
  {
    double* Xt = (double*)malloc((size_t)n * (size_t)p * sizeof(double)); /* X~_i column-major */
    double S[400], r[20];
#pragma omp for schedule(dynamic, 1)
    for (int64_t t = 0; t < nsel; ++t) {
      const int64_t i = sel[t];
      const int64_t c0 = (X_R_is_selected ? t : i) * (int64_t)pR;
      /* X_i = (X_L | X_Ri); X~_i := L^{-1} X_i column by column (Alg. 4 l.4) */
      for (int32_t k = 0; k < p; ++k) {
        const double* xcol = (k < pL) ? XL + (int64_t)k * n : XR + (c0 + (k - pL)) * ldxr;
        oracle_forward(n, L, xcol, Xt + (int64_t)k * n);
      }
      /* S_i := X~_i^T X~_i,  r_i := X~_i^T y~  (Alg. 4 l.5-6) */
      for (int32_t a = 0; a < p; ++a) {
        const double* xa = Xt + (int64_t)a * n;
        for (int32_t c = 0; c < p; ++c) {
          const double* xc = Xt + (int64_t)c * n;
          double s = 0.0;
          for (int64_t q = 0; q < n; ++q) s += xa[q] * xc[q];
          S[a + c * p] = s;
        }
        double s = 0.0;
        for (int64_t q = 0; q < n; ++q) s += xa[q] * yt[q];
        r[a] = s;
      }
      /* b_i := S_i^{-1} r_i (Alg. 4 l.7) */
      status[t] = oracle_spd_solve(p, S, r, b_out + t * p);
    }
    free(Xt);
  }
  free(yt);
}
