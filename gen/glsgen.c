/*
 * glsgen.c -- seeded synthetic inputs for the GLS-sequence problem (CPU side).
 *
 * This module holds NONE of the method's arithmetic (no Cholesky, no triangular
 * solve, no normal equations).  It only draws the workload of BASELINE.json
 * `configs` (SURVEY.md §8(d) "Generators"):
 *
 *   M   = 0.5 * Z Z^T / 256 + 0.5 * I,      Z n x 256 N(0,1)            (stream 0)
 *   X_L = [1 | N(0,1) covariates | sex]     covariates stream 1, sex stream 2
 *   y   = X_L beta_L + eps,                 beta_L ~ N(0,1) (stream 3), eps ~ N(0,1) (stream 4)
 *   X_R column c: q_c = 0.05 + 0.45 u       (stream 5)
 *                 g(c, r) = [u_a < q_c] + [u_b < q_c] in {0,1,2}   (stream 6)
 *
 * Random numbers come from a counter-based Philox4x32-10 generator (Salmon et al.,
 * SC'11), key = seed, counter = (index lo, index hi, sub, stream).  The GPU-side
 * genotype generator (paper_1210_7325_b200/csrc/gen_device.cu) implements the same
 * generator independently; genotypes are integer-exact, so both sides agree bit for bit.
 *
 * Build: gcc -O2 -fopenmp -ffp-contract=off -shared -fPIC (see gen/__init__.py).
 * -ffp-contract=off matters: q_c = 0.05 + 0.45*u must round identically on CPU and GPU.
 */
#include <math.h>
#include <stdint.h>
#include <stdlib.h>
#include <string.h>

#define PHILOX_M0 0xD2511F53u
#define PHILOX_M1 0xCD9E8D57u
#define PHILOX_W0 0x9E3779B9u
#define PHILOX_W1 0xBB67AE85u

static inline void philox4x32_10(const uint32_t ctr_in[4], uint64_t seed, uint32_t out[4]) {
  uint32_t c0 = ctr_in[0], c1 = ctr_in[1], c2 = ctr_in[2], c3 = ctr_in[3];
  uint32_t k0 = (uint32_t)seed, k1 = (uint32_t)(seed >> 32);
  for (int r = 0; r < 10; ++r) {
    uint64_t p0 = (uint64_t)PHILOX_M0 * c0;
    uint64_t p1 = (uint64_t)PHILOX_M1 * c2;
    uint32_t hi0 = (uint32_t)(p0 >> 32), lo0 = (uint32_t)p0;
    uint32_t hi1 = (uint32_t)(p1 >> 32), lo1 = (uint32_t)p1;
    uint32_t n0 = hi1 ^ c1 ^ k0;
    uint32_t n1 = lo1;
    uint32_t n2 = hi0 ^ c3 ^ k1;
    uint32_t n3 = lo0;
    c0 = n0; c1 = n1; c2 = n2; c3 = n3;
    k0 += PHILOX_W0;
    k1 += PHILOX_W1;
  }
  out[0] = c0; out[1] = c1; out[2] = c2; out[3] = c3;
}

/* Raw access for tests: 4 words for (stream, index, sub). */
void glsgen_philox(uint64_t seed, uint32_t stream, uint64_t index, uint32_t sub, uint32_t out[4]) {
  uint32_t ctr[4] = {(uint32_t)index, (uint32_t)(index >> 32), sub, stream};
  philox4x32_10(ctr, seed, out);
}

static const double TWO_M32 = 2.3283064365386963e-10; /* 2^-32, exact */

static inline double unit_open(uint32_t u) { return ((double)u + 0.5) * TWO_M32; } /* exact, in (0,1) */

/* Box-Muller on the first two words of counter (index, 0, 0, stream). */
static inline double normal_at(uint64_t seed, uint32_t stream, uint64_t index) {
  uint32_t w[4];
  glsgen_philox(seed, stream, index, 0, w);
  double u1 = unit_open(w[0]), u2 = unit_open(w[1]);
  return sqrt(-2.0 * log(u1)) * cos(6.283185307179586 * u2);
}

void glsgen_normals(uint64_t seed, uint32_t stream, uint64_t start, int64_t count, double* out) {
#pragma omp parallel for schedule(static)
  for (int64_t j = 0; j < count; ++j) out[j] = normal_at(seed, stream, start + (uint64_t)j);
}

/* Allele frequency of X_R column c (stream 5). */
double glsgen_q(uint64_t seed, uint64_t col) {
  uint32_t w[4];
  glsgen_philox(seed, 5u, col, 0, w);
  double u = unit_open(w[0]);
  volatile double t = 0.45 * u; /* keep the product rounded separately from the sum */
  return 0.05 + t;
}

/* X_R columns [col0, col0+ncols) into X (column-major, leading dimension ld >= n).
 * Genotype (c, r) = [u_a < q_c] + [u_b < q_c], u from counter (c, r, stream 6). */
void glsgen_xr(uint64_t seed, int64_t n, uint64_t col0, int64_t ncols, double* X, int64_t ld) {
#pragma omp parallel for schedule(static)
  for (int64_t j = 0; j < ncols; ++j) {
    uint64_t c = col0 + (uint64_t)j;
    double q = glsgen_q(seed, c);
    double* col = X + j * ld;
    for (int64_t r = 0; r < n; ++r) {
      uint32_t w[4];
      glsgen_philox(seed, 6u, c, (uint32_t)r, w);
      col[r] = (double)((unit_open(w[0]) < q) + (unit_open(w[1]) < q));
    }
  }
}

/* M = 0.5 * Z Z^T / 256 + 0.5 I, Z (n x 256) from stream 0 with Z[r, k] = normal(index r*256+k).
 * Fixed summation order k = 0..255 for every entry, so M is bitwise independent of thread count.
 * M is written full (both triangles), column-major. */
void glsgen_M(uint64_t seed, int64_t n, double* M) {
  const int64_t K = 256;
  static const double scale = 0.001953125; /* 0.5/256 = 2^-9, exact */
  double* Zt = (double*)malloc((size_t)n * K * sizeof(double)); /* Z row-major, n x 256 */
  if (!Zt) return;
  glsgen_normals(seed, 0u, 0, n * K, Zt);
#pragma omp parallel for schedule(dynamic, 16)
  for (int64_t i = 0; i < n; ++i) {
    const double* zi = Zt + i * K;
    for (int64_t j = 0; j <= i; ++j) {
      const double* zj = Zt + j * K;
      double s = 0.0;
      for (int64_t k = 0; k < K; ++k) s += zi[k] * zj[k];
      double v = s * scale;
      if (i == j) v += 0.5;
      M[j * n + i] = v;
      M[i * n + j] = v;
    }
  }
  free(Zt);
}

/* X_L (n x pL, column-major): column 0 = 1 (intercept) when pL >= 1; if with_sex and pL >= 2
 * the last column is sex ~ Bernoulli(0.5) (stream 2: u < 2^31); every other column k is an
 * N(0,1) covariate drawn from stream 1 at index k*n + r. */
void glsgen_xl(uint64_t seed, int64_t n, int32_t pL, int32_t with_sex, double* XL) {
  for (int32_t k = 0; k < pL; ++k) {
    double* col = XL + (int64_t)k * n;
    if (k == 0) {
      for (int64_t r = 0; r < n; ++r) col[r] = 1.0;
    } else if (with_sex && pL >= 2 && k == pL - 1) {
      for (int64_t r = 0; r < n; ++r) {
        uint32_t w[4];
        glsgen_philox(seed, 2u, (uint64_t)r, 0, w);
        col[r] = (w[0] < 0x80000000u) ? 1.0 : 0.0;
      }
    } else {
      glsgen_normals(seed, 1u, (uint64_t)k * (uint64_t)n, n, col);
    }
  }
}

/* beta_L ~ N(0,1) (stream 3, index k); y = X_L beta_L + noise * eps (eps stream 4, index r).
 * Sum order k = 0..pL-1, then + eps.  noise = 0 gives the planted noise-free phenotype. */
void glsgen_y(uint64_t seed, int64_t n, int32_t pL, const double* XL, double noise,
              double* beta_out, double* y) {
  for (int32_t k = 0; k < pL; ++k) beta_out[k] = normal_at(seed, 3u, (uint64_t)k);
#pragma omp parallel for schedule(static)
  for (int64_t r = 0; r < n; ++r) {
    double s = 0.0;
    for (int32_t k = 0; k < pL; ++k) s += XL[(int64_t)k * n + r] * beta_out[k];
    if (noise != 0.0) s += noise * normal_at(seed, 4u, (uint64_t)r);
    y[r] = s;
  }
}
