// chol_inv.cu -- once-per-context factorisation: M = L L^T (potrf, Alg. 5 line 1)
// and the explicit lower-triangular inverse T = L^{-1} that the hot kernel applies blockwise
// (DESIGN.md "Design A: the blocked solve as a product with T").
//
// Recursive, all contractions on the FP64 tensor pipe through dgemm():
//   chol_inv([[A11, .], [A21, A22]]):
//     (L11, T11) = chol_inv(A11)
//     L21  = A21 T11^T                 (= A21 L11^{-T}, the panel solve)
//     A22 -= L21 L21^T                 (trailing SYRK, lower tiles only)
//     (L22, T22) = chol_inv(A22)
//     T21  = -T22 (L21 T11)            ([[L11,0],[L21,L22]]^{-1} = [[T11,0],[-T22 L21 T11, T22]])
// Leaves (n <= 64) factor and invert one diagonal block inside one CTA in a single sweep.
// NotSPD (reading A5): a pivot d_j <= 2^-52 * max_k M_kk records min(j) in st->fail.
#include <climits>
#include <cstdlib>
#include <mutex>
#include <vector>

#include "gls_internal.cuh"

namespace gls {
namespace {

constexpr int LEAF = 64;
#ifndef GLS_LEAF_THREADS
#define GLS_LEAF_THREADS 512
#endif
constexpr int LEAF_THREADS = GLS_LEAF_THREADS;
constexpr int LEAF_TY = LEAF_THREADS / 32;  // thread rows of the update phase
constexpr int LLD = LEAF + 1;

__global__ void maxdiag_kernel(int64_t n, const double* A, int64_t ld, CholStatus* st) {
  __shared__ double red[256];
  double m = 0.0;
  for (int64_t k = threadIdx.x; k < n; k += blockDim.x) m = fmax(m, A[k + k * ld]);
  red[threadIdx.x] = m;
  __syncthreads();
  for (int w = 128; w > 0; w >>= 1) {
    if (threadIdx.x < w) red[threadIdx.x] = fmax(red[threadIdx.x], red[threadIdx.x + w]);
    __syncthreads();
  }
  if (threadIdx.x == 0) {
    st->tol = ldexp(1.0, -52) * red[0];
    st->fail = ULLONG_MAX;
  }
}

// One CTA: Cholesky of the nb x nb diagonal block at A (lower read) and, in the same sweep, its
// inverse by forward elimination on [L | I] (leaf_sweep2: after columns j, j+1 of L are final,
// rows j, j+1 of T are scaled and every later row gets the rank-2 update, so that on exit L T = I).
// Writes L into A's lower triangle and T = L^{-1} (zeros above the diagonal).
// The sweep of a leaf on shared-memory copies: L (lower nb x nb, zeros above) becomes its Cholesky
// factor and Ti (= I on entry) its inverse, by forward elimination on [L | I] two columns at a time
// (one barrier per pair; every thread of the block calls it, and it ends with a barrier).  Measured
// against the one-column sweep: create 40.5 -> 38.1 ms at n = 1e4, 2.70 -> 2.29 ms at n = 1500.
// For the pair (j, j+1):
//   rinv0 = 1/sqrt(d_j), a = L[j+1][j] rinv0, d_{j+1} -= a^2, rinv1 = 1/sqrt(d_{j+1});
//   c0[x] = L[x][j] rinv0,  c1[x] = (L[x][j+1] - c0[x] a) rinv1             (the two new columns)
//   L[i][k] -= c0[i] c0[k] + c1[i] c1[k]                  (i >= k >= j+2: the trailing triangle)
//   t0 = T[j] rinv0,  t1 = (T[j+1] - a t0) rinv1,  T[i] -= c0[i] t0 + c1[i] t1   (i >= j+2)
// Readers form c0, c1, t0, t1 on the fly; the pair's columns and rows are written back in the next
// step.  An odd last column takes a one-column step.
__device__ void leaf_sweep2(int nb, double* L, double* Ti, double tol, int64_t goff, CholStatus* st,
                            int* failed) {
  const int tid = threadIdx.x;
  const int ty = tid >> 5, tx = tid & 31;
  constexpr int RY = LEAF / LEAF_TY;
  constexpr int R = LEAF / 32;
  const double qnan = __longlong_as_double(0x7ff8000000000000LL);
  // previous pair (write-back state)
  int jp = -1, np = 0;  // first column, 1 or 2 columns
  double p_r0 = 0.0, p_r1 = 0.0, p_a = 0.0, p_l0 = 0.0, p_l1 = 0.0;
  for (int j = 0; j < nb; j += 2) {
    const bool two = j + 1 < nb;
    const double d0 = L[j * LLD + j];
    const double lj1 = two ? L[(j + 1) * LLD + j] : 0.0;
    const double dd1 = two ? L[(j + 1) * LLD + j + 1] : 0.0;
    double r0 = 0.0, r1 = 0.0, a = 0.0, l0 = 0.0, l1 = 0.0;
    bool bad0 = false, bad1 = false;
    if ((tid & 31) == 0) {
      const bool f = *(volatile int*)failed;
      bad0 = !(d0 > tol) || f;
      r0 = bad0 ? qnan : rsqrt(d0);
      l0 = d0 * r0;
      if (two) {
        a = lj1 * r0;
        const double d1 = dd1 - a * a;
        bad1 = bad0 || !(d1 > tol);
        r1 = bad1 ? qnan : rsqrt(d1);
        l1 = d1 * r1;
      }
    }
    r0 = __shfl_sync(0xffffffffu, r0, 0);
    r1 = __shfl_sync(0xffffffffu, r1, 0);
    a = __shfl_sync(0xffffffffu, a, 0);
    l0 = __shfl_sync(0xffffffffu, l0, 0);
    l1 = __shfl_sync(0xffffffffu, l1, 0);
    if (tid == 0 && !*failed && (bad0 || bad1)) {
      atomicMin(&st->fail, (unsigned long long)(goff + j + (bad0 ? 0 : 1)));
      *failed = 1;  // read by every thread after this step's barrier
    }
    // deferred write-back of the previous pair: its columns (scaled) and T rows
    if (jp >= 0) {
      const int rows = nb - jp;  // rows jp .. nb-1
      for (int x = tid; x < rows + jp + 2; x += blockDim.x) {
        if (x < rows) {
          const int r = jp + x;
          if (r == jp) {
            L[jp * LLD + jp] = p_l0;
          } else {
            const double c0 = L[r * LLD + jp] * p_r0;
            L[r * LLD + jp] = c0;
            if (np == 2) {
              if (r == jp + 1) L[r * LLD + r] = p_l1;
              else L[r * LLD + jp + 1] = (L[r * LLD + jp + 1] - c0 * p_a) * p_r1;
            }
          }
        } else {
          const int k2 = x - rows;  // T columns 0 .. jp+1
          if (k2 <= jp + np - 1) {
            const double t0 = Ti[jp * LLD + k2] * p_r0;
            Ti[jp * LLD + k2] = t0;
            if (np == 2) Ti[(jp + 1) * LLD + k2] = (Ti[(jp + 1) * LLD + k2] - p_a * t0) * p_r1;
          }
        }
      }
    }
    // rank-2 (or, for a last single column, rank-1) update of the trailing triangle and of the T rows
    const int jn = j + (two ? 2 : 1);  // first row / column not in the pair
#pragma unroll
    for (int q = 0; q < RY; ++q) {
      const int i = jn + ty + LEAF_TY * q;
      if (i < nb) {
        const double ci0 = L[i * LLD + j] * r0;
        const double ci1 = two ? (L[i * LLD + j + 1] - ci0 * a) * r1 : 0.0;
        double ck0[R], ck1[R], li[R], t0[R], t1[R], ti[R];
#pragma unroll
        for (int c = 0; c < R; ++c) {
          const int k = jn + tx + 32 * c;
          const bool v = k <= i;
          ck0[c] = v ? L[k * LLD + j] * r0 : 0.0;
          ck1[c] = (v && two) ? (L[k * LLD + j + 1] - ck0[c] * a) * r1 : 0.0;
          li[c] = v ? L[i * LLD + k] : 0.0;
          const int k2 = tx + 32 * c;
          const bool v2 = k2 < jn;
          t0[c] = v2 ? Ti[j * LLD + k2] * r0 : 0.0;
          t1[c] = (v2 && two) ? (Ti[(j + 1) * LLD + k2] - a * t0[c]) * r1 : 0.0;
          ti[c] = v2 ? Ti[i * LLD + k2] : 0.0;
        }
#pragma unroll
        for (int c = 0; c < R; ++c) {
          const int k = jn + tx + 32 * c;
          if (k <= i) L[i * LLD + k] = li[c] - ci0 * ck0[c] - ci1 * ck1[c];
          const int k2 = tx + 32 * c;
          if (k2 < jn) Ti[i * LLD + k2] = ti[c] - ci0 * t0[c] - ci1 * t1[c];
        }
      }
    }
    jp = j;
    np = two ? 2 : 1;
    p_r0 = r0;
    p_r1 = r1;
    p_a = a;
    p_l0 = l0;
    p_l1 = l1;
    __syncthreads();
  }
  if (jp >= 0) {  // write-back of the last pair
    const int rows = nb - jp;
    for (int x = tid; x < rows + jp + 2; x += blockDim.x) {
      if (x < rows) {
        const int r = jp + x;
        if (r == jp) {
          L[jp * LLD + jp] = p_l0;
        } else {
          const double c0 = L[r * LLD + jp] * p_r0;
          L[r * LLD + jp] = c0;
          if (np == 2) {
            if (r == jp + 1) L[r * LLD + r] = p_l1;
            else L[r * LLD + jp + 1] = (L[r * LLD + jp + 1] - c0 * p_a) * p_r1;
          }
        }
      } else {
        const int k2 = x - rows;
        if (k2 <= jp + np - 1) {
          const double t0 = Ti[jp * LLD + k2] * p_r0;
          Ti[jp * LLD + k2] = t0;
          if (np == 2) Ti[(jp + 1) * LLD + k2] = (Ti[(jp + 1) * LLD + k2] - p_a * t0) * p_r1;
        }
      }
    }
    __syncthreads();
  }
}

// One CTA: Cholesky of the nb x nb diagonal block at A (lower read) and, in the same sweep, its
// inverse by forward elimination on [L | I] (leaf_sweep2: after columns j, j+1 of L are final,
// rows j, j+1 of T are scaled and every later row gets the rank-2 update, so that on exit L T = I).
// Writes L into A's lower triangle and T = L^{-1} (zeros above the diagonal).
__global__ void __launch_bounds__(LEAF_THREADS) chol_inv_leaf(int nb, double* A, double* T, int64_t ld,
                                                     int64_t goff, CholStatus* st) {
  extern __shared__ double leaf_smem[];
  double* L = leaf_smem;
  double* Ti = leaf_smem + LEAF * LLD;
  __shared__ int failed;
  const int tid = threadIdx.x;
  for (int idx = tid; idx < nb * nb; idx += blockDim.x) {
    const int i = idx % nb, j = idx / nb;
    L[i * LLD + j] = (i >= j) ? A[i + (int64_t)j * ld] : 0.0;
    Ti[i * LLD + j] = (i == j) ? 1.0 : 0.0;
  }
  if (tid == 0) failed = 0;
  __syncthreads();
  leaf_sweep2(nb, L, Ti, st->tol, goff, st, &failed);
  for (int idx = tid; idx < nb * nb; idx += blockDim.x) {
    const int i = idx % nb, j = idx / nb;
    if (i >= j) A[i + (int64_t)j * ld] = L[i * LLD + j];
    T[i + (int64_t)j * ld] = (i >= j) ? Ti[i * LLD + j] : 0.0;
  }
}

// 64 x 64 product on shared-memory blocks (row stride LLD), 512 threads, 8 outputs per thread
// (rows ty + 16 a, columns tx + 32 b): out[i][k] = sum_m A(i, m) B(m, k) with the operand accessors
// given; OP receives (i, k, value).
template <class FA, class FB, class OP>
__device__ __forceinline__ void smem_gemm64(FA fa, FB fb, OP op) {
  const int ty = threadIdx.x >> 5, tx = threadIdx.x & 31;
  double acc[4][2] = {{0.0, 0.0}, {0.0, 0.0}, {0.0, 0.0}, {0.0, 0.0}};
#pragma unroll 4
  for (int m = 0; m < LEAF; ++m) {
    double a[4], bv[2];
#pragma unroll
    for (int u = 0; u < 4; ++u) a[u] = fa(ty + 16 * u, m);
#pragma unroll
    for (int v = 0; v < 2; ++v) bv[v] = fb(m, tx + 32 * v);
#pragma unroll
    for (int u = 0; u < 4; ++u)
#pragma unroll
      for (int v = 0; v < 2; ++v) acc[u][v] = fma(a[u], bv[v], acc[u][v]);
  }
#pragma unroll
  for (int u = 0; u < 4; ++u)
#pragma unroll
    for (int v = 0; v < 2; ++v) op(ty + 16 * u, tx + 32 * v, acc[u][v]);
}

// A node of n = 64 + h2 (0 < h2 <= 64) rows in one CTA: the recursion's two leaves and its four
// small products (L21 = A21 T11^T, A22 -= L21 L21^T, Y = L21 T11, T21 = -T22 Y) on shared-memory
// blocks -- one launch instead of two leaves, three main-stream GEMMs and an aux-stream GEMM.
__global__ void __launch_bounds__(LEAF_THREADS) chol_inv_node128(int n, double* A, double* T, int64_t ld,
                                                        int64_t goff, CholStatus* st) {
  extern __shared__ double leaf_smem[];
  constexpr int B = LEAF * LLD;
  double* L1 = leaf_smem;       // A11 -> L11
  double* T1 = L1 + B;          // I -> T11
  double* P = T1 + B;           // A21, later Y
  double* Q = P + B;            // L21
  double* L2 = Q + B;           // A22 -> L22
  double* T2 = L2 + B;          // I -> T22
  __shared__ int failed;
  const int tid = threadIdx.x;
  const int h2 = n - LEAF;
  double* A21 = A + LEAF;
  double* A22 = A + LEAF + (int64_t)LEAF * ld;
  for (int idx = tid; idx < LEAF * LEAF; idx += blockDim.x) {
    const int i = idx % LEAF, j = idx / LEAF;
    L1[i * LLD + j] = (i >= j) ? A[i + (int64_t)j * ld] : 0.0;
    T1[i * LLD + j] = (i == j) ? 1.0 : 0.0;
    P[i * LLD + j] = (i < h2) ? A21[i + (int64_t)j * ld] : 0.0;
    L2[i * LLD + j] = (i < h2 && j <= i) ? A22[i + (int64_t)j * ld] : 0.0;
    T2[i * LLD + j] = (i == j && i < h2) ? 1.0 : 0.0;
  }
  if (tid == 0) failed = 0;
  __syncthreads();
  const double tol = st->tol;
  leaf_sweep2(LEAF, L1, T1, tol, goff, st, &failed);
  // L21 = A21 T11^T  (T11 is zero above its diagonal)
  smem_gemm64([&](int i, int m) { return P[i * LLD + m]; }, [&](int m, int k) { return T1[k * LLD + m]; },
              [&](int i, int k, double v) { Q[i * LLD + k] = v; });
  __syncthreads();
  // A22 -= L21 L21^T (lower triangle)
  smem_gemm64([&](int i, int m) { return Q[i * LLD + m]; }, [&](int m, int k) { return Q[k * LLD + m]; },
              [&](int i, int k, double v) {
                if (k <= i) L2[i * LLD + k] -= v;
              });
  __syncthreads();
  leaf_sweep2(h2, L2, T2, tol, goff + LEAF, st, &failed);
  // Y = L21 T11 (into P: A21 is no longer needed)
  smem_gemm64([&](int i, int m) { return Q[i * LLD + m]; }, [&](int m, int k) { return T1[m * LLD + k]; },
              [&](int i, int k, double v) { P[i * LLD + k] = v; });
  __syncthreads();
  // T21 = -T22 Y, straight to global memory
  smem_gemm64([&](int i, int m) { return T2[i * LLD + m]; }, [&](int m, int k) { return P[m * LLD + k]; },
              [&](int i, int k, double v) {
                if (i < h2) T[LEAF + i + (int64_t)k * ld] = -v;
              });
  for (int idx = tid; idx < LEAF * LEAF; idx += blockDim.x) {
    const int i = idx % LEAF, j = idx / LEAF;
    if (i >= j) A[i + (int64_t)j * ld] = L1[i * LLD + j];
    T[i + (int64_t)j * ld] = (i >= j) ? T1[i * LLD + j] : 0.0;
    if (i < h2) {
      A21[i + (int64_t)j * ld] = Q[i * LLD + j];
      if (j < h2) {
        if (i >= j) A22[i + (int64_t)j * ld] = L2[i * LLD + j];
        T[LEAF + i + (int64_t)(LEAF + j) * ld] = (i >= j) ? T2[i * LLD + j] : 0.0;
      }
    }
  }
}

// ------------------------------------------------------------------------------------------------
// Blocked leaf of up to 128 rows on the FP64 tensor pipe (round 2).  The column sweeps above are
// bound by shared-memory traffic (every pair step re-reads the whole trailing triangle and T block:
// ~1.7 us per pair, 97 us for a 128-row node).  Here the block is factored 16 columns at a time,
// right-looking (the same recursion as chol_inv_rec, unrolled at 16-row granularity):
//   step k:  (L_kk, T_kk) = chol16(A_kk)                      one warp, registers + shuffles
//            L_ik = A_ik T_kk^T                (i > k)          DMMA, 8-row strips
//            A_ij -= L_ik L_jk^T               (i >= j > k)     DMMA, 16 x 16 blocks
//            T_kj = -T_kk sum_{l=j}^{k-1} L_kl T_lj  (j < k)    DMMA, 16 x 8 strips (row block k of
//                                                               T = L^{-1}, from [[L11,0],[L21,L22]]^-1)
// Shared memory holds the block column-major (Mat(r, c) = S[c LD + r], LD = 132 = 4 mod 16 so both the
// m8n8k4 row- and column-fragment patterns are conflict-free per half-warp); L fills the lower
// triangle, the off-diagonal blocks of T are kept transposed in the strict upper blocks
// (Mat(c, r) = T(r, c)), the diagonal blocks T_kk in Td.  A ragged block (nb % 16 != 0) is padded with
// the identity, whose pivots are 1 and never fail the NotSPD test.
// GLS_LEAF_PROF (diagnostics, tools/leaf_probe): clock64 per phase of chol_inv_leaf128, summed by thread 0
// over launches into g_leaf_prof[0: load, 1: diag16, 2: panel, 3: trailing + T rows, 4: write back].
#ifdef GLS_LEAF_PROF
__device__ unsigned long long g_leaf_prof[8];
#define LEAF_PROF_START() long long _lp_t = clock64()
#define LEAF_PROF(q)                                      \
  do {                                                    \
    if (threadIdx.x == 0) {                               \
      const long long _lp_n = clock64();                  \
      atomicAdd(&g_leaf_prof[q], (unsigned long long)(_lp_n - _lp_t)); \
      _lp_t = _lp_n;                                      \
    }                                                     \
  } while (0)
#else
#define LEAF_PROF_START()
#define LEAF_PROF(q)
#endif

namespace blk {
constexpr int NB = 128, B = 16, NBK = NB / B, LD = 132, TLD = 20, THREADS = 256, NW = THREADS / 32;
constexpr size_t SMEM = (size_t)(NB * LD + NBK * B * TLD + NW * B * TLD) * sizeof(double);
}  // namespace blk

__device__ __forceinline__ void dmma884(double (&c)[2], double a, double b) {
  asm volatile("mma.sync.aligned.m8n8k4.row.col.f64.f64.f64.f64 {%0,%1}, {%2}, {%3}, {%0,%1};\n"
               : "+d"(c[0]), "+d"(c[1])
               : "d"(a), "d"(b));
}

// chol16 + inverse of one 16 x 16 diagonal block by one warp (the critical path of the leaf).
// Cholesky: lanes 0-15 hold row i = lane of the block (R[c], c <= i); column j: pivot d = L[j][j]
// (lane j, shuffled), r = 1/sqrt(d), c_i = L[i][j] r (i > j) broadcast through shared memory (double
// buffered, one __syncwarp per column), L[i][k] -= c_i c_k (j < k <= i).  Inverse: lane c solves
// L t = e_c by right-looking forward substitution, t_i = (delta_ic + s_i) / L_ii, s_i' -= L[i'][i] t_i.
// Writes L (zeros above the diagonal) into D and T = L^{-1} into Tk.  cb: 80 doubles of scratch.
// (A first version that also swept T = [L | I] with shuffles took 18.8k cycles per block.)
__device__ __forceinline__ void diag16(double* D, double* Tk, double* cb, double tol, int64_t gpiv,
                                       CholStatus* st, int* failed) {
  using namespace blk;
  const unsigned FULL = 0xffffffffu;
  const int lane = threadIdx.x & 31, i = lane & 15;
  const bool lo = lane < 16;
  const double qnan = __longlong_as_double(0x7ff8000000000000LL);
#ifdef GLS_LEAF_PROF
  long long _d0 = clock64();
#endif
  double R[16];
#pragma unroll
  for (int c = 0; c < 16; ++c) R[c] = (lo && c <= i) ? D[c * LD + i] : 0.0;
  const bool fl0 = *(volatile int*)failed;
  bool fl = fl0;
  int jfail = 16;  // first failing pivot of this block (no branch in the sweep)
  double* rinv = cb + 32;
  // the pivot chain runs ahead of the shared-memory update: lane j+1 forms its updated diagonal
  // L[j+1][j+1] - c_{j+1}^2 (the same operation the update below applies) right after c is known
  // (and its rsqrt, the longest link, is issued before this column's shared-memory round trip)
  double dn = __shfl_sync(FULL, R[0], 0);
  bool badn = fl || !(dn > tol);
  double rn = badn ? qnan : rsqrt(dn);
#pragma unroll
  for (int j = 0; j < 16; ++j) {
    const double d = dn, r = rn;
    const bool bad = badn;
    jfail = (bad && !fl) ? j : jfail;
    fl = bad;
    const double ci = R[j] * r;
    if (j < 15) {
      dn = __shfl_sync(FULL, R[j + 1] - ci * ci, j + 1);
      badn = bad || !(dn > tol);
      rn = badn ? qnan : rsqrt(dn);
    }
    double* col = cb + 16 * (j & 1);
    if (lo && i > j) col[i] = ci;
    if (lane == j) {
      R[j] = d * r;
      rinv[j] = r;
    }
    __syncwarp();
#pragma unroll
    for (int k = 1; k < 16; ++k) {
      if (k > j) {
        const double ck = col[k];
        if (lo && i >= k) R[k] -= ci * ck;
      }
    }
    if (lo && i > j) R[j] = ci;
  }
#pragma unroll
  for (int c = 0; c < 16; ++c)
    if (lo) D[c * LD + i] = (c <= i) ? R[c] : 0.0;
  if (lane == 0 && !fl0 && jfail < 16) {
    atomicMin(&st->fail, (unsigned long long)(gpiv + jfail));
    *(volatile int*)failed = 1;
  }
  __syncwarp();
#ifdef GLS_LEAF_PROF
  long long _d1 = clock64();
  if (threadIdx.x == 0) atomicAdd(&g_leaf_prof[5], (unsigned long long)(_d1 - _d0));
#endif
  // T = L^{-1}: lane c < 16 forms column c (t_i = 0 for i < c falls out of the recursion)
  double sacc[16];
#pragma unroll
  for (int q = 0; q < 16; ++q) sacc[q] = 0.0;
#pragma unroll
  for (int q = 0; q < 16; ++q) {
    const double tq = ((q == i) ? 1.0 + sacc[q] : sacc[q]) * rinv[q];
    sacc[q] = tq;  // sacc[q] now holds t_q
#pragma unroll
    for (int q2 = q + 1; q2 < 16; ++q2) sacc[q2] -= D[q * LD + q2] * tq;
  }
  if (lo) {
#pragma unroll
    for (int q = 0; q < 16; ++q) Tk[i * TLD + q] = sacc[q];
  }
#ifdef GLS_LEAF_PROF
  __syncwarp();
  if (threadIdx.x == 0) atomicAdd(&g_leaf_prof[6], (unsigned long long)(clock64() - _d1));
#endif
}

// L_rows = A_rows T_kk^T for one 8-row strip (both 8-column tiles), in place.
__device__ __forceinline__ void panel_strip(double* S, const double* Tk, int k0, int r0) {
  using namespace blk;
  const int lane = threadIdx.x & 31, g = lane >> 2, t = lane & 3;
  double a[4];
#pragma unroll
  for (int kk = 0; kk < 4; ++kk) a[kk] = S[(k0 + 4 * kk + t) * LD + r0 + g];
  double c[2][2] = {{0.0, 0.0}, {0.0, 0.0}};
#pragma unroll
  for (int kk = 0; kk < 4; ++kk)
#pragma unroll
    for (int ct = 0; ct < 2; ++ct) dmma884(c[ct], a[kk], Tk[(4 * kk + t) * TLD + 8 * ct + g]);
#pragma unroll
  for (int ct = 0; ct < 2; ++ct)
#pragma unroll
    for (int e = 0; e < 2; ++e) S[(k0 + 8 * ct + 2 * t + e) * LD + r0 + g] = c[ct][e];
}

// Mat[bi.., bj..] -= L[bi.., k0..] L[bj.., k0..]^T for one 16 x 16 block (lower tiles only if bi == bj).
__device__ __forceinline__ void update_block(double* S, int k0, int bi, int bj) {
  using namespace blk;
  const int lane = threadIdx.x & 31, g = lane >> 2, t = lane & 3;
  double na[2][4], b[2][4];
#pragma unroll
  for (int h = 0; h < 2; ++h)
#pragma unroll
    for (int kk = 0; kk < 4; ++kk) {
      na[h][kk] = -S[(k0 + 4 * kk + t) * LD + bi + 8 * h + g];
      b[h][kk] = S[(k0 + 4 * kk + t) * LD + bj + 8 * h + g];
    }
  double c[2][2][2];
#pragma unroll
  for (int ra = 0; ra < 2; ++ra)
#pragma unroll
    for (int cb = 0; cb < 2; ++cb)
#pragma unroll
      for (int e = 0; e < 2; ++e) c[ra][cb][e] = S[(bj + 8 * cb + 2 * t + e) * LD + bi + 8 * ra + g];
  // k outermost: the three or four tile chains interleave
#pragma unroll
  for (int kk = 0; kk < 4; ++kk)
#pragma unroll
    for (int ra = 0; ra < 2; ++ra)
#pragma unroll
      for (int cb = 0; cb < 2; ++cb)
        if (!(bi == bj && cb > ra)) dmma884(c[ra][cb], na[ra][kk], b[cb][kk]);
#pragma unroll
  for (int ra = 0; ra < 2; ++ra)
#pragma unroll
    for (int cb = 0; cb < 2; ++cb)
      if (!(bi == bj && cb > ra))
#pragma unroll
        for (int e = 0; e < 2; ++e) S[(bj + 8 * cb + 2 * t + e) * LD + bi + 8 * ra + g] = c[ra][cb][e];
}

// Columns [n0, n0 + 8) of the off-diagonal block T_kj (j < k) of T = L^{-1}:
//   W = sum_{l=j}^{k-1} L_kl T_lj,  T_kj = -T_kk W   (stored transposed at Mat(j0 + n0 + col, k0 + row)).
__device__ __forceinline__ void trow_strip(double* S, const double* Td, double* W, int k, int j, int n0) {
  using namespace blk;
  const int lane = threadIdx.x & 31, g = lane >> 2, t = lane & 3;
  const int k0 = B * k, j0 = B * j;
  const double* Tk = Td + k * B * TLD;
  double w[2][2] = {{0.0, 0.0}, {0.0, 0.0}};
  {
    const double* Tj = Td + j * B * TLD;
#pragma unroll
    for (int kk = 0; kk < 4; ++kk) {
      const double bv = Tj[(n0 + g) * TLD + 4 * kk + t];
#pragma unroll
      for (int ra = 0; ra < 2; ++ra) dmma884(w[ra], S[(j0 + 4 * kk + t) * LD + k0 + 8 * ra + g], bv);
    }
  }
  for (int l = j + 1; l < k; ++l) {
    const int l0 = B * l;
#pragma unroll
    for (int kk = 0; kk < 4; ++kk) {
      const double bv = S[(l0 + 4 * kk + t) * LD + j0 + n0 + g];
#pragma unroll
      for (int ra = 0; ra < 2; ++ra) dmma884(w[ra], S[(l0 + 4 * kk + t) * LD + k0 + 8 * ra + g], bv);
    }
  }
#pragma unroll
  for (int ra = 0; ra < 2; ++ra)
#pragma unroll
    for (int e = 0; e < 2; ++e) W[(2 * t + e) * TLD + 8 * ra + g] = w[ra][e];
  __syncwarp();
  double c[2][2] = {{0.0, 0.0}, {0.0, 0.0}};
#pragma unroll
  for (int kk = 0; kk < 4; ++kk) {
    const double bv = W[g * TLD + 4 * kk + t];
#pragma unroll
    for (int ra = 0; ra < 2; ++ra) dmma884(c[ra], -Tk[(4 * kk + t) * TLD + 8 * ra + g], bv);
  }
#pragma unroll
  for (int ra = 0; ra < 2; ++ra)
#pragma unroll
    for (int e = 0; e < 2; ++e) S[(k0 + 8 * ra + g) * LD + j0 + n0 + 2 * t + e] = c[ra][e];
  __syncwarp();
}

// Schedule (look-ahead): warp 0 carries the critical path -- the panel strips of block row k+1, the
// update of the next diagonal block and chol16 of it -- while warps 1-7 do the rest of the panel, the
// trailing update and row block k of T.  Two block-wide barriers per step.
__global__ void __launch_bounds__(blk::THREADS) chol_inv_leaf128(int nb, double* A, double* T, int64_t ld,
                                                                int64_t goff, CholStatus* st) {
  using namespace blk;
  extern __shared__ double leaf_smem[];
  double* S = leaf_smem;                 // Mat(r, c) = S[c LD + r]
  double* Td = S + NB * LD;              // T_kk(r, c) = Td[k B TLD + c TLD + r]
  double* Wsc = Td + NBK * B * TLD;      // per-warp 16 x 8 scratch (column-major, TLD); warp 0: chol16's
  __shared__ int failed;
  const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
  const int nbk = (nb + B - 1) / B, np = nbk * B;
  LEAF_PROF_START();
  // every element's load in flight at once (cp.async; 16-byte pieces when A allows)
  const bool vec = ((ld & 1) == 0) && ((((uintptr_t)A) | ((uintptr_t)T)) & 15) == 0;
  for (int c = warp; c < np; c += NW) {
    for (int r = 2 * lane; r < np; r += 64) {
      const uint32_t d = (uint32_t)__cvta_generic_to_shared(S + c * LD + r);
      if (vec && r >= c && r + 1 < nb) {
        asm volatile("cp.async.cg.shared.global [%0], [%1], 16;\n" ::"r"(d), "l"(A + r + (int64_t)c * ld) : "memory");
      } else {
#pragma unroll
        for (int e = 0; e < 2; ++e) {
          const int re = r + e;
          if (re >= c && re < nb) {
            asm volatile("cp.async.ca.shared.global [%0], [%1], 8;\n" ::"r"(d + 8 * e), "l"(A + re + (int64_t)c * ld)
                         : "memory");
          } else {
            S[c * LD + re] = (re == c) ? 1.0 : 0.0;
          }
        }
      }
    }
  }
  asm volatile("cp.async.commit_group;\n" ::: "memory");
  if (tid == 0) failed = 0;
  asm volatile("cp.async.wait_group 0;\n" ::: "memory");
  __syncthreads();
  LEAF_PROF(0);
  const double tol = st->tol;
  double* W = Wsc + warp * B * TLD;
  if (warp == 0) diag16(S, Td, W, tol, goff, st, &failed);
  __syncthreads();
  LEAF_PROF(1);
  for (int k = 0; k < nbk; ++k) {
    const int k0 = k * B;
    const double* Tk = Td + k * B * TLD;
    // panel of step k: warp 0 the two strips of block row k+1, warps 1-7 the rest
    const int nstrip = 2 * (nbk - 1 - k);
    if (warp == 0) {
      for (int u = 0; u < 2 && u < nstrip; ++u) panel_strip(S, Tk, k0, k0 + B + 8 * u);
    } else {
      for (int u = 2 + warp - 1; u < nstrip; u += NW - 1) panel_strip(S, Tk, k0, k0 + B + 8 * u);
    }
    __syncthreads();
    LEAF_PROF(2);
    if (warp == 0) {
      if (k + 1 < nbk) {
        update_block(S, k0, k0 + B, k0 + B);
        __syncwarp();
        diag16(S + (k0 + B) * LD + k0 + B, Td + (k + 1) * B * TLD, W, tol, goff + k0 + B, st, &failed);
      }
    } else {
      // trailing update except the next diagonal block, then row block k of T
      const int nt = nbk - 1 - k, nupd = nt * (nt + 1) / 2;
      const int u0 = nupd > 0 ? 1 : 0;  // unit 0 is the next diagonal block (warp 0's) when there is one
      for (int u = u0 + warp - 1; u < nupd + 2 * k; u += NW - 1) {
        if (u < nupd) {
          int i = 0, q = u;  // u -> (i, q), 0 <= q <= i < nt, row-major over the lower triangle
          while (q > i) q -= ++i;
          update_block(S, k0, k0 + B + B * i, k0 + B + B * q);
        } else {
          const int v = u - nupd;
          trow_strip(S, Td, W, k, v >> 1, 8 * (v & 1));
        }
      }
    }
    __syncthreads();
    LEAF_PROF(3);
  }
  // write back L (lower triangle of A) and T (zeros above the diagonal): a warp per column
  for (int c = warp; c < nb; c += NW) {
    const int bc = c / B;
    for (int r = 2 * lane; r < nb; r += 64) {
      double lv[2], tv[2];
#pragma unroll
      for (int e = 0; e < 2; ++e) {
        const int re = r + e, br = re / B;
        lv[e] = S[c * LD + re];
        tv[e] = 0.0;
        if (br == bc) tv[e] = Td[br * B * TLD + (c - B * bc) * TLD + (re - B * br)];
        else if (br > bc) tv[e] = S[re * LD + c];
      }
      double* pa = A + r + (int64_t)c * ld;
      double* pt = T + r + (int64_t)c * ld;
      if (vec && r + 1 < nb) {
        if (r >= c) *(double2*)pa = make_double2(lv[0], lv[1]);
        else if (r + 1 == c) pa[1] = lv[1];
        *(double2*)pt = make_double2(tv[0], tv[1]);
      } else {
#pragma unroll
        for (int e = 0; e < 2; ++e) {
          if (r + e < nb) {
            if (r + e >= c) pa[e] = lv[e];
            pt[e] = tv[e];
          }
        }
      }
    }
  }
  __syncthreads();
  LEAF_PROF(4);
}

// Streams of the recursion: the main stream s (the context's, high priority) carries the critical
// path; at each depth a low-priority "side" stream takes the part of the trailing update the next
// leaf does not need yet (look-ahead) and a high-priority "aux" stream the Y = L21 T11 product.  Each stream has
// its own split-K workspace.
constexpr int kMaxDepth = 24;
constexpr int64_t kLookaheadMin = 1024;  // smallest trailing node split for look-ahead
constexpr int kFreeSms = 16;             // SMs the off-critical-path GEMMs leave free
constexpr int kFreeSmsY = 48;            // ... the aux-stream Y products
struct RecCtx {
  cudaStream_t s;
  cudaStream_t side[kMaxDepth], aux[kMaxDepth];
  double* ws_main;
  double* ws_side[kMaxDepth];
  double* ws_aux[kMaxDepth];
  std::vector<cudaEvent_t>* events;
  CholStatus* st;
  int64_t* lc;
  int off_ctas;  // grid cap of the off-critical-path GEMMs (look-ahead and Y; 0: none)
  int off_side, off_aux;  // per stream kind (A/B: GLS_CAP_SIDE / GLS_CAP_AUX, SMs)
  const ColsReady* arriving;  // nullable: A's columns still being uploaded
};

// stream st may touch columns [0, c) of A only after their upload chunks have landed
void wait_cols(const RecCtx& rc, cudaStream_t st, int64_t c) {
  if (!rc.arriving || c <= 0) return;
  int64_t k = (c - 1) / rc.arriving->cols;
  if (k >= rc.arriving->nchunks) k = rc.arriving->nchunks - 1;
  cudaStreamWaitEvent(st, rc.arriving->ready[k], 0);
}

// GLS_TRACE_CHOL=1 (diagnostics): timing events on the main stream after every step, printed per
// (depth, step) at the end of chol_inv.
struct Mark {
  cudaEvent_t e;
  int depth;
  const char* what;
};
std::vector<Mark>* g_marks = nullptr;
void mark(cudaStream_t s, int depth, const char* what) {
  if (!g_marks) return;
  cudaEvent_t e;
  cudaEventCreate(&e);
  cudaEventRecord(e, s);
  g_marks->push_back({e, depth, what});
}

// Ordering events come from a process-wide pool per device (a create records ~300; creating and
// destroying them every time costs driver calls on the create's host path).  Every wait on an event is
// enqueued within the create that recorded it, so handing it to the next create is safe.
std::mutex g_ev_mu;
std::vector<cudaEvent_t> g_ev_pool[64];
cudaEvent_t new_event(RecCtx& rc) {
  cudaEvent_t e = nullptr;
  int dev = 0;
  cudaGetDevice(&dev);
  if (dev < 0 || dev >= 64) dev = 0;
  {
    std::lock_guard<std::mutex> lk(g_ev_mu);
    if (!g_ev_pool[dev].empty()) {
      e = g_ev_pool[dev].back();
      g_ev_pool[dev].pop_back();
    }
  }
  if (!e) cudaEventCreateWithFlags(&e, cudaEventDisableTiming);
  rc.events->push_back(e);
  return e;
}
void return_events(std::vector<cudaEvent_t>& events) {
  int dev = 0;
  cudaGetDevice(&dev);
  if (dev < 0 || dev >= 64) dev = 0;
  std::lock_guard<std::mutex> lk(g_ev_mu);
  for (cudaEvent_t e : events) g_ev_pool[dev].push_back(e);
  events.clear();
}
cudaEvent_t record(RecCtx& rc, cudaStream_t st) {
  cudaEvent_t e = new_event(rc);
  cudaEventRecord(e, st);
  return e;
}

// Leaf size of the recursion: 128 (chol_inv_leaf128, the blocked DMMA leaf; default) or 64 (the
// column-sweep leaves and 128-row nodes of round 1; GLS_LEAF128=0, kept for A/B).
int leaf_size() {
  static const int v = (getenv("GLS_LEAF128") && atoi(getenv("GLS_LEAF128")) == 0) ? LEAF : blk::NB;
  return v;
}

int64_t first_block(int64_t n) {  // size of the leading block of the split of an n x n node
  const int64_t lf = leaf_size();
  const int64_t nblk = (n + lf - 1) / lf;
  return lf * ((nblk + 1) / 2);
}

// levels of the recursion tree of an n x n node (a leaf is one level)
int tree_depth(int64_t n) {
  if (n <= leaf_size()) return 1;
  const int64_t h1 = first_block(n);
  const int a = tree_depth(h1), b = tree_depth(n - h1);
  return 1 + (a > b ? a : b);
}

// Factor and invert the n x n node at A (T receives the inverse).  On entry the node's leading
// first_block(n) x first_block(n) block is up to date in the order of the main stream; the rest of
// the node (rows below it) is up to date once `rest_ready` has fired (nullptr: already).
void chol_inv_rec(RecCtx& rc, int64_t n, double* A, double* T, int64_t ld, int64_t goff, cudaEvent_t rest_ready,
                  int depth) {
  cudaStream_t s = rc.s;
  if (leaf_size() == blk::NB && n <= blk::NB) {
    if (first_use_on_device((const void*)chol_inv_leaf128))
      cudaFuncSetAttribute(chol_inv_leaf128, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)blk::SMEM);
    if (rest_ready) cudaStreamWaitEvent(s, rest_ready, 0);
    wait_cols(rc, s, goff + n);
    mark(s, depth, "wait-rest");
    chol_inv_leaf128<<<1, blk::THREADS, blk::SMEM, s>>>((int)n, A, T, ld, goff, rc.st);
    if (rc.lc) ++*rc.lc;
    mark(s, depth, "leaf");
    return;
  }
  if (n <= LEAF) {
    constexpr int kLeafSmem = 2 * LEAF * LLD * sizeof(double);
    if (first_use_on_device((const void*)chol_inv_leaf))
      cudaFuncSetAttribute(chol_inv_leaf, cudaFuncAttributeMaxDynamicSharedMemorySize, kLeafSmem);
    if (rest_ready) cudaStreamWaitEvent(s, rest_ready, 0);
    wait_cols(rc, s, goff + n);
    mark(s, depth, "wait-rest");
    chol_inv_leaf<<<1, LEAF_THREADS, kLeafSmem, s>>>((int)n, A, T, ld, goff, rc.st);
    if (rc.lc) ++*rc.lc;
    mark(s, depth, "leaf");
    return;
  }
  if (n <= 2 * LEAF && first_block(n) == LEAF) {  // both leaves and the node's products in one CTA
    constexpr int kNodeSmem = 6 * LEAF * LLD * sizeof(double);
    if (first_use_on_device((const void*)chol_inv_node128))
      cudaFuncSetAttribute(chol_inv_node128, cudaFuncAttributeMaxDynamicSharedMemorySize, kNodeSmem);
    if (rest_ready) cudaStreamWaitEvent(s, rest_ready, 0);
    wait_cols(rc, s, goff + n);
    mark(s, depth, "wait-rest");
    chol_inv_node128<<<1, LEAF_THREADS, kNodeSmem, s>>>((int)n, A, T, ld, goff, rc.st);
    if (rc.lc) ++*rc.lc;
    mark(s, depth, "leaf");
    return;
  }
  const int d = depth < kMaxDepth ? depth : kMaxDepth - 1;
  const int64_t h1 = first_block(n), h2 = n - h1;
  double* A11 = A;
  double* A21 = A + h1;
  double* A22 = A + h1 + h1 * ld;
  double* T11 = T;
  double* T21 = T + h1;  // holds L21 until T21 is formed
  double* T22 = T + h1 + h1 * ld;
  chol_inv_rec(rc, h1, A11, T11, ld, goff, nullptr, depth + 1);
  if (rest_ready) cudaStreamWaitEvent(s, rest_ready, 0);  // A21, A22 updated by the caller's side work
  mark(s, depth, "wait-rest");
  // L21 = A21 T11^T and A22 -= L21 L21^T, split at g = the leading block of the A22 node: its rows
  // [0, g) on the main stream (all the next leaf needs), the rest on the side stream, overlapping
  // the recursion into A22's leading block.
  // (small nodes: no split -- the extra launches cost more than the overlap gains)
  const int64_t g = h2 >= kLookaheadMin ? first_block(h2) : h2;
  cudaEvent_t e_start = record(rc, s);
  dgemm(s, g, h1, h1, 1.0, A21, ld, 'N', T11, ld, 'T', 0.0, T21, ld, GEMM_KMAX_COL, rc.lc, rc.ws_main);
  mark(s, depth, "L21top");
  cudaEvent_t e_top = record(rc, s);
  wait_cols(rc, s, goff + h1 + g);
  dgemm(s, g, g, h1, -1.0, T21, ld, 'N', T21, ld, 'T', 1.0, A22, ld, GEMM_LOWER_C, rc.lc, rc.ws_main);
  mark(s, depth, "SYRK11");
  cudaEvent_t e_rest = nullptr;
  cudaStream_t sd = rc.side[d];
  if (h2 > g) {
    // the look-ahead products start after the main stream's two (GLS_SIDE_AFTER=1): persistent CTAs
    // hold their SMs for the whole product, so started together they left L21top / SYRK11 -- the
    // critical path -- a few SMs; the side work has the next leaf's whole recursion to hide behind
    static const bool after = !(getenv("GLS_SIDE_AFTER") && atoi(getenv("GLS_SIDE_AFTER")) == 0);
    cudaStreamWaitEvent(sd, after ? record(rc, s) : e_start, 0);
    dgemm(sd, h2 - g, h1, h1, 1.0, A21 + g, ld, 'N', T11, ld, 'T', 0.0, T21 + g, ld, GEMM_KMAX_COL, rc.lc,
          rc.ws_side[d], rc.off_side);
    cudaStreamWaitEvent(sd, e_top, 0);
    wait_cols(rc, sd, goff + n);
    // rows [g, h2) of the lower triangle: columns [0, g) full, [g, h2) lower
    dgemm(sd, h2 - g, g, h1, -1.0, T21 + g, ld, 'N', T21, ld, 'T', 1.0, A22 + g, ld, 0, rc.lc, rc.ws_side[d],
          rc.off_side);
    dgemm(sd, h2 - g, h2 - g, h1, -1.0, T21 + g, ld, 'N', T21 + g, ld, 'T', 1.0, A22 + g + g * ld, ld,
          GEMM_LOWER_C, rc.lc, rc.ws_side[d], rc.off_side);
    e_rest = record(rc, sd);
  }
  // Y = L21 T11 -> A21's place, on the aux stream (after every read of A21 and every write of L21)
  cudaStream_t sa = rc.aux[d];
  cudaStreamWaitEvent(sa, record(rc, s), 0);
  if (e_rest) cudaStreamWaitEvent(sa, e_rest, 0);
  dgemm(sa, h2, h1, h1, 1.0, T21, ld, 'N', T11, ld, 'N', 0.0, A21, ld, GEMM_KMIN_COL, rc.lc, rc.ws_aux[d],
        rc.off_aux);
  cudaEvent_t e_y = record(rc, sa);
  chol_inv_rec(rc, h2, A22, T22, ld, goff + h1, e_rest, depth + 1);
  // T21 = -T22 Y  (overwrites L21: Y, and with it every reader of L21, must be complete)
  cudaStreamWaitEvent(s, e_y, 0);
  mark(s, depth, "wait-Y");
  dgemm(s, h2, h1, h2, -1.0, T22, ld, 'N', A21, ld, 'N', 0.0, T21, ld, GEMM_KMAX_ROW, rc.lc, rc.ws_main);
  mark(s, depth, "T21");
}

}  // namespace

void chol_prepare(cudaStream_t s, int64_t n, const double* A, int64_t ld, CholStatus* st,
                  int64_t* lc) {
  maxdiag_kernel<<<1, 256, 0, s>>>(n, A, ld, st);
  if (lc) ++*lc;
}

void chol_inv(cudaStream_t s, int64_t n, double* A, double* T, int64_t ld, CholStatus* st,
              int64_t* lc, const ColsReady* arriving) {
  int lo = 0, hi = 0;
  cudaDeviceGetStreamPriorityRange(&lo, &hi);  // lo = least urgent
  int depth = tree_depth(n);
  if (depth > kMaxDepth) depth = kMaxDepth;
  RecCtx rc{};
  rc.s = s;
  std::vector<cudaEvent_t> events;
  rc.events = &events;
  rc.st = st;
  rc.lc = lc;
  rc.arriving = arriving && arriving->nchunks > 0 ? arriving : nullptr;
  {
    // The look-ahead GEMMs and Y (needed only at the end of their node) walk their tiles on a grid
    // that leaves kFreeSms SMs to the critical path: their long CTAs would otherwise hold back its
    // small kernels (a 128 x 128 x 128 product took 140 us instead of 10 behind a 5000^3 Y)
    int dev0 = 0, sms = 148;
    cudaGetDevice(&dev0);
    cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev0);
    static const int freeq = getenv("GLS_CHOL_FREE_SMS") ? atoi(getenv("GLS_CHOL_FREE_SMS")) : kFreeSms;
    rc.off_ctas = freeq > 0 && sms > freeq ? 2 * (sms - freeq) : 0;  // 2 CTAs per SM
    static const int cap_side = getenv("GLS_CAP_SIDE") ? atoi(getenv("GLS_CAP_SIDE")) : 0;
    static const int cap_aux = getenv("GLS_CAP_AUX") ? atoi(getenv("GLS_CAP_AUX")) : 0;
    // Y (aux) leaves 48 SMs: it often runs beside a look-ahead product of a deeper level, and two capped
    // persistent products together had taken every SM from the main stream (A/B over side / aux caps:
    // profiles/r02_create_caps_ab.txt -- 132 / 100 SMs best, 25.8 vs 26.2 ms at n = 1e4)
    rc.off_side = cap_side > 0 ? 2 * cap_side : rc.off_ctas;
    rc.off_aux = cap_aux > 0 ? 2 * cap_aux : (freeq > 0 && sms > kFreeSmsY ? 2 * (sms - kFreeSmsY) : 0);
  }
  // split-K workspaces (main + side and aux per depth) from the stream-ordered pool
  double* ws = nullptr;
  const size_t nws = 1 + 2 * (size_t)depth;
  int wsdev = 0;
  cudaGetDevice(&wsdev);
  if (gls_pool_alloc((void**)&ws, nws * kSplitKWsDoubles * sizeof(double), wsdev, s) != cudaSuccess) {
    cudaGetLastError();
    ws = nullptr;
  }
  rc.ws_main = ws;
  // side/aux streams: created once per device and kept (stream creation would cost ~0.5 ms a call)
  static cudaStream_t pool_side[64][kMaxDepth] = {}, pool_aux[64][kMaxDepth] = {};
  int dev = 0;
  cudaGetDevice(&dev);
  if (dev < 0 || dev >= 64) dev = 0;
  for (int d = 0; d < depth; ++d) {
    if (!pool_side[dev][d]) cudaStreamCreateWithPriority(&pool_side[dev][d], cudaStreamNonBlocking, lo);
    // Y is on the critical path (the node's T21 waits for it): high priority, unlike the look-ahead
    if (!pool_aux[dev][d]) cudaStreamCreateWithPriority(&pool_aux[dev][d], cudaStreamNonBlocking, hi);
    rc.side[d] = pool_side[dev][d];
    rc.aux[d] = pool_aux[dev][d];
    rc.ws_side[d] = ws ? ws + (1 + 2 * d) * kSplitKWsDoubles : nullptr;
    rc.ws_aux[d] = ws ? ws + (2 + 2 * d) * kSplitKWsDoubles : nullptr;
  }
  // the side/aux streams see the workspace allocation through this event
  cudaEvent_t e0 = record(rc, s);
  for (int d = 0; d < depth; ++d) {
    cudaStreamWaitEvent(rc.side[d], e0, 0);
    cudaStreamWaitEvent(rc.aux[d], e0, 0);
  }
  static const bool trace = getenv("GLS_TRACE_CHOL") != nullptr;
  std::vector<Mark> marks;
  if (trace) {
    g_marks = &marks;
    mark(s, -1, "start");
  }
  chol_inv_rec(rc, n, A, T, ld, 0, nullptr, 0);
  if (trace) {
    cudaStreamSynchronize(s);
    double agg[kMaxDepth][6] = {};
    const char* names[6] = {"leaf", "wait-rest", "L21top", "SYRK11", "wait-Y", "T21"};
    for (size_t k = 1; k < marks.size(); ++k) {
      float ms = 0.f;
      cudaEventElapsedTime(&ms, marks[k - 1].e, marks[k].e);
      const int dd = marks[k].depth < kMaxDepth ? marks[k].depth : kMaxDepth - 1;
      for (int q = 0; q < 6; ++q)
        if (strcmp(marks[k].what, names[q]) == 0) agg[dd][q] += ms;
    }
    float tot = 0.f;
    cudaEventElapsedTime(&tot, marks.front().e, marks.back().e);
    fprintf(stderr, "[chol] total %.3f ms on the main stream\n", tot);
    for (int dd = 0; dd < kMaxDepth; ++dd) {
      double sum = 0;
      for (int q = 0; q < 6; ++q) sum += agg[dd][q];
      if (sum > 0)
        fprintf(stderr, "[chol] depth %2d: leaf %7.3f wait-rest %7.3f L21top %7.3f SYRK11 %7.3f wait-Y %7.3f T21 %7.3f\n",
                dd, agg[dd][0], agg[dd][1], agg[dd][2], agg[dd][3], agg[dd][4], agg[dd][5]);
    }
    for (auto& m : marks) cudaEventDestroy(m.e);
    g_marks = nullptr;
  }
  // join: everything issued on the side and aux streams is ordered before later work on s
  for (int d = 0; d < depth; ++d) {
    cudaStreamWaitEvent(s, record(rc, rc.side[d]), 0);
    cudaStreamWaitEvent(s, record(rc, rc.aux[d]), 0);
  }
  if (ws) cudaFreeAsync(ws, s);  // after the join
  return_events(events);
}

}  // namespace gls
