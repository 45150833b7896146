// gwfgls.cu -- GenABEL's algorithm for GWAS (Alg. 6, "gwfgls") on the B200
// kernels: the NEXT-2 rung of the algorithm ladder, kept beside hp-gwas so that
// Table II's cost ratio (gwfgls / hp-gwas ~ 2, cost O(n^3 + m n^2 + m n p^2))
// can be measured on the same hardware.  Not the hot path: the listing is followed as written,
// including the choices the paper criticises:
//
//   1  M := M^{-1}             (getri)  -- here M^{-1} = T^T T with T = L^{-1} from the library's own
//                                          potrf + inverse (chol_inv.cu), then the full n x n product
//   2  W_L^T := X_L^T M        (gemm)   -- W_L = M^{-1} X_L (n x pL)
//      for each X_Ri
//   3    W_Ri^T := X_Ri^T M    (gemv)   -- w = M^{-1} x per column: a full symmetric matrix-vector
//                                          product, 2 n^2 flops (hp-gwas: n^2); mode GWFGLS_GEMV runs one
//                                          gemv per column as listed, mode GWFGLS_GEMM casts the block's
//                                          gemvs as one GEMM (the improvement PAPER.md:351-355 names)
//   4    S_i := W^T X_i        (gemm)   -- W = (W_L | W_Ri), X_i = (X_L | X_Ri): all p x p entries as
//                                          dot products of length n (the symmetry is not used, line 2
//                                          "breaks the symmetry")
//   5    b_i := W^T y          (gemv)
//   6    b_i := S_i^{-1} b_i   (gesv)   -- LU with partial pivoting of the p x p S_i
//
// A zero or non-finite LU pivot marks the problem RankDeficient (NaN record, status 1), as the
// hp-gwas path does for its own rank rule (reading A4); the ladder's data is full rank.
#include <climits>
#include <cmath>
#include <string>

#include "../../include/gls.h"
#include "gls_internal.cuh"

using namespace gls;

namespace {

constexpr int64_t kGwChunkCols = 8192;  // columns of W_R per GEMM chunk (n x 8192 doubles of workspace)

// y = Minv x for a symmetric Minv (column-major, ld = n): output i is column i of Minv dotted with
// x, one warp per output, lanes over contiguous rows (coalesced), fixed-order shuffle reduction.
__global__ void gw_symv_kernel(int64_t n, const double* __restrict__ Minv, const double* __restrict__ x,
                               double* __restrict__ y) {
  const int lane = threadIdx.x & 31;
  for (int64_t i = ((int64_t)blockIdx.x * blockDim.x + threadIdx.x) >> 5; i < n;
       i += ((int64_t)gridDim.x * blockDim.x) >> 5) {
    const double* col = Minv + i * n;
    double acc = 0.0;
    for (int64_t j = lane; j < n; j += 32) acc = fma(col[j], __ldg(x + j), acc);
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) acc += __shfl_xor_sync(0xffffffffu, acc, o);
    if (lane == 0) y[i] = acc;
  }
}

// Lines 4-6 for problems [0, m): one warp per problem.  WR / XR: the problems' pR columns of
// W_R = M^{-1} X_R and X_R (column-major, ld n); WL / XL: the shared pL columns.
__global__ void gw_assemble_solve_kernel(int64_t n, int pL, int pR, int64_t m, const double* __restrict__ WL,
                                         const double* __restrict__ XL, const double* __restrict__ WR,
                                         const double* __restrict__ XR, const double* __restrict__ y,
                                         double* __restrict__ b_out, int32_t* __restrict__ status_out) {
  const int lane = threadIdx.x & 31;
  const int p = pL + pR;
  for (int64_t i = ((int64_t)blockIdx.x * blockDim.x + threadIdx.x) >> 5; i < m;
       i += ((int64_t)gridDim.x * blockDim.x) >> 5) {
    auto wcol = [&](int a) { return a < pL ? WL + (int64_t)a * n : WR + (i * pR + (a - pL)) * n; };
    auto xcol = [&](int a) { return a < pL ? XL + (int64_t)a * n : XR + (i * pR + (a - pL)) * n; };
    double S[20][20], r[20];
    for (int a = 0; a < p; ++a) {
      const double* wa = wcol(a);
      for (int c = 0; c <= p; ++c) {  // c == p: the right-hand side W^T y
        const double* xc = c < p ? xcol(c) : y;
        double acc = 0.0;
        for (int64_t j = lane; j < n; j += 32) acc = fma(wa[j], xc[j], acc);
#pragma unroll
        for (int o = 16; o > 0; o >>= 1) acc += __shfl_xor_sync(0xffffffffu, acc, o);
        if (c < p) S[a][c] = acc;
        else r[a] = acc;
      }
    }
    if (lane == 0) {
      // gesv: LU with partial pivoting, then the two triangular solves
      bool bad = false;
      for (int k = 0; k < p && !bad; ++k) {
        int piv = k;
        for (int q = k + 1; q < p; ++q)
          if (fabs(S[q][k]) > fabs(S[piv][k])) piv = q;
        if (!(fabs(S[piv][k]) > 0.0) || !isfinite(S[piv][k])) {
          bad = true;
          break;
        }
        if (piv != k) {
          for (int c = 0; c < p; ++c) {
            const double t = S[k][c];
            S[k][c] = S[piv][c];
            S[piv][c] = t;
          }
          const double t = r[k];
          r[k] = r[piv];
          r[piv] = t;
        }
        for (int q = k + 1; q < p; ++q) {
          const double f = S[q][k] / S[k][k];
          for (int c = k + 1; c < p; ++c) S[q][c] -= f * S[k][c];
          r[q] -= f * r[k];
        }
      }
      double* bo = b_out + i * p;
      if (bad) {
        const double qnan = __longlong_as_double(0x7ff8000000000000LL);
        for (int a = 0; a < p; ++a) bo[a] = qnan;
      } else {
        for (int k = p - 1; k >= 0; --k) {
          double v = r[k];
          for (int c = k + 1; c < p; ++c) v -= S[k][c] * r[c];
          r[k] = v / S[k][k];
        }
        for (int a = 0; a < p; ++a) bo[a] = r[a];
      }
      if (status_out) status_out[i] = bad ? 1 : 0;
    }
  }
}

__global__ void gw_maxdiag_tol(int64_t n, const double* A, CholStatus* st) {
  __shared__ double red[256];
  double mx = 0.0;
  for (int64_t k = threadIdx.x; k < n; k += blockDim.x) mx = fmax(mx, A[k + k * n]);
  red[threadIdx.x] = mx;
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

}  // namespace

struct gls_gwfgls {
  int device = 0;
  int64_t n = 0;
  int pL = 0, pR = 0;
  cudaStream_t s = nullptr;
  double* Minv = nullptr;  // n x n, the explicit inverse (line 1)
  double* XL = nullptr;    // n x pL
  double* WL = nullptr;    // n x pL = M^{-1} X_L (line 2)
  double* y = nullptr;     // n
  double* WR = nullptr;    // n x kGwChunkCols workspace (line 3)
  double* ws = nullptr;    // split-K workspace of dgemm
  int64_t launches = 0;
};

namespace {
void gw_free(gls_gwfgls* g) {
  if (!g) return;
  cudaDeviceSynchronize();  // (a user stream may still read the buffers)
  for (double* p : {g->Minv, g->XL, g->WL, g->y, g->WR, g->ws})
    if (p) cudaFreeAsync(p, g->s);  // back to the library's stream-ordered pool
  if (g->s) {
    cudaStreamSynchronize(g->s);
    cudaStreamDestroy(g->s);
  }
  delete g;
}
}  // namespace

extern "C" int gls_gwfgls_create(int64_t n, int32_t pL, int32_t pR, const double* M, const double* X_L,
                                 const double* y, gls_gwfgls** out) {
  if (!out) return GLS_ERR_ARG;
  *out = nullptr;
  if (!M || !y || (pL > 0 && !X_L)) return GLS_ERR_ARG;
  if (pL < 0 || pR < 1 || pL + pR > 20 || n <= pL + pR || n > (int64_t)INT32_MAX / 2) return GLS_ERR_DIM;
  gls_gwfgls* g = new gls_gwfgls();
  g->n = n;
  g->pL = pL;
  g->pR = pR;
  const size_t nn = (size_t)n * n * sizeof(double);
  double *A = nullptr, *T = nullptr;
  CholStatus* st = nullptr;
  CholStatus hst;
  auto fail = [&](int rc) {
    for (void* q : {(void*)A, (void*)T, (void*)st})
      if (q) cudaFreeAsync(q, g->s);
    cudaGetLastError();
    gw_free(g);
    return rc;
  };
  if (cudaGetDevice(&g->device) != cudaSuccess || cudaStreamCreateWithFlags(&g->s, cudaStreamNonBlocking) != cudaSuccess)
    return fail(GLS_ERR_CUDA);
  // device buffers from the library's stream-ordered pool (cached across creates, no page mapping)
  auto palloc = [&](auto** q, size_t bytes) { return gls_pool_alloc((void**)q, bytes, g->device, g->s); };
  if (palloc(&A, nn) != cudaSuccess || palloc(&T, nn) != cudaSuccess || palloc(&g->Minv, nn) != cudaSuccess ||
      palloc(&g->XL, (size_t)n * (pL > 0 ? pL : 1) * sizeof(double)) != cudaSuccess ||
      palloc(&g->WL, (size_t)n * (pL > 0 ? pL : 1) * sizeof(double)) != cudaSuccess ||
      palloc(&g->y, (size_t)n * sizeof(double)) != cudaSuccess ||
      palloc(&g->WR, (size_t)n * kGwChunkCols * sizeof(double)) != cudaSuccess ||
      palloc(&g->ws, kSplitKWsDoubles * sizeof(double)) != cudaSuccess ||
      palloc(&st, sizeof(CholStatus)) != cudaSuccess)
    return fail(GLS_ERR_OOM);
  cudaStream_t s = g->s;
  if (cudaMemcpyAsync(A, M, nn, cudaMemcpyDefault, s) != cudaSuccess || cudaMemsetAsync(T, 0, nn, s) != cudaSuccess ||
      (pL > 0 && cudaMemcpyAsync(g->XL, X_L, (size_t)n * pL * sizeof(double), cudaMemcpyDefault, s) != cudaSuccess) ||
      cudaMemcpyAsync(g->y, y, (size_t)n * sizeof(double), cudaMemcpyDefault, s) != cudaSuccess)
    return fail(GLS_ERR_CUDA);
  // line 1: M^{-1} = L^{-T} L^{-1} = T^T T (T from the library's potrf + inverse)
  gw_maxdiag_tol<<<1, 256, 0, s>>>(n, A, st);
  chol_inv(s, n, A, T, n, st, &g->launches);
  if (cudaMemcpyAsync(&hst, st, sizeof hst, cudaMemcpyDeviceToHost, s) != cudaSuccess ||
      cudaStreamSynchronize(s) != cudaSuccess)
    return fail(GLS_ERR_CUDA);
  if (hst.fail != ULLONG_MAX) return fail(GLS_ERR_NOT_SPD);
  // C[i][j] = sum_k T[k][i] T[k][j]; op(B) = T is lower triangular, so k >= j (GEMM_KMIN_COL)
  dgemm(s, n, n, n, 1.0, T, n, 'T', T, n, 'N', 0.0, g->Minv, n, GEMM_KMIN_COL, &g->launches, g->ws);
  // line 2: W_L = M^{-1} X_L
  if (pL > 0) dgemm(s, n, pL, n, 1.0, g->Minv, n, 'N', g->XL, n, 'N', 0.0, g->WL, n, 0, &g->launches, g->ws);
  if (cudaStreamSynchronize(s) != cudaSuccess || cudaGetLastError() != cudaSuccess) return fail(GLS_ERR_CUDA);
  cudaFreeAsync(A, s);
  cudaFreeAsync(T, s);
  cudaFreeAsync(st, s);
  A = T = nullptr;
  st = nullptr;
  if (cudaStreamSynchronize(s) != cudaSuccess) return fail(GLS_ERR_CUDA);  // buffers usable from any stream
  *out = g;
  return GLS_OK;
}

extern "C" int gls_gwfgls_solve(gls_gwfgls* g, const double* X_R, int64_t m_blk, double* b_out,
                                int32_t* status_out, int32_t mode) {
  if (!g || !X_R || !b_out || (mode != GLS_GWFGLS_GEMV && mode != GLS_GWFGLS_GEMM)) return GLS_ERR_ARG;
  if (m_blk < 1) return GLS_ERR_DIM;
  const int64_t n = g->n, pR = g->pR, p = g->pL + g->pR;
  cudaStream_t s = g->s;
  const int64_t chunk_groups = kGwChunkCols / pR;
  for (int64_t g0 = 0; g0 < m_blk; g0 += chunk_groups) {
    const int64_t gc = (m_blk - g0 < chunk_groups) ? m_blk - g0 : chunk_groups;
    const double* X = X_R + g0 * pR * n;
    if (mode == GLS_GWFGLS_GEMM) {
      // line 3 for the whole chunk as one product W_R = M^{-1} X_R
      dgemm(s, n, gc * pR, n, 1.0, g->Minv, n, 'N', X, n, 'N', 0.0, g->WR, n, 0, &g->launches, g->ws);
    } else {
      // line 3 as listed: one symmetric matrix-vector product per column
      const unsigned blocks = (unsigned)((n * 32 + 255) / 256 < 148 * 8 ? (n * 32 + 255) / 256 : 148 * 8);
      for (int64_t c = 0; c < gc * pR; ++c) {
        gw_symv_kernel<<<blocks, 256, 0, s>>>(n, g->Minv, X + c * n, g->WR + c * n);
        ++g->launches;
      }
    }
    // lines 4-6 (one warp per problem)
    const int64_t warps = gc;
    const unsigned blocks = (unsigned)((warps * 32 + 255) / 256 < 148 * 16 ? (warps * 32 + 255) / 256 : 148 * 16);
    gw_assemble_solve_kernel<<<blocks, 256, 0, s>>>(n, g->pL, g->pR, gc, g->WL, g->XL, g->WR, X, g->y,
                                                    b_out + g0 * p, status_out ? status_out + g0 : nullptr);
    ++g->launches;
  }
  if (cudaStreamSynchronize(s) != cudaSuccess || cudaGetLastError() != cudaSuccess) return GLS_ERR_CUDA;
  return GLS_OK;
}

extern "C" int64_t gls_gwfgls_launches(const gls_gwfgls* g) { return g ? g->launches : -1; }

extern "C" void gls_gwfgls_destroy(gls_gwfgls* g) { gw_free(g); }
