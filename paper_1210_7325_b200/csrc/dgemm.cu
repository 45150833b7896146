// dgemm.cu -- generic FP64 GEMM on the B200 FP64 tensor pipe (mma.sync m8n8k4 f64 -> DMMA.8x8x4).
//
// Used only by the once-per-context setup (gls_create): the recursive Cholesky + inverse of M
// (Alg. 5 line 1), X~_L = L^{-1} X_L, y~ = L^{-1} y
// (Alg. 5 lines 2, 4) and S_TL / b_T (Alg. 5 lines 5, 6).  Not on the per-block hot path.
//
// Tile 64 x 64 x 16, 4 warps (2 x 2, 32 x 32 each), register-prefetched double buffer.
// Triangular operands skip all-zero K ranges through GemmFlags.
#include "gls_internal.cuh"

namespace gls {
namespace {

constexpr int BM = 64, BN = 64, BK = 16, LDS_ = 20;  // smem row stride 20 doubles: conflict-free frags

__device__ __forceinline__ void dmma(double (&c)[2], double a, double b) {
  asm volatile("mma.sync.aligned.m8n8k4.row.col.f64.f64.f64.f64 {%0,%1}, {%2}, {%3}, {%0,%1};\n"
               : "+d"(c[0]), "+d"(c[1])
               : "d"(a), "d"(b));
}

struct GemmParams {
  int64_t M, N, K;
  const double* A;
  int64_t lda;
  const double* B;
  int64_t ldb;
  double* C;
  int64_t ldc;
  double alpha, beta;
  int flags;
};

template <bool TA, bool TB>
__global__ void __launch_bounds__(128) dgemm_kernel(GemmParams p) {
  __shared__ double As[2][BM * LDS_];
  __shared__ double Bs[2][BN * LDS_];
  const int64_t r0 = (int64_t)blockIdx.x * BM, c0 = (int64_t)blockIdx.y * BN;
  if ((p.flags & GEMM_LOWER_C) && c0 >= r0 + BM) return;
  int64_t kb = 0, ke = p.K;
  if (p.flags & GEMM_KMIN_COL) kb = (c0 / BK) * BK;
  if (p.flags & GEMM_KMAX_ROW) ke = min(ke, r0 + BM);
  if (p.flags & GEMM_KMAX_COL) ke = min(ke, c0 + BN);

  const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
  const int wm = warp & 1, wn = warp >> 1;
  double acc[4][4][2];
#pragma unroll
  for (int t = 0; t < 4; ++t)
#pragma unroll
    for (int s = 0; s < 4; ++s) acc[t][s][0] = acc[t][s][1] = 0.0;

  double ra[8], rb[8];
  auto load = [&](int64_t k0) {
#pragma unroll
    for (int j = 0; j < 8; ++j) {
      const int idx = tid + j * 128;
      // op(A)[m][k]
      int m, k;
      if (!TA) { m = idx % BM; k = idx / BM; } else { k = idx % BK; m = idx / BK; }
      const int64_t gm = r0 + m, gk = k0 + k;
      double v = 0.0;
      if (gm < p.M && gk < ke && gk >= kb) v = TA ? p.A[gk + gm * p.lda] : p.A[gm + gk * p.lda];
      ra[j] = v;
      // op(B)[k][n]
      int n;
      if (!TB) { k = idx % BK; n = idx / BK; } else { n = idx % BN; k = idx / BN; }
      const int64_t gn = c0 + n, gk2 = k0 + k;
      double w = 0.0;
      if (gn < p.N && gk2 < ke && gk2 >= kb) w = TB ? p.B[gn + gk2 * p.ldb] : p.B[gk2 + gn * p.ldb];
      rb[j] = w;
    }
  };
  auto store = [&](int buf) {
#pragma unroll
    for (int j = 0; j < 8; ++j) {
      const int idx = tid + j * 128;
      int m, k, n;
      if (!TA) { m = idx % BM; k = idx / BM; } else { k = idx % BK; m = idx / BK; }
      As[buf][m * LDS_ + k] = ra[j];
      if (!TB) { k = idx % BK; n = idx / BK; } else { n = idx % BN; k = idx / BN; }
      Bs[buf][n * LDS_ + k] = rb[j];
    }
  };

  const int l4 = lane >> 2, kk = lane & 3;
  int buf = 0;
  if (kb < ke) {
    load(kb);
    store(0);
  }
  __syncthreads();
  for (int64_t k0 = kb; k0 < ke; k0 += BK) {
    const bool more = k0 + BK < ke;
    if (more) load(k0 + BK);
#pragma unroll
    for (int ks = 0; ks < 4; ++ks) {
      double a[4], b[4];
#pragma unroll
      for (int t = 0; t < 4; ++t) a[t] = As[buf][(wm * 32 + t * 8 + l4) * LDS_ + ks * 4 + kk];
#pragma unroll
      for (int s = 0; s < 4; ++s) b[s] = Bs[buf][(wn * 32 + s * 8 + l4) * LDS_ + ks * 4 + kk];
#pragma unroll
      for (int t = 0; t < 4; ++t)
#pragma unroll
        for (int s = 0; s < 4; ++s) dmma(acc[t][s], a[t], b[s]);
    }
    if (more) store(buf ^ 1);
    __syncthreads();
    buf ^= 1;
  }
  // epilogue: lane holds C[m = l4][n = 2kk + e] of each 8x8 tile
#pragma unroll
  for (int t = 0; t < 4; ++t)
#pragma unroll
    for (int s = 0; s < 4; ++s)
#pragma unroll
      for (int e = 0; e < 2; ++e) {
        const int64_t gm = r0 + wm * 32 + t * 8 + l4;
        const int64_t gn = c0 + wn * 32 + s * 8 + 2 * kk + e;
        if (gm < p.M && gn < p.N) {
          double* cp = p.C + gm + gn * p.ldc;
          double v = p.alpha * acc[t][s][e];
          if (p.beta != 0.0) v += p.beta * *cp;
          *cp = v;
        }
      }
}

}  // namespace

void dgemm(cudaStream_t s, int64_t M, int64_t N, int64_t K, double alpha, const double* A,
           int64_t lda, char opA, const double* B, int64_t ldb, char opB, double beta, double* C,
           int64_t ldc, int flags, int64_t* launch_counter) {
  if (M <= 0 || N <= 0) return;
  GemmParams p{M, N, K, A, lda, B, ldb, C, ldc, alpha, beta, flags};
  dim3 grid((unsigned)((M + BM - 1) / BM), (unsigned)((N + BN - 1) / BN));
  const bool ta = (opA == 'T'), tb = (opB == 'T');
  if (!ta && !tb) dgemm_kernel<false, false><<<grid, 128, 0, s>>>(p);
  else if (!ta && tb) dgemm_kernel<false, true><<<grid, 128, 0, s>>>(p);
  else if (ta && !tb) dgemm_kernel<true, false><<<grid, 128, 0, s>>>(p);
  else dgemm_kernel<true, true><<<grid, 128, 0, s>>>(p);
  if (launch_counter) ++*launch_counter;
}

}  // namespace gls
