// dgemm.cu -- generic FP64 GEMM on the B200 FP64 tensor pipe (mma.sync m8n8k4 f64 -> DMMA.8x8x4).
//
// Used only by the once-per-context setup (gls_create): the recursive Cholesky + inverse of M
// (Alg. 5 line 1), X~_L = L^{-1} X_L, y~ = L^{-1} y
// (Alg. 5 lines 2, 4) and S_TL / b_T (Alg. 5 lines 5, 6).  Not on the per-block hot path.
//
// Tile 128 x 64 x 16, 8 warps (4 x 2, 32 x 32 each), 3-stage cp.async (LDGSTS) pipeline with
// zero-fill for ragged edges, any leading dimension / transpose.  Shared tiles are [row][k] with a
// 20-double row stride: the m8n8k4 fragment loads (lane (m, k) = (l/4, l%4)) are conflict-free.
// Triangular operands skip all-zero K ranges through GemmFlags.
#include <cuda.h>

#include <algorithm>
#include <climits>
#include <cstdio>
#include <cstdlib>

#include "gls_internal.cuh"

namespace gls {
namespace {

#ifndef GLS_DGEMM_BK
#define GLS_DGEMM_BK 16
#endif
#ifndef GLS_DGEMM_STAGES
#define GLS_DGEMM_STAGES 3
#endif
#ifndef GLS_DGEMM_BN
#define GLS_DGEMM_BN 64
#endif
constexpr int BM = 128, BN = GLS_DGEMM_BN, BK = GLS_DGEMM_BK, LDS_ = BK + 4, STAGES = GLS_DGEMM_STAGES,
              THREADS = 256;
// warp grid: 8 warps as WM x WN, warp tile (BM / WM) x (BN / WN) = TM x TN DMMA 8x8 tiles
constexpr int WM = BN == 64 ? 4 : 2, WN = 8 / WM, TM = BM / WM / 8, TN = BN / WN / 8;
constexpr int A_TILE = BM * LDS_, B_TILE = BN * LDS_;
constexpr int SMEM_BYTES = STAGES * (A_TILE + B_TILE) * 8;

__device__ __forceinline__ void dmma(double (&c)[2], double a, double b) {
  asm volatile("mma.sync.aligned.m8n8k4.row.col.f64.f64.f64.f64 {%0,%1}, {%2}, {%3}, {%0,%1};\n"
               : "+d"(c[0]), "+d"(c[1])
               : "d"(a), "d"(b));
}
__device__ __forceinline__ void cp_async8(double* dst, const double* src, bool valid) {
  const uint32_t d = (uint32_t)__cvta_generic_to_shared(dst);
  const int sz = valid ? 8 : 0;  // src-size 0 -> zero fill
  asm volatile("cp.async.ca.shared.global [%0], [%1], 8, %2;\n" ::"r"(d), "l"(src), "r"(sz) : "memory");
}
__device__ __forceinline__ void cp_async_commit() { asm volatile("cp.async.commit_group;\n" ::: "memory"); }
template <int N>
__device__ __forceinline__ void cp_async_wait() { asm volatile("cp.async.wait_group %0;\n" ::"n"(N) : "memory"); }

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
  int nsplit;   // split-K: blockIdx.z takes K tiles [z*nk/nsplit, (z+1)*nk/nsplit) ...
  double* ws;   // ... and writes its raw partial tile to ws[z][m + n*M] (reduced by dgemm_splitk_reduce)
};

__device__ __forceinline__ bool tile_skipped(const GemmParams& p, int64_t r0, int64_t c0) {
  return (p.flags & GEMM_LOWER_C) && c0 >= r0 + BM;
}

template <bool TA, bool TB>
__global__ void __launch_bounds__(THREADS, BN == 64 ? 2 : 1) dgemm_kernel(GemmParams p) {
  extern __shared__ double sm[];
  double* As = sm;
  double* Bs = sm + STAGES * A_TILE;
  // one output tile per CTA on the full grid; a capped grid (dgemm's max_ctas) walks the tiles
  const int64_t tm = (p.M + BM - 1) / BM, ntiles = tm * ((p.N + BN - 1) / BN);
  for (int64_t tile = blockIdx.x + (int64_t)blockIdx.y * gridDim.x; tile < ntiles;
       tile += (int64_t)gridDim.x * gridDim.y) {
  const int64_t r0 = (tile % tm) * BM, c0 = (tile / tm) * BN;
  if (tile_skipped(p, r0, c0)) continue;
  int64_t kb = 0, ke = p.K;
  if (p.flags & GEMM_KMIN_COL) kb = (c0 / BK) * BK;
  if (p.flags & GEMM_KMAX_ROW) ke = min(ke, r0 + BM);
  if (p.flags & GEMM_KMAX_COL) ke = min(ke, c0 + BN);
  const int64_t kbeg = kb;  // element-level lower bound for the zero fill
  kb = (kb / BK) * BK;
  int nk = (ke > kb) ? (int)((ke - kb + BK - 1) / BK) : 0;
  if (p.nsplit > 1) {  // this split's share of the K tiles
    const int z = blockIdx.z;
    const int t0 = (int)((int64_t)z * nk / p.nsplit), t1 = (int)((int64_t)(z + 1) * nk / p.nsplit);
    kb += (int64_t)t0 * BK;
    nk = t1 - t0;
  }

  const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
  const int wm = warp % WM, wn = warp / WM;

  auto issue = [&](int kt, int stg) {
    const int64_t k0 = kb + (int64_t)kt * BK;
    double* as = As + stg * A_TILE;
    double* bs = Bs + stg * B_TILE;
#pragma unroll
    for (int j = 0; j < (BM * BK) / THREADS; ++j) {  // 8
      const int idx = tid + j * THREADS;
      int m, k;
      if (!TA) { m = idx % BM; k = idx / BM; } else { k = idx % BK; m = idx / BK; }
      const int64_t gm = r0 + m, gk = k0 + k;
      const bool v = gm < p.M && gk < ke && gk >= kbeg;
      const double* src = v ? (TA ? p.A + gk + gm * p.lda : p.A + gm + gk * p.lda) : p.A;
      cp_async8(as + m * LDS_ + k, src, v);
    }
#pragma unroll
    for (int j = 0; j < (BN * BK) / THREADS; ++j) {  // 4
      const int idx = tid + j * THREADS;
      int n, k;
      if (!TB) { k = idx % BK; n = idx / BK; } else { n = idx % BN; k = idx / BN; }
      const int64_t gn = c0 + n, gk = k0 + k;
      const bool v = gn < p.N && gk < ke && gk >= kbeg;
      const double* src = v ? (TB ? p.B + gn + gk * p.ldb : p.B + gk + gn * p.ldb) : p.B;
      cp_async8(bs + n * LDS_ + k, src, v);
    }
  };

  double acc[TM][TN][2];
#pragma unroll
  for (int t = 0; t < TM; ++t)
#pragma unroll
    for (int s = 0; s < TN; ++s) acc[t][s][0] = acc[t][s][1] = 0.0;

  const int l4 = lane >> 2, kk = lane & 3;
#pragma unroll
  for (int s = 0; s < STAGES - 1; ++s) {
    if (s < nk) issue(s, s);
    cp_async_commit();
  }
  for (int kt = 0; kt < nk; ++kt) {
    cp_async_wait<STAGES - 2>();
    __syncthreads();
    const int nxt = kt + STAGES - 1;
    if (nxt < nk) issue(nxt, nxt % STAGES);
    cp_async_commit();
    const double* as = As + (kt % STAGES) * A_TILE;
    const double* bs = Bs + (kt % STAGES) * B_TILE;
#pragma unroll
    for (int ks = 0; ks < BK / 4; ++ks) {
      double a[TM], b[TN];
#pragma unroll
      for (int t = 0; t < TM; ++t) a[t] = as[(wm * TM * 8 + t * 8 + l4) * LDS_ + ks * 4 + kk];
#pragma unroll
      for (int s = 0; s < TN; ++s) b[s] = bs[(wn * TN * 8 + s * 8 + l4) * LDS_ + ks * 4 + kk];
#pragma unroll
      for (int t = 0; t < TM; ++t)
#pragma unroll
        for (int s = 0; s < TN; ++s) dmma(acc[t][s], a[t], b[s]);
    }
  }
  cp_async_wait<0>();
  // epilogue: lane holds C[m = l4][n = 2kk + e] of each 8x8 tile
#pragma unroll
  for (int t = 0; t < TM; ++t)
#pragma unroll
    for (int s = 0; s < TN; ++s)
#pragma unroll
      for (int e = 0; e < 2; ++e) {
        const int64_t gm = r0 + wm * TM * 8 + t * 8 + l4;
        const int64_t gn = c0 + wn * TN * 8 + s * 8 + 2 * kk + e;
        if (gm < p.M && gn < p.N) {
          if (p.nsplit > 1) {
            p.ws[(int64_t)blockIdx.z * p.M * p.N + gm + gn * p.M] = acc[t][s][e];
          } else {
            double* cp = p.C + gm + gn * p.ldc;
            double v = p.alpha * acc[t][s][e];
            if (p.beta != 0.0) v += p.beta * *cp;
            *cp = v;
          }
        }
      }
  __syncthreads();  // the next tile's prologue reuses the stages
  }
}

// C = alpha * sum_z ws[z] + beta * C, splits summed in a fixed order (deterministic).
__global__ void dgemm_splitk_reduce(GemmParams p) {
  for (int64_t o = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; o < p.M * p.N;
       o += (int64_t)gridDim.x * blockDim.x) {
    const int64_t gm = o % p.M, gn = o / p.M;
    if (tile_skipped(p, (gm / BM) * BM, (gn / BN) * BN)) continue;
    double v = 0.0;
    for (int z = 0; z < p.nsplit; ++z) v += p.ws[(int64_t)z * p.M * p.N + o];
    double* cp = p.C + gm + gn * p.ldc;
    v *= p.alpha;
    if (p.beta != 0.0) v += p.beta * *cp;
    *cp = v;
  }
}

// ---------------------------------------------------------------- TMA-fed DMMA GEMM (op(A) = A)
// The large products of gls_create (L21 = A21 T11^T, the SYRK, Y = L21 T11, T21 = -T22 Y) all read A
// untransposed.  A persistent CTA per SM walks its output tiles (BM x BN = 128 x 64); warp 8 is a TMA
// producer (one lane) filling an 8-stage ring of [BK = 16] x (A: 128 rows, B: 64 columns) tiles under
// full / empty mbarriers, warps 0-7 (4 x 2, 32 x 32 each) issue mma.sync.m8n8k4.f64 (DMMA.8x8x4) from
// LDS.128 fragment loads: every 16-byte load feeds two DMMA tiles.
//   A (M-major in memory, m contiguous): smem [k][128 m], no swizzle; a lane's LDS.128 at (k, m pair
//     2 l4, 2 l4 + 1) gives the A fragments of two row tiles -- tile t covers rows 16 (t >> 1) + 2 l4 +
//     (t & 1) of the warp's 32 (a row permutation the epilogue undoes); 4 k rows 1 KB apart: 4 wavefronts
//     per 512 bytes, conflict-free.
//   B^T (BT, op(B) = B^T with B N x K, n contiguous): smem [k][64 n], the same pairing on the columns.
//   B (K-major, op(B) = B with B K x N, k contiguous): smem [64 n][16 k] with the 128-byte swizzle; an
//     LDS.128 gives two consecutive k of one column (chunk (2 kk + P) ^ (n & 7)); the k-steps use the
//     matching k permutation (DMMA k index kk <-> k = 4 kk + 2 P + e) on both operands.
// Ragged M / N edges only touch outputs that are not stored; the K tail is zeroed in registers.  Triangular K ranges skip whole 16-wide stages; the
// skipped and the partially covered stages' extra elements are zeros of the triangular operand (every
// call site's operand holds zeros there), so no element masking is needed.
namespace tg {
constexpr int BM = 128, BN = 64, BK = 16, CW = 8, THREADS = (CW + 1) * 32, STAGES = 8;
constexpr int A_BYTES = BM * BK * 8, B_BYTES = BN * BK * 8, STAGE_BYTES = A_BYTES + B_BYTES;
constexpr int SMEM = STAGES * STAGE_BYTES + 2 * STAGES * 8 + 1024;

struct Params {
  int64_t M, N, K;
  double* C;
  int64_t ldc;
  double alpha, beta;
  int flags;
  int64_t tm, ntiles;
  int64_t tn, nvalid;  // tile columns; tiles actually computed (LOWER_C: those meeting the lower triangle)
  int order;           // tile order (ORD_*): longest K range first
  int snake;           // CTA b takes ordered tiles q G + b (q even) / q G + G - 1 - b (q odd)
};

__device__ __forceinline__ uint32_t su32(const void* p) { return (uint32_t)__cvta_generic_to_shared(p); }
__device__ __forceinline__ void bar_init(uint64_t* b, uint32_t c) {
  asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;\n" ::"r"(su32(b)), "r"(c));
}
__device__ __forceinline__ void bar_expect(uint64_t* b, uint32_t bytes) {
  asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;\n" ::"r"(su32(b)), "r"(bytes) : "memory");
}
__device__ __forceinline__ void bar_arrive(uint64_t* b) {
  asm volatile("mbarrier.arrive.shared::cta.b64 _, [%0];\n" ::"r"(su32(b)) : "memory");
}
__device__ __forceinline__ void bar_wait(uint64_t* b, uint32_t ph) {
  asm volatile(
      "{\n.reg .pred P1;\nW_%=:\nmbarrier.try_wait.parity.shared::cta.b64 P1, [%0], %1;\n@!P1 bra W_%=;\n}\n" ::"r"(
          su32(b)),
      "r"(ph)
      : "memory");
}
__device__ __forceinline__ void tma2d(void* dst, const CUtensorMap* m, int c0, int c1, uint64_t* b) {
  asm volatile(
      "cp.async.bulk.tensor.2d.shared::cluster.global.tile.mbarrier::complete_tx::bytes [%0], [%1, {%2, %3}], "
      "[%4];\n" ::"r"(su32(dst)),
      "l"(m), "r"(c0), "r"(c1), "r"(su32(b))
      : "memory");
}
__device__ __forceinline__ void lds128(uint32_t a, double& x, double& y) {
  asm volatile("ld.shared.v2.f64 {%0, %1}, [%2];\n" : "=d"(x), "=d"(y) : "r"(a));
}

// Tile schedule.  A triangular operand makes the tiles' K ranges (their cost) linear in the tile's row
// or column, and LOWER_C leaves only the tiles meeting the lower triangle; a plain round-robin over the
// tile grid then gives some CTAs twice the work of others (measured: mid-size products of the
// recursion at 10-17 TF/s).  The computed tiles are enumerated longest first and dealt to the
// persistent CTAs in a snake order (round q: CTA b takes q G + b, or q G + G - 1 - b when q is odd),
// which balances linear cost profiles.  Which tiles a CTA computes and in what order changes no bit of
// any tile (each tile's K loop is fixed).
enum { ORD_NATURAL = 0, ORD_COL_DESC = 1, ORD_COL_ASC = 2, ORD_ROW_DESC = 3, ORD_LOWER = 4 };
__device__ __forceinline__ bool tile_at(const Params& p, int64_t q, int64_t& r0, int64_t& c0) {
  const int64_t G = gridDim.x, b = blockIdx.x;
  const int64_t idx = q * G + ((p.snake && (q & 1)) ? G - 1 - b : b);
  if (idx >= p.nvalid) return false;
  int64_t i, j;
  switch (p.order) {
    case ORD_COL_DESC: j = p.tn - 1 - idx / p.tm; i = idx % p.tm; break;
    case ORD_COL_ASC: j = idx / p.tm; i = idx % p.tm; break;
    case ORD_ROW_DESC: i = p.tm - 1 - idx / p.tn; j = idx % p.tn; break;
    case ORD_LOWER: {  // row i holds the columns j with j BN < (i + 1) BM
      int64_t rem = idx;
      i = 0;
      for (;; ++i) {
        int64_t cnt = ((i + 1) * BM + BN - 1) / BN;
        if (cnt > p.tn) cnt = p.tn;
        if (rem < cnt) break;
        rem -= cnt;
      }
      j = rem;
      break;
    }
    default: i = idx % p.tm; j = idx / p.tm; break;
  }
  r0 = i * BM;
  c0 = j * BN;
  return true;
}

// K range of an output tile (the old kernel's triangular rules, at stage granularity)
__device__ __forceinline__ void krange(const Params& p, int64_t r0, int64_t c0, int64_t& kb, int& nk) {
  int64_t b = 0, e = p.K;
  if (p.flags & GEMM_KMIN_COL) b = c0;
  if (p.flags & GEMM_KMAX_ROW) e = min(e, r0 + BM);
  if (p.flags & GEMM_KMAX_COL) e = min(e, c0 + BN);
  b = (b / BK) * BK;
  kb = b;
  nk = e > b ? (int)((e - b + BK - 1) / BK) : 0;
}

// The fragments of one half-stage (8 K values): a[j][t] / b[j][s] for the two DMMA k-steps j.
struct Frag {
  double a[2][4], b[2][4];
};
// BT (B N-major): half h holds k-steps 2h, 2h+1 (k = 4 (2h + j) + kk).  !BT (B K-major): half P holds
// k = 4 kk + 2 P + j.  Fragments of k >= kvalid are zeroed (K tail).
template <bool BT>
__device__ __forceinline__ void load_half(Frag& f, uint32_t as, uint32_t bs, uint32_t a_lane, int wn, int l4, int kk,
                                          int h, int kvalid) {
#pragma unroll
  for (int j = 0; j < 2; ++j) {
    const int k = BT ? 4 * (2 * h + j) + kk : 4 * kk + 2 * h + j;
    lds128(as + k * (BM * 8) + a_lane, f.a[j][0], f.a[j][1]);
    lds128(as + k * (BM * 8) + a_lane + 128, f.a[j][2], f.a[j][3]);
    if (BT) {
      lds128(bs + k * (BN * 8) + (wn * 32 + 2 * l4) * 8, f.b[j][0], f.b[j][1]);
      lds128(bs + k * (BN * 8) + (wn * 32 + 2 * l4) * 8 + 128, f.b[j][2], f.b[j][3]);
    }
  }
  if (!BT) {
#pragma unroll
    for (int s = 0; s < 4; ++s) {
      const int n = wn * 32 + 8 * s + l4;
      lds128(bs + n * 128 + ((((2 * kk + h) ^ (n & 7)) & 7) << 4), f.b[0][s], f.b[1][s]);
    }
  }
  if (kvalid < BK) {
#pragma unroll
    for (int j = 0; j < 2; ++j) {
      const int k = BT ? 4 * (2 * h + j) + kk : 4 * kk + 2 * h + j;
      if (k >= kvalid) {
#pragma unroll
        for (int q = 0; q < 4; ++q) f.a[j][q] = f.b[j][q] = 0.0;
      }
    }
  }
}
__device__ __forceinline__ void mma_half(double (&acc)[4][4][2], const Frag& f) {
#pragma unroll
  for (int j = 0; j < 2; ++j)
#pragma unroll
    for (int t = 0; t < 4; ++t)
#pragma unroll
      for (int s = 0; s < 4; ++s) dmma(acc[t][s], f.a[j][t], f.b[j][s]);
}

template <bool BT>
__global__ void __launch_bounds__(THREADS, 1) dgemm_tma_kernel(const __grid_constant__ CUtensorMap amap,
                                                              const __grid_constant__ CUtensorMap bmap, const Params p) {
  extern __shared__ uint8_t smem_raw[];
  uint8_t* smem = (uint8_t*)(((uintptr_t)smem_raw + 1023) & ~(uintptr_t)1023);
  uint8_t* sA = smem;
  uint8_t* sB = smem + STAGES * A_BYTES;
  uint64_t* full = (uint64_t*)(sB + STAGES * B_BYTES);
  uint64_t* empty = full + STAGES;
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  if (threadIdx.x == 0) {
    for (int s = 0; s < STAGES; ++s) {
      bar_init(&full[s], 1);
      bar_init(&empty[s], CW);
    }
    asm volatile("fence.mbarrier_init.release.cluster;\n" ::: "memory");
  }
  __syncthreads();
  if (warp == CW) {
    // ------------------------------------------------------------ TMA producer
    if (lane == 0) {
      asm volatile("prefetch.tensormap [%0];\n" ::"l"(&amap) : "memory");
      asm volatile("prefetch.tensormap [%0];\n" ::"l"(&bmap) : "memory");
      int st = 0;
      uint32_t ph = 0;
      int64_t r0, c0;
      for (int64_t q = 0; tile_at(p, q, r0, c0); ++q) {
        if ((p.flags & GEMM_LOWER_C) && c0 >= r0 + BM) continue;  // (natural order only)
        int64_t kb;
        int nk;
        krange(p, r0, c0, kb, nk);
        for (int kt = 0; kt < nk; ++kt) {
          const int k0 = (int)(kb + (int64_t)kt * BK);
          bar_wait(&empty[st], ph ^ 1);
          bar_expect(&full[st], STAGE_BYTES);
          tma2d(sA + st * A_BYTES, &amap, (int)r0, k0, &full[st]);
          if (BT)
            tma2d(sB + st * B_BYTES, &bmap, (int)c0, k0, &full[st]);
          else
            tma2d(sB + st * B_BYTES, &bmap, k0, (int)c0, &full[st]);
          if (++st == STAGES) {
            st = 0;
            ph ^= 1;
          }
        }
      }
    }
    return;
  }
  // -------------------------------------------------------------- DMMA consumers
  const int wm = warp & 3, wn = warp >> 2;
  const int l4 = lane >> 2, kk = lane & 3;
  const uint32_t a_base = su32(sA), b_base = su32(sB);
  const uint32_t a_lane = (uint32_t)((wm * 32 + 2 * l4) * 8);
  int st = 0;
  uint32_t ph = 0;
  int64_t r0, c0;
  for (int64_t q = 0; tile_at(p, q, r0, c0); ++q) {
    if ((p.flags & GEMM_LOWER_C) && c0 >= r0 + BM) continue;
    int64_t kb;
    int nk;
    krange(p, r0, c0, kb, nk);
    double acc[4][4][2];
#pragma unroll
    for (int t = 0; t < 4; ++t)
#pragma unroll
      for (int s = 0; s < 4; ++s) acc[t][s][0] = acc[t][s][1] = 0.0;
    // Software pipeline over half-stages (8 LDS.128 -> 32 DMMAs each): the fragments of half-stage h+1
    // (the next stage's first half after waiting for it) are loaded while half-stage h's DMMAs issue.
    Frag F0, F1;
    int cur = st;
    uint32_t cph = ph;
    if (nk > 0) {
      bar_wait(&full[cur], cph);
      load_half<BT>(F0, a_base + cur * A_BYTES, b_base + cur * B_BYTES, a_lane, wn, l4, kk, 0,
                    (int)min((int64_t)BK, p.K - kb));
    }
    for (int kt = 0; kt < nk; ++kt) {
      // the last stage of a K not divisible by 16: the rows of the box beyond K are not zero in shared
      // memory (measured: a box cut along its outer dimension leaves them stale), so load_half zeroes
      // the fragments of k >= K in registers (a select, not a product: stale bits may be NaN)
      const int kvalid = (int)min((int64_t)BK, p.K - (kb + (int64_t)kt * BK));
      load_half<BT>(F1, a_base + cur * A_BYTES, b_base + cur * B_BYTES, a_lane, wn, l4, kk, 1, kvalid);
      mma_half(acc, F0);
      const int done = cur;
      if (++cur == STAGES) {
        cur = 0;
        cph ^= 1;
      }
      if (kt + 1 < nk) {
        bar_wait(&full[cur], cph);
        load_half<BT>(F0, a_base + cur * A_BYTES, b_base + cur * B_BYTES, a_lane, wn, l4, kk, 0,
                      (int)min((int64_t)BK, p.K - (kb + (int64_t)(kt + 1) * BK)));
      }
      mma_half(acc, F1);
      __syncwarp();
      if (lane == 0) bar_arrive(&empty[done]);
    }
    st = cur;
    ph = cph;
    // epilogue: lane holds C[m_d = l4][n_d = 2 kk + e] of each DMMA tile (t, s)
#pragma unroll
    for (int t = 0; t < 4; ++t) {
      const int64_t gm = r0 + wm * 32 + 16 * (t >> 1) + 2 * l4 + (t & 1);
#pragma unroll
      for (int s = 0; s < 4; ++s)
#pragma unroll
        for (int e = 0; e < 2; ++e) {
          const int64_t gn = BT ? c0 + wn * 32 + 16 * (s >> 1) + 2 * (2 * kk + e) + (s & 1)
                                : c0 + wn * 32 + 8 * s + 2 * kk + e;
          if (gm < p.M && gn < p.N) {
            double* cp = p.C + gm + gn * p.ldc;
            double v = p.alpha * acc[t][s][e];
            if (p.beta != 0.0) v += p.beta * *cp;
            *cp = v;
          }
        }
    }
  }
}
}  // namespace tg

typedef CUresult (*PFN_encodeTiled_g)(CUtensorMap*, CUtensorMapDataType, cuuint32_t, void*, const cuuint64_t*,
                                      const cuuint64_t*, const cuuint32_t*, const cuuint32_t*, CUtensorMapInterleave,
                                      CUtensorMapSwizzle, CUtensorMapL2promotion, CUtensorMapFloatOOBfill);
PFN_encodeTiled_g encode_fn() {
  static PFN_encodeTiled_g fn = nullptr;
  if (!fn) {
    void* q = nullptr;
    cudaDriverEntryPointQueryResult r;
    if (cudaGetDriverEntryPoint("cuTensorMapEncodeTiled", &q, cudaEnableDefault, &r) == cudaSuccess &&
        r == cudaDriverEntryPointSuccess)
      fn = (PFN_encodeTiled_g)q;
  }
  return fn;
}

// The TMA GEMM when it applies (op(A) = A; 16-byte aligned bases, even leading dimensions): true if
// launched.  GLS_DGEMM_TMA=0 turns it off (A/B diagnostics).
bool try_tma(cudaStream_t s, int64_t M, int64_t N, int64_t K, double alpha, const double* A, int64_t lda, char opA,
             const double* B, int64_t ldb, char opB, double beta, double* C, int64_t ldc, int flags, int max_ctas) {
  static const int on = getenv("GLS_DGEMM_TMA") ? atoi(getenv("GLS_DGEMM_TMA")) : 1;
  if (!on || opA != 'N' || K <= 0) return false;
  if ((((uintptr_t)A | (uintptr_t)B) & 15) || (lda & 1) || (ldb & 1)) return false;
  if (M > INT32_MAX || N > INT32_MAX || K > INT32_MAX) return false;
  PFN_encodeTiled_g enc = encode_fn();
  if (!enc) return false;
  const bool bt = opB == 'T';
  CUtensorMap am, bm;
  const cuuint32_t estr[2] = {1, 1};
  {
    cuuint64_t dim[2] = {(cuuint64_t)M, (cuuint64_t)K};
    cuuint64_t str[1] = {(cuuint64_t)lda * 8};
    cuuint32_t box[2] = {(cuuint32_t)tg::BM, (cuuint32_t)tg::BK};
    if (enc(&am, CU_TENSOR_MAP_DATA_TYPE_FLOAT64, 2, (void*)A, dim, str, box, estr, CU_TENSOR_MAP_INTERLEAVE_NONE,
            CU_TENSOR_MAP_SWIZZLE_NONE, CU_TENSOR_MAP_L2_PROMOTION_L2_256B, CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE) !=
        CUDA_SUCCESS)
      return false;
  }
  {
    cuuint64_t dim[2], str[1] = {(cuuint64_t)ldb * 8};
    cuuint32_t box[2];
    CUtensorMapSwizzle sw;
    if (bt) {  // B stored N x K (n contiguous)
      dim[0] = (cuuint64_t)N;
      dim[1] = (cuuint64_t)K;
      box[0] = tg::BN;
      box[1] = tg::BK;
      sw = CU_TENSOR_MAP_SWIZZLE_NONE;
    } else {   // B stored K x N (k contiguous)
      dim[0] = (cuuint64_t)K;
      dim[1] = (cuuint64_t)N;
      box[0] = tg::BK;
      box[1] = tg::BN;
      sw = CU_TENSOR_MAP_SWIZZLE_128B;
    }
    if (enc(&bm, CU_TENSOR_MAP_DATA_TYPE_FLOAT64, 2, (void*)B, dim, str, box, estr, CU_TENSOR_MAP_INTERLEAVE_NONE, sw,
            CU_TENSOR_MAP_L2_PROMOTION_L2_256B, CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE) != CUDA_SUCCESS)
      return false;
  }
  tg::Params p;
  p.M = M;
  p.N = N;
  p.K = K;
  p.C = C;
  p.ldc = ldc;
  p.alpha = alpha;
  p.beta = beta;
  p.flags = flags;
  p.tm = (M + tg::BM - 1) / tg::BM;
  p.tn = (N + tg::BN - 1) / tg::BN;
  p.ntiles = p.tm * p.tn;
  // tile order: longest K range first (the flags the recursion uses come alone; anything else keeps
  // the natural order)
  static const int sched = getenv("GLS_DGEMM_SCHED") ? atoi(getenv("GLS_DGEMM_SCHED")) : 1;
  p.order = tg::ORD_NATURAL;
  p.nvalid = p.ntiles;
  p.snake = 0;
  if (flags == GEMM_LOWER_C) {
    p.order = tg::ORD_LOWER;
    p.nvalid = 0;
    for (int64_t i = 0; i < p.tm; ++i) p.nvalid += std::min<int64_t>(p.tn, ((i + 1) * tg::BM + tg::BN - 1) / tg::BN);
  } else if (sched) {
    if (flags == GEMM_KMAX_COL) p.order = tg::ORD_COL_DESC;
    else if (flags == GEMM_KMIN_COL) p.order = tg::ORD_COL_ASC;
    else if (flags == GEMM_KMAX_ROW) p.order = tg::ORD_ROW_DESC;
  }
  if (sched) p.snake = p.order != tg::ORD_NATURAL && p.order != tg::ORD_LOWER ? 1 : 0;
  if (!sched && flags == GEMM_LOWER_C) {  // A/B: the round-1 walk (skipped tiles stay in the round-robin)
    p.order = tg::ORD_NATURAL;
    p.nvalid = p.ntiles;
  }
  int dev = 0, sms = 148;
  cudaGetDevice(&dev);
  cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev);
  int64_t grid = max_ctas > 0 ? std::max(1, max_ctas / 2) : sms;  // one CTA per SM (max_ctas counts two per SM)
  if (grid > p.nvalid) grid = p.nvalid;
  if (bt) {
    if (first_use_on_device((const void*)tg::dgemm_tma_kernel<true>))
      cudaFuncSetAttribute(tg::dgemm_tma_kernel<true>, cudaFuncAttributeMaxDynamicSharedMemorySize, tg::SMEM);
    tg::dgemm_tma_kernel<true><<<(unsigned)grid, tg::THREADS, tg::SMEM, s>>>(am, bm, p);
  } else {
    if (first_use_on_device((const void*)tg::dgemm_tma_kernel<false>))
      cudaFuncSetAttribute(tg::dgemm_tma_kernel<false>, cudaFuncAttributeMaxDynamicSharedMemorySize, tg::SMEM);
    tg::dgemm_tma_kernel<false><<<(unsigned)grid, tg::THREADS, tg::SMEM, s>>>(am, bm, p);
  }
  return true;
}

// ---------------------------------------------------------------- small products (latency)
// The recursion's deep levels multiply blocks of a few hundred rows: 128 x 64 tiles leave most SMs
// idle and split-K adds a reduction launch (~20 us per product on the critical path).  Here a CTA
// computes a 32 x 32 output tile; its 8 warps are 2 (16-row halves) x 4 (k-steps of each 16-wide K
// slice), each with eight 8 x 8 DMMA accumulators, and the four partial tiles are summed in a fixed
// order through shared memory at the end (deterministic).  Operands are staged by cp.async in a
// 3-stage ring of [32 rows][BK = 16 (+4 pad)] tiles (conflict-free fragment loads).  op(A) = A only.
namespace sg {
constexpr int BM = 32, BN = 32, BK = 16, LDK = BK + 4, STAGES = 3, THREADS = 256;
constexpr int A_T = BM * LDK, B_T = BN * LDK;
constexpr int SMEM_DOUBLES = (STAGES * (A_T + B_T) > 4 * BM * BN) ? STAGES * (A_T + B_T) : 4 * BM * BN;
}  // namespace sg

template <bool TB>
__global__ void __launch_bounds__(sg::THREADS) dgemm_small_kernel(GemmParams p) {
  constexpr int BM = sg::BM, BN = sg::BN, BK = sg::BK, LDK = sg::LDK, STAGES = sg::STAGES, THREADS = sg::THREADS,
                A_T = sg::A_T, B_T = sg::B_T, SMEM_DOUBLES = sg::SMEM_DOUBLES;
  __shared__ __align__(16) double sm[SMEM_DOUBLES];
  double* As = sm;
  double* Bs = sm + STAGES * A_T;
  const int64_t tm = (p.M + BM - 1) / BM;
  const int64_t tile = blockIdx.x;
  const int64_t r0 = (tile % tm) * BM, c0 = (tile / tm) * BN;
  if ((p.flags & GEMM_LOWER_C) && c0 >= r0 + BM) return;
  int64_t kb = 0, ke = p.K;
  if (p.flags & GEMM_KMIN_COL) kb = c0;
  if (p.flags & GEMM_KMAX_ROW) ke = min(ke, r0 + BM);
  if (p.flags & GEMM_KMAX_COL) ke = min(ke, c0 + BN);
  const int64_t kbeg = kb;
  kb = (kb / BK) * BK;
  const int nk = (ke > kb) ? (int)((ke - kb + BK - 1) / BK) : 0;
  const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
  const int wm = warp & 1, wk = warp >> 1;  // rows [16 wm, 16 wm + 16), k-step wk of each BK slice
  const int g = lane >> 2, t = lane & 3;
  auto issue = [&](int kt, int stg) {
    const int64_t k0 = kb + (int64_t)kt * BK;
    double* as = As + stg * A_T;
    double* bs = Bs + stg * B_T;
#pragma unroll
    for (int j = 0; j < (BM * BK) / THREADS; ++j) {  // 2
      const int idx = tid + j * THREADS;
      const int m = idx % BM, k = idx / BM;
      const int64_t gm = r0 + m, gk = k0 + k;
      const bool v = gm < p.M && gk < ke && gk >= kbeg;
      cp_async8(as + m * LDK + k, v ? p.A + gm + gk * p.lda : p.A, v);
    }
#pragma unroll
    for (int j = 0; j < (BN * BK) / THREADS; ++j) {  // 2
      const int idx = tid + j * THREADS;
      int n, k;
      if (!TB) { k = idx % BK; n = idx / BK; } else { n = idx % BN; k = idx / BN; }
      const int64_t gn = c0 + n, gk = k0 + k;
      const bool v = gn < p.N && gk < ke && gk >= kbeg;
      cp_async8(bs + n * LDK + k, v ? (TB ? p.B + gn + gk * p.ldb : p.B + gk + gn * p.ldb) : p.B, v);
    }
  };
  double acc[2][4][2];
#pragma unroll
  for (int a = 0; a < 2; ++a)
#pragma unroll
    for (int b = 0; b < 4; ++b) acc[a][b][0] = acc[a][b][1] = 0.0;
#pragma unroll
  for (int s = 0; s < STAGES - 1; ++s) {
    if (s < nk) issue(s, s);
    cp_async_commit();
  }
  for (int kt = 0; kt < nk; ++kt) {
    cp_async_wait<STAGES - 2>();
    __syncthreads();
    const int nxt = kt + STAGES - 1;
    if (nxt < nk) issue(nxt, nxt % STAGES);
    cp_async_commit();
    const double* as = As + (kt % STAGES) * A_T + (16 * wm + g) * LDK + 4 * wk + t;
    const double* bs = Bs + (kt % STAGES) * B_T + g * LDK + 4 * wk + t;
    double a[2], b[4];
#pragma unroll
    for (int i = 0; i < 2; ++i) a[i] = as[8 * i * LDK];
#pragma unroll
    for (int j = 0; j < 4; ++j) b[j] = bs[8 * j * LDK];
#pragma unroll
    for (int i = 0; i < 2; ++i)
#pragma unroll
      for (int j = 0; j < 4; ++j) dmma(acc[i][j], a[i], b[j]);
  }
  cp_async_wait<0>();
  __syncthreads();
  // partial tiles of the four k-step groups -> shared memory, summed in the order wk = 0, 1, 2, 3
  double* red = sm;  // [wk][n][m] (32 x 32 per group)
#pragma unroll
  for (int i = 0; i < 2; ++i)
#pragma unroll
    for (int j = 0; j < 4; ++j)
#pragma unroll
      for (int e = 0; e < 2; ++e) red[wk * BM * BN + (8 * j + 2 * t + e) * BM + 16 * wm + 8 * i + g] = acc[i][j][e];
  __syncthreads();
  for (int o = tid; o < BM * BN; o += THREADS) {
    const int m = o % BM, n = o / BM;
    const int64_t gm = r0 + m, gn = c0 + n;
    if (gm < p.M && gn < p.N) {
      const double v = ((red[o] + red[BM * BN + o]) + red[2 * BM * BN + o]) + red[3 * BM * BN + o];
      double* cp = p.C + gm + gn * p.ldc;
      double r = p.alpha * v;
      if (p.beta != 0.0) r += p.beta * *cp;
      *cp = r;
    }
  }
}

template <bool TA, bool TB>
void launch(cudaStream_t s, dim3 grid, const GemmParams& p) {
  if (first_use_on_device((const void*)dgemm_kernel<TA, TB>))
    cudaFuncSetAttribute(dgemm_kernel<TA, TB>, cudaFuncAttributeMaxDynamicSharedMemorySize, SMEM_BYTES);
  dgemm_kernel<TA, TB><<<grid, THREADS, SMEM_BYTES, s>>>(p);
}

// ---------------------------------------------------------------- skinny products with T
// W = T B (T n x n lower triangular, B n x k, k <= 21): memory-bound (T read once).  Grid = row
// blocks of 128 x K segments; thread = one row, reading T column-major (a warp reads 32 consecutive
// rows of one column); partial sums per segment, reduced in a fixed order (deterministic).
constexpr int kSkinnySeg = 32;
__global__ void trmm_skinny_partial(int64_t n, int k, const double* __restrict__ T, int64_t ldt,
                                    const double* __restrict__ B, int64_t ldb, double* __restrict__ part) {
  const int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  const int seg = blockIdx.y;
  const int64_t span = (n + kSkinnySeg - 1) / kSkinnySeg;
  const int64_t j0 = seg * span, j1 = (j0 + span < n) ? j0 + span : n;
  double acc[21];
#pragma unroll
  for (int w = 0; w < 21; ++w) acc[w] = 0.0;
  if (i < n) {
    const int64_t jend = (i + 1 < j1) ? i + 1 : j1;  // lower triangular: j <= i
#pragma unroll 8
    for (int64_t j = j0; j < jend; ++j) {
      const double t = T[i + j * ldt];
#pragma unroll
      for (int w = 0; w < 21; ++w)
        if (w < k) acc[w] = fma(t, __ldg(B + j + w * ldb), acc[w]);
    }
#pragma unroll
    for (int w = 0; w < 21; ++w)
      if (w < k) part[((int64_t)seg * k + w) * n + i] = acc[w];
  }
}
__global__ void trmm_skinny_reduce(int64_t n, int k, const double* __restrict__ part, double* __restrict__ W,
                                   int64_t ldw) {
  for (int64_t o = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; o < n * k; o += (int64_t)gridDim.x * blockDim.x) {
    const int64_t i = o % n;
    const int w = (int)(o / n);
    double v = 0.0;
    for (int seg = 0; seg < kSkinnySeg; ++seg) v += part[((int64_t)seg * k + w) * n + i];
    W[i + w * ldw] = v;
  }
}
// V = T^T W (V[j, w] = sum_{i >= j} T[i, j] W[i, w]): one warp per column j of T (contiguous),
// lanes stride over i, fixed-order shuffle reduction.
__global__ void trmm_t_skinny(int64_t n, int k, const double* __restrict__ T, int64_t ldt,
                              const double* __restrict__ W, int64_t ldw, double* __restrict__ V, int64_t ldv) {
  const int lane = threadIdx.x & 31;
  for (int64_t j = ((int64_t)blockIdx.x * blockDim.x + threadIdx.x) >> 5; j < n;
       j += ((int64_t)gridDim.x * blockDim.x) >> 5) {
    double acc[21];
#pragma unroll
    for (int w = 0; w < 21; ++w) acc[w] = 0.0;
#pragma unroll 8
    for (int64_t i = j + lane; i < n; i += 32) {
      const double t = T[i + j * ldt];
#pragma unroll
      for (int w = 0; w < 21; ++w)
        if (w < k) acc[w] = fma(t, __ldg(W + i + w * ldw), acc[w]);
    }
#pragma unroll
    for (int w = 0; w < 21; ++w) {
      if (w < k) {
        double v = acc[w];
#pragma unroll
        for (int o = 16; o > 0; o >>= 1) v += __shfl_xor_sync(0xffffffffu, v, o);
        if (lane == 0) V[j + w * ldv] = v;
      }
    }
  }
}

}  // namespace

void trmm_lower_skinny(cudaStream_t s, int64_t n, int k, const double* T, int64_t ldt, const double* B,
                       int64_t ldb, double* W, int64_t ldw, double* part, int64_t* lc) {
  dim3 grid((unsigned)((n + 127) / 128), kSkinnySeg);
  trmm_skinny_partial<<<grid, 128, 0, s>>>(n, k, T, ldt, B, ldb, part);
  const int64_t tot = n * k;
  trmm_skinny_reduce<<<(unsigned)((tot + 255) / 256 < 1024 ? (tot + 255) / 256 : 1024), 256, 0, s>>>(n, k, part, W,
                                                                                                      ldw);
  if (lc) *lc += 2;
}

void trmm_lower_t_skinny(cudaStream_t s, int64_t n, int k, const double* T, int64_t ldt, const double* W,
                         int64_t ldw, double* V, int64_t ldv, int64_t* lc) {
  int64_t blocks = (n * 32 + 255) / 256;
  if (blocks > 148 * 16) blocks = 148 * 16;
  trmm_t_skinny<<<(unsigned)blocks, 256, 0, s>>>(n, k, T, ldt, W, ldw, V, ldv);
  if (lc) ++*lc;
}

#ifdef GLS_AB_CUBLAS
}  // namespace gls
#include <cublas_v2.h>
namespace gls {
// A/B diagnostics only (build with -DGLS_AB_CUBLAS, run with GLS_DGEMM_CUBLAS=1): the same products
// through cuBLAS DGEMM (full K ranges, full C) to price the GEMM kernel's efficiency in gls_create.
static bool ab_cublas(cudaStream_t s, int64_t M, int64_t N, int64_t K, double alpha, const double* A, int64_t lda,
                      char opA, const double* B, int64_t ldb, char opB, double beta, double* C, int64_t ldc) {
  static const bool on = getenv("GLS_DGEMM_CUBLAS") != nullptr;
  if (!on) return false;
  static cublasHandle_t h[64] = {};
  int dev = 0;
  cudaGetDevice(&dev);
  if (!h[dev]) cublasCreate(&h[dev]);
  cublasSetStream(h[dev], s);
  cublasDgemm(h[dev], opA == 'T' ? CUBLAS_OP_T : CUBLAS_OP_N, opB == 'T' ? CUBLAS_OP_T : CUBLAS_OP_N, (int)M, (int)N,
              (int)K, &alpha, A, (int)lda, B, (int)ldb, &beta, C, (int)ldc);
  return true;
}
#endif

void dgemm(cudaStream_t s, int64_t M, int64_t N, int64_t K, double alpha, const double* A,
           int64_t lda, char opA, const double* B, int64_t ldb, char opB, double beta, double* C,
           int64_t ldc, int flags, int64_t* launch_counter, double* ws, int max_ctas) {
  if (M <= 0 || N <= 0) return;
#ifdef GLS_AB_CUBLAS
  if (ab_cublas(s, M, N, K, alpha, A, lda, opA, B, ldb, opB, beta, C, ldc)) {
    if (launch_counter) ++*launch_counter;
    return;
  }
#endif
  GemmParams p{M, N, K, A, lda, B, ldb, C, ldc, alpha, beta, flags, 1, nullptr};
  static const bool trace = getenv("GLS_TRACE_GEMM") != nullptr;  // diagnostics: one line per product
  if (trace)
    fprintf(stderr, "[gemm] %lld %lld %lld %c%c flags %d stream %p cap %d\n", (long long)M, (long long)N,
            (long long)K, opA, opB, flags, (void*)s, max_ctas);
  dim3 grid((unsigned)((M + BM - 1) / BM), (unsigned)((N + BN - 1) / BN));
  const int64_t tiles = (int64_t)grid.x * grid.y;
  const int64_t ktiles = (K + BK - 1) / BK;
  // small output: 32 x 32 tiles, no split-K launch (GLS_DGEMM_SMALL=0 restores the split-K path)
  static const bool small_on = !(getenv("GLS_DGEMM_SMALL") && atoi(getenv("GLS_DGEMM_SMALL")) == 0);
  if (small_on && opA == 'N' && tiles < 74 && max_ctas <= 0) {
    const int64_t st = ((M + sg::BM - 1) / sg::BM) * ((N + sg::BN - 1) / sg::BN);
    if (opB == 'T') dgemm_small_kernel<true><<<(unsigned)st, sg::THREADS, 0, s>>>(p);
    else dgemm_small_kernel<false><<<(unsigned)st, sg::THREADS, 0, s>>>(p);
    if (launch_counter) ++*launch_counter;
    return;
  }
  // small output, long K: split K so the launch fills the machine (the recursion's deep levels)
  if (tiles < 74 && ktiles >= 8) {
    int sp = (int)((148 + tiles - 1) / tiles);
    if (sp > ktiles / 4) sp = (int)(ktiles / 4);
    if (sp > 16) sp = 16;
    if (sp > 1 && ws && (size_t)sp * M * N <= kSplitKWsDoubles) {
      p.nsplit = sp;
      p.ws = ws;
      grid.z = sp;
    }
  }
  if (p.nsplit == 1 && try_tma(s, M, N, K, alpha, A, lda, opA, B, ldb, opB, beta, C, ldc, flags, max_ctas)) {
    if (launch_counter) ++*launch_counter;
    return;
  }
  if (max_ctas > 0 && p.nsplit == 1 && tiles > max_ctas) grid = dim3((unsigned)max_ctas);
  const bool ta = (opA == 'T'), tb = (opB == 'T');
  if (!ta && !tb) launch<false, false>(s, grid, p);
  else if (!ta && tb) launch<false, true>(s, grid, p);
  else if (ta && !tb) launch<true, false>(s, grid, p);
  else launch<true, true>(s, grid, p);
  if (launch_counter) ++*launch_counter;
  if (p.nsplit > 1) {
    const int64_t tot = M * N;
    int64_t blocks = (tot + 255) / 256;
    if (blocks > 1024) blocks = 1024;
    dgemm_splitk_reduce<<<(unsigned)blocks, 256, 0, s>>>(p);
    if (launch_counter) ++*launch_counter;
  }
}

}  // namespace gls
