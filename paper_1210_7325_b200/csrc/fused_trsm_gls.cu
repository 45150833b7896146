// fused_trsm_gls.cu -- the hot path: Alg. 5 line 3 fused with lines 7-11 (
// Alg. 8 lines 9-14) for one block of SNP columns.
//
// For a panel of SNP columns x (one CTA at a time, persistent over panels) and each row block i
// of nb = 128 rows:
//
//     z_i  = sum_{j <= i} T_ij x_j                 T = L^{-1}, so z = L^{-1} x = X~_R  (trsm)
//     acc_W += z_i^T W_i,  W = [X~_L | y~]         -> S_BL_i (pL values), b_B_i        (gemv, dot)
//     acc_G += z_i^T z_i (group diagonal blocks)   -> S_BR_i                             (dot)
//
// z_i lives only in registers: it is produced by DMMA as the accumulator of z^T = X^T T^T and fed
// straight back into DMMA as the A (and B) operand of the two reductions -- the m8n8k4 accumulator
// layout is a valid operand layout under a K permutation -- so X~_R never touches memory
// ("X~_R never returns to HBM", BASELINE.json north_star).  After the last row block the four
// warp slices are summed in a fixed order, S_i = [[S_TL, S_BL^T], [S_BL, S_BR]] and [b_T; b_B]
// are assembled (Fig. 1, full y~ in both halves -- reading A1) and solved by
// Cholesky (posv, Alg. 5 line 11) with the rank rule of reading A4, one lane per problem.
//
// Pipeline: warp 8 is a TMA producer (one elected lane): per stage a 16 KiB packed-T tile
// (cp.async.bulk) and a 16-row x 64-column X tile (cp.async.bulk.tensor.2d, 128B swizzle,
// out-of-bounds rows/columns zero-filled) land in shared memory under a full/empty mbarrier pair;
// warps 0-7 (2 column halves x 4 z-row slices, 32 x 32 each) issue mma.sync.m8n8k4.f64 (SASS
// DMMA.8x8x4, the B200 FP64 tensor pipe -- tcgen05 has no f64 kind).
#include <cuda.h>

#include <cstdio>

#include "gls_internal.cuh"

namespace gls {
namespace {

constexpr int kConsumerWarps = 8;
constexpr int kThreads = (kConsumerWarps + 1) * 32;
constexpr int kXStageBytes = kMaxPanelCols * kKT * 8;  // 8 KiB
constexpr int kTStageBytes = kTileDoubles * 8;         // 16 KiB

__device__ __forceinline__ uint32_t smem_u32(const void* p) {
  return (uint32_t)__cvta_generic_to_shared(p);
}
__device__ __forceinline__ void mbar_init(uint64_t* bar, uint32_t count) {
  asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;\n" ::"r"(smem_u32(bar)), "r"(count));
}
__device__ __forceinline__ void mbar_arrive_expect_tx(uint64_t* bar, uint32_t bytes) {
  asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;\n" ::"r"(smem_u32(bar)),
               "r"(bytes)
               : "memory");
}
__device__ __forceinline__ void mbar_arrive(uint64_t* bar) {
  asm volatile("mbarrier.arrive.shared::cta.b64 _, [%0];\n" ::"r"(smem_u32(bar)) : "memory");
}
__device__ __forceinline__ void mbar_wait(uint64_t* bar, uint32_t phase) {
  asm volatile(
      "{\n"
      ".reg .pred P1;\n"
      "WAIT_%=:\n"
      "mbarrier.try_wait.parity.shared::cta.b64 P1, [%0], %1;\n"
      "@!P1 bra WAIT_%=;\n"
      "}\n" ::"r"(smem_u32(bar)),
      "r"(phase)
      : "memory");
}
__device__ __forceinline__ void bulk_g2s(void* dst, const void* src, uint32_t bytes, uint64_t* bar) {
  asm volatile(
      "cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];\n" ::"r"(
          smem_u32(dst)),
      "l"(src), "r"(bytes), "r"(smem_u32(bar))
      : "memory");
}
__device__ __forceinline__ void tma_2d_g2s(void* dst, const CUtensorMap* map, int c0, int c1,
                                           uint64_t* bar) {
  asm volatile(
      "cp.async.bulk.tensor.2d.shared::cluster.global.tile.mbarrier::complete_tx::bytes [%0], [%1, {%2, %3}], "
      "[%4];\n" ::"r"(smem_u32(dst)),
      "l"(map), "r"(c0), "r"(c1), "r"(smem_u32(bar))
      : "memory");
}
__device__ __forceinline__ void named_bar_sync(int id, int count) {
  asm volatile("bar.sync %0, %1;\n" ::"r"(id), "r"(count) : "memory");
}
__device__ __forceinline__ void dmma(double (&c)[2], double a, double b) {
  asm volatile("mma.sync.aligned.m8n8k4.row.col.f64.f64.f64.f64 {%0,%1}, {%2}, {%3}, {%0,%1};\n"
               : "+d"(c[0]), "+d"(c[1])
               : "d"(a), "d"(b));
}

struct KParams {
  const double* Tpk;
  const double* Wpk;
  const double* G;  // (pL+1)^2, column-major, ld = pL+1
  double* b_out;
  int32_t* status_out;
  const int* gate;  // nullable: when set, run only if *gate != 0 (int8 path rejected the block)
  const int* pflag;  // nullable: solve and store only problems g with pflag[g] != 0; skip other panels
  const int* m_dev;  // nullable: only the first min(m_blk, *m_dev) problems (a compacted block)
  int gate_lo, gate_hi;  // with gate: run only if gate_lo < *gate <= gate_hi
  unsigned long long* ran;  // nullable: block 0 adds 1 when the kernel does its work
  int64_t m_blk;
  int64_t num_panels;
  int NB;
  int pad;  // n_pad - n: virtual rows [0, pad) are zero padding at the TOP
  int kt0;  // first K tile that is not all padding = pad / 16
  int pL, pR, p;
  int gw, cpw, cpp, gpp;
};

template <int NW, bool FULL>
struct KCfg {
  static constexpr int NG = FULL ? 10 : 4;  // Gram tiles per warp
  static constexpr int kWBytes = 1024 * NW * 8;  // packed W per row block
  static constexpr int kRedDoubles = (4 * NW + NG) * 64;
  // as many 24 KiB stages as fit next to the W double buffer and the reduction scratch (<= 8)
  static constexpr int kSmemCap = 232448 - 1024 - 256;
  static constexpr int kFixed = 2 * kWBytes + 2 * kRedDoubles * 8;
  static constexpr int kFit = (kSmemCap - kFixed) / (kXStageBytes + kTStageBytes);
  static constexpr int STAGES = kFit < 8 ? kFit : 8;
  static_assert(STAGES >= 3, "shared memory budget");
  static constexpr uint32_t off_X = 0;
  static constexpr uint32_t off_T = off_X + STAGES * kXStageBytes;
  static constexpr uint32_t off_W = off_T + STAGES * kTStageBytes;
  static constexpr uint32_t off_R = off_W + 2 * kWBytes;
  static constexpr uint32_t off_B = off_R + 2 * kRedDoubles * 8;
  static constexpr uint32_t bytes = off_B + (2 * STAGES + 2) * 8 + 1024;  // + alignment slack
};

// Pair index of Gram tile (t, t2), t <= t2 < 4, for FULL mode.
__host__ __device__ constexpr int gram_pair(int t, int t2) {
  return t * 4 - (t * (t - 1)) / 2 + (t2 - t);  // rows: t=0 -> 0..3, t=1 -> 4..6, t=2 -> 7..8, t=3 -> 9
}

__device__ __forceinline__ void lds128(uint32_t addr, double& x, double& y) {
  asm volatile("ld.shared.v2.f64 {%0, %1}, [%2];\n" : "=d"(x), "=d"(y) : "r"(addr));
}

// One stage's operand fragments for one P half (K rows 4kk+2P, 4kk+2P+1 of the 16-row tile).
struct Frag {
  double a[4][2];  // X^T: 4 column tiles t
  double b[4][2];  // T^T: 4 z-row subtiles s
};

template <bool ALIGNED>
__device__ __forceinline__ void load_frag(Frag& f, uint32_t xs, uint32_t ts, const uint32_t (&xoff)[4][2],
                                          uint32_t toff0, int P) {
#pragma unroll
  for (int t = 0; t < 4; ++t) {
    const uint32_t o = ALIGNED ? xoff[0][P] + t * 1024 : xoff[t][P];
    lds128(xs + o, f.a[t][0], f.a[t][1]);
  }
#pragma unroll
  for (int s = 0; s < 4; ++s) lds128(ts + toff0 + s * 1024 + P * 512, f.b[s][0], f.b[s][1]);
}

__device__ __forceinline__ void mma_frag(double (&acc)[4][4][2], const Frag& f) {
#pragma unroll
  for (int e = 0; e < 2; ++e)
#pragma unroll
    for (int t = 0; t < 4; ++t)
#pragma unroll
      for (int s = 0; s < 4; ++s) dmma(acc[t][s], f.a[t][e], f.b[s][e]);
}

// Per-problem path choice: a panel without a flagged problem is left to the int8 kernel (the producer and
// every consumer decide alike from the same flags, so their stage counters stay in step).
__device__ __forceinline__ bool panel_wanted(const KParams& kp, int64_t panel, int64_t m_eff) {
  if (panel * kp.gpp >= m_eff) return false;
  if (!kp.pflag) return true;
  const int64_t g1 = (panel + 1) * kp.gpp < kp.m_blk ? (panel + 1) * kp.gpp : kp.m_blk;
  for (int64_t g = panel * kp.gpp; g < g1; ++g)
    if (kp.pflag[g]) return true;
  return false;
}

template <int NW, bool FULL, bool ALIGNED>
__global__ void __launch_bounds__(kThreads, 1)
    fused_trsm_gls_kernel(const __grid_constant__ CUtensorMap xmap, const KParams kp) {
  if (kp.gate) {  // uniform across the grid
    const int g = *(volatile const int*)kp.gate;
    if (g <= kp.gate_lo || g > kp.gate_hi) return;
  }
  const int64_t m_eff = kp.m_dev && *(volatile const int*)kp.m_dev < kp.m_blk ? *(volatile const int*)kp.m_dev
                                                                              : kp.m_blk;
  if (kp.ran && blockIdx.x == 0 && threadIdx.x == 0) atomicAdd(kp.ran, 1ull);
  using C = KCfg<NW, FULL>;
  extern __shared__ uint8_t smem_raw[];
  // 1024-byte alignment for the 128B-swizzled TMA destination, in the shared window
  const uint32_t sbase = (smem_u32(smem_raw) + 1023u) & ~1023u;
  uint8_t* smem = smem_raw + (sbase - smem_u32(smem_raw));
  const uint32_t sX = sbase + C::off_X;
  const uint32_t sT = sbase + C::off_T;
  double* sW = (double*)(smem + C::off_W);
  double* sR = (double*)(smem + C::off_R);
  uint64_t* full = (uint64_t*)(smem + C::off_B);
  uint64_t* empty = full + C::STAGES;
  uint64_t* wempty = empty + C::STAGES;  // W double buffer: consumers release after the epilogue

  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  if (threadIdx.x == 0) {
    for (int s = 0; s < C::STAGES; ++s) {
      mbar_init(&full[s], 1);
      mbar_init(&empty[s], kConsumerWarps);
    }
    mbar_init(&wempty[0], kConsumerWarps);
    mbar_init(&wempty[1], kConsumerWarps);
    asm volatile("fence.mbarrier_init.release.cluster;\n" ::: "memory");
  }
  __syncthreads();

  const int NB = kp.NB;
  const int kt0 = kp.kt0;
  if (warp == kConsumerWarps) {
    // ------------------------------------------------------------------ TMA producer
    if (lane == 0) {
      asm volatile("prefetch.tensormap [%0];\n" ::"l"(&xmap) : "memory");
      int st = 0;
      uint32_t ph = 0;
      uint32_t rbc = 0;  // running row-block counter (W buffer = rbc & 1, its use = rbc >> 1)
      const uint32_t xbytes = (uint32_t)(kKT * kp.cpp * 8);
      for (int64_t panel = blockIdx.x; panel < kp.num_panels; panel += gridDim.x) {
        if (!panel_wanted(kp, panel, m_eff)) continue;
        const int col0 = (int)(panel * kp.cpp);
        for (int i = 0; i < NB; ++i, ++rbc) {
          const double* Trb = kp.Tpk + tpk_tile_offset(i) * kTileDoubles;
          const int nkt = (i + 1) * kKTPerRB;
          for (int kt = kt0; kt < nkt; ++kt) {
            mbar_wait(&empty[st], ph ^ 1);
            const bool first = (kt == kt0);
            if (first) mbar_wait(&wempty[rbc & 1], ((rbc >> 1) & 1) ^ 1);
            const uint32_t bytes = kTStageBytes + xbytes + (first ? C::kWBytes : 0);
            mbar_arrive_expect_tx(&full[st], bytes);
            bulk_g2s(smem + C::off_T + (size_t)st * kTStageBytes, Trb + (size_t)kt * kTileDoubles,
                     kTStageBytes, &full[st]);
            // virtual row kt*16 is real row kt*16 - pad; negative rows are zero-filled by TMA
            tma_2d_g2s(smem + C::off_X + (size_t)st * kXStageBytes, &xmap, kt * kKT - kp.pad, col0,
                       &full[st]);
            if (first)
              bulk_g2s(sW + (size_t)(rbc & 1) * (C::kWBytes / 8), kp.Wpk + (size_t)i * (C::kWBytes / 8),
                       C::kWBytes, &full[st]);
            if (++st == C::STAGES) {
              st = 0;
              ph ^= 1;
            }
          }
        }
      }
    }
    return;
  }

  // ------------------------------------------------------------------ DMMA consumers
  // warp -> (column half mw, z-row slice ns).  Warp w issues on SM sub-partition w % 4; slices are
  // paired {0,3} on SMSPs 0-1 and {1,2} on SMSPs 2-3 so that the skipped all-zero tiles of the
  // diagonal block (slice ns needs only its first 2ns+2 K tiles there) save the same time on every
  // SMSP: 10 of 16 tile-units instead of 16.
  const int smsp = warp & 3, half = warp >> 2;
  const int mw = smsp & 1;                                             // column half
  const int ns = (smsp < 2) ? (half ? 3 : 0) : (half ? 2 : 1);         // z-row slice (32 rows)
  const int diag_keep = 2 * ns + 1;  // last useful K tile (within the diagonal block) of this slice
  const int kk = lane & 3, l4 = lane >> 2;

  // X^T fragment addresses: smem row = panel-local column, 16-byte chunk c = 2kk+P holds K rows
  // 2c, 2c+1; TMA SWIZZLE_128B stores chunk c of row r at chunk position c ^ (r & 7).
  uint32_t xoff[4][2];
#pragma unroll
  for (int t = 0; t < 4; ++t) {
    int lc = t * 8 + l4;
    if (lc >= kp.cpw) lc = kp.cpw - 1;  // padding lanes duplicate a valid column (results unused)
    const int row = mw * kp.cpw + lc;
#pragma unroll
    for (int P = 0; P < 2; ++P) xoff[t][P] = row * 128 + (((2 * kk + P) ^ (row & 7)) << 4);
  }
  // T^T fragment address in the packed tile: [subtile g = ns*4+s][P][lane][2 doubles]
  const uint32_t toff0 = (uint32_t)((ns * 4 * 2 * 32 + lane) * 16);

  double acc[4][4][2];
  double accW[4][NW][2];
  double accG[C::NG][2];
#pragma unroll
  for (int t = 0; t < 4; ++t)
#pragma unroll
    for (int w = 0; w < NW; ++w) accW[t][w][0] = accW[t][w][1] = 0.0;
#pragma unroll
  for (int g = 0; g < C::NG; ++g) accG[g][0] = accG[g][1] = 0.0;

  int st = 0;
  uint32_t ph = 0;
  uint32_t rbc = 0;
  Frag F0, F1;
  for (int64_t panel = blockIdx.x; panel < kp.num_panels; panel += gridDim.x) {
    if (!panel_wanted(kp, panel, m_eff)) continue;
    for (int i = 0; i < NB; ++i, ++rbc) {
#pragma unroll
      for (int t = 0; t < 4; ++t)
#pragma unroll
        for (int s = 0; s < 4; ++s) acc[t][s][0] = acc[t][s][1] = 0.0;
      const int nkt = (i + 1) * kKTPerRB;
      // software pipeline: the P=0 fragments of stage k+1 are loaded while stage k's P=1 DMMAs run
      mbar_wait(&full[st], ph);
      load_frag<ALIGNED>(F0, sX + st * kXStageBytes, sT + st * kTStageBytes, xoff, toff0, 0);
      for (int kt = kt0; kt < nkt; ++kt) {
        // all-zero T tile for this slice (strictly above the diagonal of T_ii): loads and barriers
        // stay in lock step, the DMMAs are skipped
        const bool active = (kt - 8 * i) <= diag_keep;
        load_frag<ALIGNED>(F1, sX + st * kXStageBytes, sT + st * kTStageBytes, xoff, toff0, 1);
        if (active) mma_frag(acc, F0);
        const int cur = st;
        if (++st == C::STAGES) {
          st = 0;
          ph ^= 1;
        }
        if (kt + 1 < nkt) {
          mbar_wait(&full[st], ph);
          load_frag<ALIGNED>(F0, sX + st * kXStageBytes, sT + st * kTStageBytes, xoff, toff0, 0);
        }
        if (active) mma_frag(acc, F1);
        __syncwarp();
        if (lane == 0) mbar_arrive(&empty[cur]);
      }
      // ---- row-block epilogue: reductions of z_i on the tensor pipe (z_i stays in registers)
      const double* wb = sW + (size_t)(rbc & 1) * (C::kWBytes / 8);
#pragma unroll
      for (int w = 0; w < NW; ++w)
#pragma unroll
        for (int s = 0; s < 4; ++s) {
          const double2 wf = *(const double2*)(wb + ((((ns * NW + w) * 4 + s) * 32 + lane) * 2));
#pragma unroll
          for (int t = 0; t < 4; ++t) {
            dmma(accW[t][w], acc[t][s][0], wf.x);
            dmma(accW[t][w], acc[t][s][1], wf.y);
          }
        }
      __syncwarp();
      if (lane == 0) mbar_arrive(&wempty[rbc & 1]);
      if (!FULL) {
#pragma unroll
        for (int t = 0; t < 4; ++t)
#pragma unroll
          for (int s = 0; s < 4; ++s) {
            dmma(accG[t], acc[t][s][0], acc[t][s][0]);
            dmma(accG[t], acc[t][s][1], acc[t][s][1]);
          }
      } else {
#pragma unroll
        for (int t = 0; t < 4; ++t)
#pragma unroll
          for (int t2 = t; t2 < 4; ++t2)
#pragma unroll
            for (int s = 0; s < 4; ++s) {
              dmma(accG[gram_pair(t, t2)], acc[t][s][0], acc[t2][s][0]);
              dmma(accG[gram_pair(t, t2)], acc[t][s][1], acc[t2][s][1]);
            }
      }
    }

    // ---- panel epilogue: fixed-order sum over the 4 z-row slices, then per-problem solve
    double* red = sR + (size_t)mw * C::kRedDoubles;
    const int eidx = l4 * 8 + 2 * kk;  // C-tile element (m = l4, n = 2kk + e)
    named_bar_sync(1, kConsumerWarps * 32);
    for (int r = 0; r < 4; ++r) {
      if (ns == r) {
#pragma unroll
        for (int t = 0; t < 4; ++t)
#pragma unroll
          for (int w = 0; w < NW; ++w)
#pragma unroll
            for (int e = 0; e < 2; ++e) {
              double* q = red + (t * NW + w) * 64 + eidx + e;
              *q = (r == 0) ? accW[t][w][e] : *q + accW[t][w][e];
            }
#pragma unroll
        for (int g = 0; g < C::NG; ++g)
#pragma unroll
          for (int e = 0; e < 2; ++e) {
            double* q = red + (4 * NW + g) * 64 + eidx + e;
            *q = (r == 0) ? accG[g][e] : *q + accG[g][e];
          }
      }
      named_bar_sync(1, kConsumerWarps * 32);
    }
#pragma unroll
    for (int t = 0; t < 4; ++t)
#pragma unroll
      for (int w = 0; w < NW; ++w) accW[t][w][0] = accW[t][w][1] = 0.0;
#pragma unroll
    for (int g = 0; g < C::NG; ++g) accG[g][0] = accG[g][1] = 0.0;

    const int gl = threadIdx.x;  // one thread per problem of the panel
    const int64_t gidx = panel * kp.gpp + gl;
    if (gl < kp.gpp && gidx < m_eff && !(kp.pflag && !kp.pflag[gidx])) {
      const int pL = kp.pL, pR = kp.pR, p = kp.p;
      const int gmw = gl / kp.gw, gg = gl % kp.gw;
      const double* rd = sR + (size_t)gmw * C::kRedDoubles;
      double S[20 * 20];
      double rhs[20];
      const int ldg = pL + 1;
      for (int a = 0; a < pL; ++a) {
        for (int b = 0; b < pL; ++b) S[a + b * 20] = kp.G[a + b * ldg];
        rhs[a] = kp.G[a + pL * ldg];
      }
      for (int a = 0; a < pR; ++a) {
        const int c = gg * pR + a, t = c >> 3, m = c & 7;
        for (int k = 0; k <= pL; ++k) {
          const double v = rd[(t * NW + (k >> 3)) * 64 + m * 8 + (k & 7)];
          if (k < pL) {
            S[(pL + a) + k * 20] = v;
            S[k + (pL + a) * 20] = v;
          } else {
            rhs[pL + a] = v;
          }
        }
        for (int b = 0; b <= a; ++b) {
          const int c2 = gg * pR + b, t2 = c2 >> 3, m2 = c2 & 7;
          double v;
          if (!FULL) {
            v = rd[(4 * NW + t) * 64 + m * 8 + m2];
          } else {
            v = (t2 <= t) ? rd[(4 * NW + gram_pair(t2, t)) * 64 + m2 * 8 + m]
                          : rd[(4 * NW + gram_pair(t, t2)) * 64 + m * 8 + m2];
          }
          S[(pL + a) + (pL + b) * 20] = v;
          S[(pL + b) + (pL + a) * 20] = v;
        }
      }
      // posv: S = R R^T (lower, in place), rank rule pivot <= 1e-10 * S_jj (reading A4)
      int bad = 0;
      for (int j = 0; j < p && !bad; ++j) {
        const double sjj = S[j + j * 20];
        double d = sjj;
        for (int k = 0; k < j; ++k) d -= S[j + k * 20] * S[j + k * 20];
        if (!(d > 1e-10 * sjj)) {
          bad = 1;
          break;
        }
        const double r = sqrt(d);
        S[j + j * 20] = r;
        for (int i2 = j + 1; i2 < p; ++i2) {
          double v = S[i2 + j * 20];
          for (int k = 0; k < j; ++k) v -= S[i2 + k * 20] * S[j + k * 20];
          S[i2 + j * 20] = v / r;
        }
      }
      double* bo = kp.b_out + gidx * p;
      if (bad) {
        for (int j = 0; j < p; ++j) bo[j] = __longlong_as_double(0x7ff8000000000000LL);
      } else {
        for (int i2 = 0; i2 < p; ++i2) {
          double v = rhs[i2];
          for (int k = 0; k < i2; ++k) v -= S[i2 + k * 20] * rhs[k];
          rhs[i2] = v / S[i2 + i2 * 20];
        }
        for (int i2 = p - 1; i2 >= 0; --i2) {
          double v = rhs[i2];
          for (int k = i2 + 1; k < p; ++k) v -= S[k + i2 * 20] * rhs[k];
          rhs[i2] = v / S[i2 + i2 * 20];
        }
        for (int j = 0; j < p; ++j) bo[j] = rhs[j];
      }
      if (kp.status_out) kp.status_out[gidx] = bad;
    }
  }
}

// ---------------------------------------------------------------- packing kernels
__global__ void pack_T_kernel(const double* __restrict__ T, int64_t ld, int64_t n, int64_t NB,
                              double* __restrict__ Tpk) {
  const int64_t tile = blockIdx.x;  // one CTA per 2048-double tile
  int64_t i = (int64_t)((sqrt(1.0 + (double)tile) - 1.0) * 0.5);
  while (tpk_tile_offset(i + 1) <= tile) ++i;
  while (tpk_tile_offset(i) > tile) --i;
  const int64_t kt = tile - tpk_tile_offset(i);
  for (int w = threadIdx.x; w < kTileDoubles; w += blockDim.x) {
    const int g = w >> 7, rem = w & 127, P = rem >> 6, ln = (rem & 63) >> 1, e = rem & 1;
    // virtual (row, col) -> real (row - pad, col - pad); the padding sits at the top-left
    const int64_t pad = row_pad(n, NB);
    const int64_t row = i * kNB + g * 8 + (ln >> 2) - pad;
    const int64_t col = kt * kKT + 4 * (ln & 3) + 2 * P + e - pad;
    Tpk[tile * kTileDoubles + w] =
        (row >= 0 && row < n && col >= 0 && col <= row) ? T[row + col * ld] : 0.0;
  }
}

__global__ void pack_W_kernel(const double* __restrict__ W, int64_t ld, int64_t n, int ncolsW,
                              int NW, double* __restrict__ Wpk, int64_t total) {
  for (int64_t o = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; o < total;
       o += (int64_t)gridDim.x * blockDim.x) {
    // o = ((((i*4 + ns)*NW + w)*4 + s)*32 + lane)*2 + e
    int64_t r = o;
    const int e = r & 1; r >>= 1;
    const int lane = r & 31; r >>= 5;
    const int s = r & 3; r >>= 2;
    const int w = (int)(r % NW); r /= NW;
    const int ns = r & 3; r >>= 2;
    const int64_t i = r;
    const int64_t pad = row_pad(n, (n + kNB - 1) / kNB);
    const int64_t row = i * kNB + ns * 32 + s * 8 + 2 * (lane & 3) + e - pad;
    const int col = w * 8 + (lane >> 2);
    Wpk[o] = (row >= 0 && row < n && col < ncolsW) ? W[row + col * ld] : 0.0;
  }
}

// ---------------------------------------------------------------- tensor map
typedef CUresult (*PFN_encodeTiled)(CUtensorMap*, CUtensorMapDataType, cuuint32_t, void*,
                                    const cuuint64_t*, const cuuint64_t*, const cuuint32_t*,
                                    const cuuint32_t*, CUtensorMapInterleave, CUtensorMapSwizzle,
                                    CUtensorMapL2promotion, CUtensorMapFloatOOBfill);

PFN_encodeTiled get_encode() {
  static PFN_encodeTiled fn = nullptr;
  if (!fn) {
    void* p = nullptr;
    cudaDriverEntryPointQueryResult q;
    if (cudaGetDriverEntryPoint("cuTensorMapEncodeTiled", &p, cudaEnableDefault, &q) == cudaSuccess &&
        q == cudaDriverEntryPointSuccess)
      fn = (PFN_encodeTiled)p;
  }
  return fn;
}

template <int NW, bool FULL, bool ALIGNED>
cudaError_t launch_variant(cudaStream_t s, const CUtensorMap& map, const KParams& kp, int num_sms) {
  using C = KCfg<NW, FULL>;
  if (first_use_on_device((const void*)fused_trsm_gls_kernel<NW, FULL, ALIGNED>)) {
    cudaError_t e = cudaFuncSetAttribute(fused_trsm_gls_kernel<NW, FULL, ALIGNED>,
                                         cudaFuncAttributeMaxDynamicSharedMemorySize, (int)C::bytes);
    if (e != cudaSuccess) return e;
  }
  int64_t grid = kp.num_panels < num_sms ? kp.num_panels : num_sms;
  // GLS_FP64_CTAS (tests): a smaller persistent grid -- another panel schedule, the same bits
  static const int ctas_cap = getenv("GLS_FP64_CTAS") ? atoi(getenv("GLS_FP64_CTAS")) : 0;
  if (ctas_cap > 0 && ctas_cap < grid) grid = ctas_cap;
  fused_trsm_gls_kernel<NW, FULL, ALIGNED><<<(unsigned)grid, kThreads, C::bytes, s>>>(map, kp);
  return cudaGetLastError();
}

}  // namespace

void pack_T(cudaStream_t s, const double* T, int64_t ld, int64_t n, int64_t NB, double* Tpk,
            int64_t* lc) {
  pack_T_kernel<<<(unsigned)tpk_total_tiles(NB), 256, 0, s>>>(T, ld, n, NB, Tpk);
  if (lc) ++*lc;
}

void pack_W(cudaStream_t s, const double* W, int64_t ld, int64_t n, int ncolsW, int64_t NB, int NW,
            double* Wpk, int64_t* lc) {
  const int64_t total = NB * wpk_rb_doubles(NW);
  const int64_t blocks = (total + 255) / 256;
  pack_W_kernel<<<(unsigned)(blocks < 4096 ? blocks : 4096), 256, 0, s>>>(W, ld, n, ncolsW, NW, Wpk,
                                                                          total);
  if (lc) ++*lc;
}

// ---------------------------------------------------------------- compacted FP64 fallback (reading A16)
// After a block's int8 launches, its flagged problems (usually few) are gathered into a dense block,
// solved there by full panels (many SMs at once instead of one partly used panel per flagged problem,
// each a long one-CTA trsm) and their records scattered back; the per-column arithmetic does not depend
// on a column's panel position, so the bits are those of an in-place FP64 solve.  fb_index_kernel
// writes the block's flagged count to *count (0 when none); the others run only if 0 < *count <= cap.
__device__ __forceinline__ int gated_count(const int* count, int cap) {
  const int c = *(volatile const int*)count;
  return (c > 0 && c <= cap) ? c : 0;
}
// flagged problem indices in ascending order: one CTA, a block-wide scan per 1024 problems
__global__ void __launch_bounds__(1024) fb_index_kernel(const int* __restrict__ pflag, int64_t groups,
                                                        const int* __restrict__ ccount, int nchunks, int cap,
                                                        int* __restrict__ idx, int* __restrict__ count) {
  __shared__ int wsum[32];
  __shared__ int base_s;
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  if (threadIdx.x == 0) {
    int t = 0;
    for (int j = 0; j < nchunks; ++j) t += ccount[j];  // the chunks' flagged counts
    base_s = t;
  }
  __syncthreads();
  const int total = base_s;
  __syncthreads();
  if (total == 0 || total > cap) {  // nothing to gather (none, or the in-place path takes them)
    if (threadIdx.x == 0) *count = total;
    return;
  }
  if (threadIdx.x == 0) base_s = 0;
  __syncthreads();
  for (int64_t g0 = 0; g0 < groups; g0 += 1024) {
    const int64_t g = g0 + threadIdx.x;
    const int f = (g < groups && pflag[g]) ? 1 : 0;
    const unsigned bal = __ballot_sync(0xffffffffu, f);
    const int wpre = __popc(bal & ((1u << lane) - 1u));
    if (lane == 0) wsum[warp] = __popc(bal);
    __syncthreads();
    if (warp == 0) {  // inclusive scan of the 32 warp counts
      int v = wsum[lane];
#pragma unroll
      for (int o = 1; o < 32; o <<= 1) {
        const int t = __shfl_up_sync(0xffffffffu, v, o);
        if (lane >= o) v += t;
      }
      wsum[lane] = v;
    }
    __syncthreads();
    const int base = base_s;
    if (f) idx[base + (warp ? wsum[warp - 1] : 0) + wpre] = (int)g;
    __syncthreads();
    if (threadIdx.x == 0) base_s = base + wsum[31];
    __syncthreads();
  }
  if (threadIdx.x == 0) *count = total;
}
// the flagged problems' pR columns (all ldx rows) -> the dense block Xc (same leading dimension)
__global__ void fb_gather_kernel(const double* __restrict__ X, int64_t ldx, int pR, const int* __restrict__ idx,
                                 const int* count, int cap, double* __restrict__ Xc) {
  const int c = gated_count(count, cap);
  for (int64_t col = blockIdx.x; col < (int64_t)c * pR; col += gridDim.x) {
    const int64_t k = col / pR, a = col - k * pR;
    const double2* src = (const double2*)(X + ((int64_t)idx[k] * pR + a) * ldx);
    double2* dst = (double2*)(Xc + col * ldx);
    for (int64_t r = threadIdx.x; r < ldx / 2; r += blockDim.x) dst[r] = src[r];
  }
}
__global__ void fb_scatter_kernel(const double* __restrict__ bc, const int32_t* __restrict__ sc,
                                  const int* __restrict__ idx, const int* count, int cap, int p,
                                  double* __restrict__ b, int32_t* __restrict__ st) {
  const int c = gated_count(count, cap);
  for (int64_t t = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; t < (int64_t)c * p;
       t += (int64_t)gridDim.x * blockDim.x) {
    const int64_t k = t / p, j = t - k * p;
    b[(int64_t)idx[k] * p + j] = bc[t];
    if (j == 0 && st) st[idx[k]] = sc[k];
  }
}
void fb_compact(cudaStream_t s, const int* pflag, int64_t groups, const int* ccount, int nchunks, int cap, int* idx,
                int* count, const double* X, int64_t ldx, int pR, double* Xc, int num_sms, int64_t* lc) {
  fb_index_kernel<<<1, 1024, 0, s>>>(pflag, groups, ccount, nchunks, cap, idx, count);
  fb_gather_kernel<<<(unsigned)(2 * num_sms), 256, 0, s>>>(X, ldx, pR, idx, count, cap, Xc);
  if (lc) *lc += 2;
}
void fb_scatter(cudaStream_t s, const double* bc, const int32_t* sc, const int* idx, const int* count, int cap,
                int p, double* b, int32_t* st, int num_sms, int64_t* lc) {
  fb_scatter_kernel<<<(unsigned)num_sms, 256, 0, s>>>(bc, sc, idx, count, cap, p, b, st);
  if (lc) ++*lc;
}

cudaError_t launch_fused_trsm_gls(cudaStream_t s, const SolveArgs& a, int num_sms, std::string* msg,
                                  int64_t* lc, const int* gate, unsigned long long* ran) {
  PFN_encodeTiled enc = get_encode();
  if (!enc) {
    if (msg) *msg = "cuTensorMapEncodeTiled unavailable from the driver";
    return cudaErrorNotSupported;
  }
  const PanelGeom pg = panel_geom(a.pR);
  CUtensorMap map;
  const int64_t cols = a.m_blk * a.pR;
  // dim0 = ldx (>= n, even): rows in [n, ldx) are the zero pad row of the staged copy (odd n).
  cuuint64_t gdim[2] = {(cuuint64_t)a.ldx, (cuuint64_t)cols};
  cuuint64_t gstride[1] = {(cuuint64_t)(a.ldx * 8)};
  cuuint32_t box[2] = {(cuuint32_t)kKT, (cuuint32_t)pg.cpp};
  cuuint32_t estr[2] = {1, 1};
  CUresult r = enc(&map, CU_TENSOR_MAP_DATA_TYPE_FLOAT64, 2, (void*)a.X, gdim, gstride, box, estr,
                   CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_128B,
                   CU_TENSOR_MAP_L2_PROMOTION_L2_256B, CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
  if (r != CUDA_SUCCESS) {
    if (msg) {
      char buf[160];
      snprintf(buf, sizeof buf, "cuTensorMapEncodeTiled failed (CUresult %d; n=%lld ld=%lld)", (int)r,
               (long long)a.n, (long long)a.ldx);
      *msg = buf;
    }
    return cudaErrorInvalidValue;
  }
  KParams kp;
  kp.Tpk = a.Tpk;
  kp.Wpk = a.Wpk;
  kp.G = a.G;
  kp.b_out = a.b_out;
  kp.status_out = a.status_out;
  kp.gate = gate;
  kp.pflag = a.pflag;
  kp.m_dev = a.m_dev;
  kp.gate_lo = a.gate_lo;
  kp.gate_hi = a.gate_hi;
  kp.ran = ran;
  kp.m_blk = a.m_blk;
  kp.num_panels = (a.m_blk + pg.gpp - 1) / pg.gpp;
  kp.NB = (int)a.NB;
  kp.pad = (int)row_pad(a.n, a.NB);
  kp.kt0 = kp.pad / kKT;
  kp.pL = a.pL;
  kp.pR = a.pR;
  kp.p = a.pL + a.pR;
  kp.gw = pg.gw;
  kp.cpw = pg.cpw;
  kp.cpp = pg.cpp;
  kp.gpp = pg.gpp;
  const int NW = (a.pL + 1 + 7) / 8;
  cudaError_t e;
  // ALIGNED: every warp's column range starts on an 8-column boundary (pR divides 32), so the
  // swizzle phase is the same for the 4 column tiles and fragment addresses are immediates.
  const bool aligned = (pg.cpw % 8) == 0;
  if (!pg.full_gram) {
    e = NW == 1 ? launch_variant<1, false, true>(s, map, kp, num_sms)
      : NW == 2 ? launch_variant<2, false, true>(s, map, kp, num_sms)
                : launch_variant<3, false, true>(s, map, kp, num_sms);
  } else if (aligned) {
    e = NW == 1 ? launch_variant<1, true, true>(s, map, kp, num_sms)
      : NW == 2 ? launch_variant<2, true, true>(s, map, kp, num_sms)
                : launch_variant<3, true, true>(s, map, kp, num_sms);
  } else {
    e = NW == 1 ? launch_variant<1, true, false>(s, map, kp, num_sms)
      : NW == 2 ? launch_variant<2, true, false>(s, map, kp, num_sms)
                : launch_variant<3, true, false>(s, map, kp, num_sms);
  }
  if (lc) ++*lc;
  if (e != cudaSuccess && msg) *msg = std::string("fused_trsm_gls launch: ") + cudaGetErrorString(e);
  return e;
}

}  // namespace gls
