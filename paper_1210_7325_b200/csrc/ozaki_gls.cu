// ozaki_gls.cu -- the int8 tensor-core hot path: Alg. 5 line 3 fused with lines 7-11
// (Alg. 8 lines 9-14) on tcgen05 kind::i8.
//
// Why int8 for an FP64 method (reading A15): the trsm is z = T x with T = L^{-1}
// (design A, reading A13) and x a column of SNP genotypes, which are small integers (0, 1, 2 in
// every configuration; "SNPs").  Each row r of T is written as a 55-bit fixed-point
// integer V_r,j = rint(T_r,j * 2^(e_r + 48)), e_r chosen so that max_j |T_r,j| 2^e_r <= 127, and V is
// split into 7 signed base-256 digits d_0 (|d_0| <= 127) .. d_6 (in [-128, 127]):
//
//     V_r,j = sum_s d_s,r,j 256^(6-s)          (exact, int64 arithmetic at setup)
//     z_r   = 2^-(e_r+48) sum_s 256^(6-s) (sum_j d_s,r,j x_j)
//
// Every inner product sum_j d x_j is an exact int32 (|d x| <= 2^14, n <= 131072) computed by the
// 5th-generation tensor core with int32 accumulators in tensor memory; the only roundings are the
// one of T to 55 significant bits per row (2^-55 relative to the row maximum, below FP64's own
// 2^-53 per element) and the FP64 combination of the 7 partial sums.  The result is an FP64-accurate
// z at int8 tensor throughput: 7 int8 MACs replace one FP64 MAC, and B200's dense int8 rate is
// ~120x its FP64 DMMA rate.  The data-dependent guard: a block whose X_R is not all integers in
// [-128, 127] is solved by the FP64 DMMA kernel instead (fused_trsm_gls.cu), decided on the device.
//
// Kernel layout (one CTA per SM, persistent over tiles of 128 SNP columns):
//   warp 0      TMA producer: per stage the X tile (128 columns x 128 K, int8, 4 boxes of 32
//               columns, 128B swizzle) and the packed T tile (7 digits x 32 z rows x 128 K, int8,
//               pre-swizzled, one bulk copy), under full/empty mbarriers;
//   warp 1      MMA issuer: D[128 cols x 224] += X^T[128 x 128] T^T[128 x 224] as 4
//               tcgen05.mma.kind::i8 (M=128, N=224, K=32) per stage, D double-buffered in TMEM
//               (2 x 224 of 512 columns); commits free the stage and hand D to the epilogue;
//   warps 2-9   epilogue: thread = one SNP column (TMEM lane), half h of the 32 z rows: combine
//               the 7 digit products into z in FP64, then acc_W += z W~_row, acc_G += z z (Fig. 1
//               S_BL, b_B, S_BR) -- X~_R never leaves registers.  After the last row block the two
//               halves are summed in a fixed order and one lane per problem assembles S_i and
//               solves it by Cholesky with the rank rule of reading A4 (Alg. 5 line 11).
#include <cuda.h>

#include <cstdio>

#include "gls_internal.cuh"
#include "umma.cuh"

namespace gls {
namespace {

using namespace umma;

constexpr int kR = kOzR;                 // z rows per row block
constexpr int kKC = kOzKC;               // K per stage (one 128-byte swizzle span of int8)
constexpr int kNSL = kOzSlices;          // digits per T element
constexpr int kBN = kNSL * kR;           // MMA N = 224
constexpr int kATile = 128 * kKC;        // 16 KiB
constexpr int kBTile = kBN * kKC;        // 28 KiB
constexpr int kStages = 4;
constexpr int kEpiWarps = 8;
constexpr int kThreads = (2 + kEpiWarps) * 32;
constexpr uint32_t kTmemCols = 512;
constexpr uint32_t kIdesc = idesc_i8(128, kBN);
static_assert(kOzTileBytes == kBTile, "packed T tile size");

struct OzParams {
  const int8_t* T8;     // packed digit tiles (oz_tile_offset)
  const double* aux;    // per virtual row: [sigma, W~_0 .. W~_pL], stride pL + 2
  const double* G;      // (pL+1)^2 column-major: S_TL = G[0:pL,0:pL], b_T = G[0:pL,pL]
  const int* gate;      // non-zero: X_R is not int8-representable -> this kernel does nothing
  unsigned long long* ran;
  double* b_out;
  int32_t* status_out;
  int64_t cols;         // m_blk * pR
  int64_t m_blk;
  int num_tiles;
  int NBR;              // row blocks of 32
  int pL, pR, p;
  int cpw;              // columns per warp quadrant = floor(32 / pR) * pR
};

template <int NA>
__device__ __forceinline__ void zero_acc(double (&acc)[NA]) {
#pragma unroll
  for (int k = 0; k < NA; ++k) acc[k] = 0.0;
}

// Cholesky solve of one p x p system with the rank rule of reading A4 (same as the DMMA kernel).
__device__ void posv_store(double* S, double* rhs, int p, double* bo, int32_t* st) {
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
  if (st) *st = bad;
}

// NA: accumulators per column (>= pL + 1 + pR); PR1: pR == 1 (Gram = z^2, no shuffles).
template <int NA, bool PR1>
__global__ void __launch_bounds__(kThreads, 1)
    ozaki_trsm_gls_kernel(const __grid_constant__ CUtensorMap xmap, const OzParams kp) {
  extern __shared__ __align__(1024) uint8_t smem_raw[];
  uint8_t* smem = (uint8_t*)(((uintptr_t)smem_raw + 1023) & ~(uintptr_t)1023);
  uint8_t* sA = smem;
  uint8_t* sB = sA + kStages * kATile;
  double* red = (double*)(sB + kStages * kBTile);  // 128 columns x NA
  uint64_t* bars = (uint64_t*)(red + 128 * NA);
  uint64_t* full = bars;
  uint64_t* empty = bars + kStages;
  uint64_t* tfull = bars + 2 * kStages;
  uint64_t* tempty = bars + 2 * kStages + 2;
  uint32_t* tslot = (uint32_t*)(bars + 2 * kStages + 4);

  if (kp.gate && *(volatile const int*)kp.gate != 0) return;  // uniform across the grid
  if (kp.ran && blockIdx.x == 0 && threadIdx.x == 0) atomicAdd(kp.ran, 1ull);

  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  if (threadIdx.x == 0) {
    for (int s = 0; s < kStages; ++s) {
      mbar_init(&full[s], 1);
      mbar_init(&empty[s], 1);
    }
    for (int b = 0; b < 2; ++b) {
      mbar_init(&tfull[b], 1);
      mbar_init(&tempty[b], kEpiWarps);
    }
    fence_barrier_init();
  }
  if (warp == 1) tmem_alloc(tslot, kTmemCols);
  tc_fence_before();
  __syncthreads();
  tc_fence_after();
  const uint32_t tbase = *tslot;
  const int cpt = 4 * kp.cpw;  // columns per tile

  if (warp == 0) {
    // ------------------------------------------------------------ TMA producer
    if (lane == 0) {
      prefetch_tmap(&xmap);
      int stage = 0;
      uint32_t ph = 0;
      for (int tile = blockIdx.x; tile < kp.num_tiles; tile += gridDim.x) {
        const int col0 = tile * cpt;
        for (int i = 0; i < kp.NBR; ++i) {
          const int nc = (i >> 2) + 1;
          const int8_t* tsrc = kp.T8 + oz_tile_offset(i) * (int64_t)kBTile;
          for (int c = 0; c < nc; ++c) {
            mbar_wait(&empty[stage], ph ^ 1);
            mbar_arrive_expect_tx(&full[stage], kATile + kBTile);
#pragma unroll
            for (int q = 0; q < 4; ++q)
              tma_2d_g2s(sA + stage * kATile + q * 4096, &xmap, c * kKC, col0 + q * kp.cpw, &full[stage]);
            bulk_g2s(sB + stage * kBTile, tsrc + (int64_t)c * kBTile, kBTile, &full[stage]);
            if (++stage == kStages) {
              stage = 0;
              ph ^= 1;
            }
          }
        }
      }
    }
  } else if (warp == 1) {
    // ------------------------------------------------------------ MMA issuer
    if (lane == 0) {
      int stage = 0;
      uint32_t ph = 0;
      uint32_t rbc = 0;
      const uint32_t a0 = smem_u32(sA), b0 = smem_u32(sB);
      for (int tile = blockIdx.x; tile < kp.num_tiles; tile += gridDim.x) {
        for (int i = 0; i < kp.NBR; ++i, ++rbc) {
          const int nc = (i >> 2) + 1;
          const uint32_t buf = rbc & 1, tph = (rbc >> 1) & 1;
          mbar_wait(&tempty[buf], tph ^ 1);
          tc_fence_after();
          const uint32_t dt = tbase + buf * 256;
          for (int c = 0; c < nc; ++c) {
            mbar_wait(&full[stage], ph);
            tc_fence_after();
            const uint64_t ad = sdesc_k128(a0 + stage * kATile);
            const uint64_t bd = sdesc_k128(b0 + stage * kBTile);
#pragma unroll
            for (int kk = 0; kk < kKC / 32; ++kk)
              mma_i8(dt, ad + (uint64_t)(2 * kk), bd + (uint64_t)(2 * kk), kIdesc, (c | kk) != 0);
            mma_commit(&empty[stage]);
            if (++stage == kStages) {
              stage = 0;
              ph ^= 1;
            }
          }
          mma_commit(&tfull[buf]);
        }
      }
    }
  } else {
    // ------------------------------------------------------------ epilogue
    const int ew = warp - 2;
    const int q = warp & 3;      // TMEM lane quadrant this warp may access
    const int h = ew >> 2;       // which 16 of the 32 z rows
    const int tc = q * 32 + lane;  // column of the tile held by this thread (TMEM lane)
    const int pl1 = kp.pL + 1;
    const int as = kp.pL + 2;      // aux row stride
    const int a_in = PR1 ? 0 : lane % kp.pR;  // position inside the group
    const uint32_t trow = tbase + ((uint32_t)(q * 32) << 16) + h * 16;
    double acc[NA];
    zero_acc(acc);
    uint32_t rbc = 0;
    for (int tile = blockIdx.x; tile < kp.num_tiles; tile += gridDim.x) {
      for (int i = 0; i < kp.NBR; ++i, ++rbc) {
        const uint32_t buf = rbc & 1, tph = (rbc >> 1) & 1;
        mbar_wait(&tfull[buf], tph);
        tc_fence_after();
        double z[16];
        {
          int32_t v[16];
          tmem_ld16(trow + buf * 256, v);
          tmem_wait_ld();
#pragma unroll
          for (int r = 0; r < 16; ++r) z[r] = (double)v[r];
        }
#pragma unroll 1
        for (int s = 1; s < kNSL; ++s) {
          int32_t v[16];
          tmem_ld16(trow + buf * 256 + s * kR, v);
          tmem_wait_ld();
#pragma unroll
          for (int r = 0; r < 16; ++r) z[r] = fma(z[r], 256.0, (double)v[r]);
        }
        tc_fence_before();
        __syncwarp();
        if (lane == 0) mbar_arrive(&tempty[buf]);
        const double* arow = kp.aux + (int64_t)(i * kR + h * 16) * as;
#pragma unroll
        for (int r = 0; r < 16; ++r) {
          const double* a = arow + r * as;
          const double zr = z[r] * __ldg(a);
#pragma unroll
          for (int w = 0; w < NA; ++w)
            if (w < pl1) acc[w] = fma(zr, __ldg(a + 1 + w), acc[w]);
          if (PR1) {
            acc[pl1 < NA ? pl1 : NA - 1] = fma(zr, zr, acc[pl1 < NA ? pl1 : NA - 1]);
          } else {
#pragma unroll
            for (int b = 0; b < NA; ++b) {
              if (b < kp.pR) {
                const double zb = __shfl_sync(0xffffffffu, zr, lane - a_in + b);
                if (pl1 + b < NA) acc[pl1 + b] = fma(zr, zb, acc[pl1 + b]);
              }
            }
          }
        }
      }
      // ---- per-tile finalisation: sum the two row halves, assemble S_i, posv
      named_bar_sync(1, kEpiWarps * 32);
      if (h == 1) {
#pragma unroll
        for (int w = 0; w < NA; ++w) red[tc * NA + w] = acc[w];
      }
      named_bar_sync(2, kEpiWarps * 32);
      if (h == 0) {
#pragma unroll
        for (int w = 0; w < NA; ++w) red[tc * NA + w] = acc[w] + red[tc * NA + w];
        __syncwarp();
        const int64_t col = (int64_t)tile * cpt + q * kp.cpw + lane;
        if (lane < kp.cpw && a_in == 0 && col < kp.cols) {
          const int64_t g = col / kp.pR;
          const int p = kp.p, pL = kp.pL, pR = kp.pR;
          double S[400];
          double rhs[20];
          for (int a2 = 0; a2 < pL; ++a2) {
            for (int b2 = 0; b2 < pL; ++b2) S[a2 + b2 * 20] = __ldg(kp.G + a2 + b2 * pl1);
            rhs[a2] = __ldg(kp.G + a2 + pL * pl1);
          }
          for (int a2 = 0; a2 < pR; ++a2) {
            const double* rr = red + (tc + a2) * NA;
            for (int k = 0; k < pL; ++k) {
              S[(pL + a2) + k * 20] = rr[k];
              S[k + (pL + a2) * 20] = rr[k];
            }
            rhs[pL + a2] = rr[pL];
            for (int b2 = 0; b2 < pR; ++b2) S[(pL + a2) + (pL + b2) * 20] = rr[pl1 + b2];
          }
          posv_store(S, rhs, p, kp.b_out + g * p, kp.status_out ? kp.status_out + g : nullptr);
        }
      }
      zero_acc(acc);
    }
  }
  tc_fence_before();
  __syncthreads();
  if (warp == 1) tmem_dealloc(tbase, kTmemCols);
}

// ---------------------------------------------------------------- setup kernels
// Row scale: e_r with max_j |T_rj| 2^e_r <= 127; sigma_r = 2^-(e_r + 48).  One CTA per 32 rows,
// 8 column strands per row (T column-major, so a warp reads 32 consecutive rows of one column).
__global__ void oz_rowscale_kernel(const double* __restrict__ T, int64_t ld, int64_t n,
                                   int* __restrict__ escale, double* __restrict__ aux, int as) {
  __shared__ double sm[8][32];
  const int rl = threadIdx.x & 31, strand = threadIdx.x >> 5;
  const int64_t r = (int64_t)blockIdx.x * 32 + rl;
  double mx = 0.0;
  if (r < n)
    for (int64_t j = strand; j <= r; j += 8) mx = fmax(mx, fabs(T[r + j * ld]));
  sm[strand][rl] = mx;
  __syncthreads();
  if (strand == 0) {
    for (int k = 1; k < 8; ++k) mx = fmax(mx, sm[k][rl]);
    int e = 0;
    double sig = 0.0;
    if (mx > 0.0) {
      int E;
      const double f = frexp(mx, &E);  // mx = f 2^E, f in [0.5, 1)
      e = (f * 128.0 <= 127.0) ? 7 - E : 6 - E;
      sig = ldexp(1.0, -(e + 48));
    }
    escale[r] = e;
    aux[r * as] = sig;  // rows >= n: sigma = 0 (their T digits are zero too)
  }
}

// Digits of every element of every packed tile: tile (i, c) holds rows 32i..32i+31, K columns
// 128c..128c+127; B row s*32 + rr holds digit s of row 32i + rr, swizzled (umma::swz128).
__global__ void oz_pack_kernel(const double* __restrict__ T, int64_t ld, int64_t n,
                               const int* __restrict__ escale, int NBR, int8_t* __restrict__ T8) {
  const int64_t tile = blockIdx.x;
  int i = (int)sqrt(2.0 * (double)tile);  // invert oz_tile_offset
  while (i > 0 && oz_tile_offset(i) > tile) --i;
  while (i + 1 <= NBR && oz_tile_offset(i + 1) <= tile) ++i;
  const int c = (int)(tile - oz_tile_offset(i));
  int8_t* dst = T8 + tile * (int64_t)kOzTileBytes;
  const int rr = threadIdx.x & 31;
  const int64_t r = (int64_t)i * kR + rr;
  const int e = (r < n) ? escale[r] : 0;
  for (int k = threadIdx.x >> 5; k < kKC; k += blockDim.x >> 5) {
    const int64_t j = (int64_t)c * kKC + k;
    long long V = 0;
    if (r < n && j <= r) V = llrint(ldexp(T[r + j * ld], e + 48));
    int8_t d[kNSL];
#pragma unroll
    for (int s = kNSL - 1; s > 0; --s) {  // signed base-256 digits, least significant first
      const int8_t lo = (int8_t)(V & 0xff);
      d[s] = lo;
      V = (V - lo) >> 8;
    }
    d[0] = (int8_t)V;  // |top| <= 127 because |V| <= 127 * 2^48
#pragma unroll
    for (int s = 0; s < kNSL; ++s) dst[swz128(s * kR + rr, k)] = d[s];
  }
}

__global__ void oz_aux_w_kernel(const double* __restrict__ W, int64_t ldw, int64_t n, int pl1,
                                int64_t rows, double* __restrict__ aux) {
  const int as = pl1 + 1;
  for (int64_t o = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; o < rows * pl1;
       o += (int64_t)gridDim.x * blockDim.x) {
    const int64_t r = o / pl1;
    const int w = (int)(o % pl1);
    aux[r * as + 1 + w] = (r < n) ? W[r + w * ldw] : 0.0;
  }
}

// X (double, column-major, ld = ldx) -> X8 (int8, column-major, ld = ld8), flagging any value that
// is not an integer in [-128, 127] (NaN included).  One thread per 8 rows of one column.
__global__ void oz_x_to_i8_kernel(const double* __restrict__ X, int64_t ldx, int64_t n, int64_t cols,
                                  int8_t* __restrict__ X8, int64_t ld8, int* __restrict__ flag) {
  const int64_t per_col = (n + 7) >> 3;
  const int64_t total = per_col * cols;
  int bad = 0;
  for (int64_t o = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; o < total;
       o += (int64_t)gridDim.x * blockDim.x) {
    const int64_t col = o / per_col;
    const int64_t r0 = (o - col * per_col) << 3;
    const double* src = X + col * ldx + r0;
    uint32_t w[2] = {0, 0};
#pragma unroll
    for (int k = 0; k < 8; ++k) {
      const double v = (r0 + k < n) ? __ldcs(src + k) : 0.0;
      const double t = rint(v);
      bad |= !(t == v && fabs(v) <= 127.0);
      const uint32_t b = (uint32_t)(uint8_t)(int8_t)(int)t;
      w[k >> 2] |= b << (8 * (k & 3));
    }
    if (r0 + 8 <= ld8) {
      *(uint2*)(X8 + col * ld8 + r0) = make_uint2(w[0], w[1]);
    } else {
      for (int k = 0; r0 + k < ld8; ++k) X8[col * ld8 + r0 + k] = (int8_t)(w[k >> 2] >> (8 * (k & 3)));
    }
  }
  if (__any_sync(0xffffffffu, bad) && (threadIdx.x & 31) == 0) atomicOr(flag, 1);
}

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

template <int NA, bool PR1>
cudaError_t launch_oz_variant(cudaStream_t s, const CUtensorMap& map, const OzParams& kp, int num_sms) {
  constexpr int smem = kStages * (kATile + kBTile) + 128 * NA * 8 + 16 * 8 + 1024;
  static bool attr_done = false;
  if (!attr_done) {
    cudaError_t e = cudaFuncSetAttribute(ozaki_trsm_gls_kernel<NA, PR1>,
                                         cudaFuncAttributeMaxDynamicSharedMemorySize, smem);
    if (e != cudaSuccess) return e;
    attr_done = true;
  }
  const int grid = kp.num_tiles < num_sms ? kp.num_tiles : num_sms;
  ozaki_trsm_gls_kernel<NA, PR1><<<grid, kThreads, smem, s>>>(map, kp);
  return cudaGetLastError();
}

}  // namespace

int64_t oz_total_tiles(int64_t NBR) { return oz_tile_offset(NBR); }

void oz_setup(cudaStream_t s, const double* T, int64_t ld, int64_t n, const double* W, int pl1,
              int8_t* T8, double* aux, int* escale, int64_t* lc) {
  const int NBR = (int)((n + kR - 1) / kR);
  const int as = pl1 + 1;
  oz_rowscale_kernel<<<NBR, 256, 0, s>>>(T, ld, n, escale, aux, as);
  oz_pack_kernel<<<(unsigned)oz_total_tiles(NBR), 256, 0, s>>>(T, ld, n, escale, NBR, T8);
  const int64_t rows = (int64_t)NBR * kR;
  const int64_t tot = rows * pl1;
  oz_aux_w_kernel<<<(unsigned)((tot + 255) / 256 < 2048 ? (tot + 255) / 256 : 2048), 256, 0, s>>>(
      W, n, n, pl1, rows, aux);
  if (lc) *lc += 3;
}

void oz_convert(cudaStream_t s, const double* X, int64_t ldx, int64_t n, int64_t cols, int8_t* X8,
                int64_t ld8, int* flag, int num_sms, int64_t* lc) {
  const int64_t total = ((n + 7) >> 3) * cols;
  int64_t blocks = (total + 255) / 256;
  if (blocks > (int64_t)num_sms * 16) blocks = (int64_t)num_sms * 16;
  if (blocks < 1) blocks = 1;
  oz_x_to_i8_kernel<<<(unsigned)blocks, 256, 0, s>>>(X, ldx, n, cols, X8, ld8, flag);
  if (lc) ++*lc;
}

cudaError_t launch_ozaki_gls(cudaStream_t s, const OzArgs& a, int num_sms, std::string* msg,
                             int64_t* lc) {
  PFN_encodeTiled enc = get_encode();
  if (!enc) {
    if (msg) *msg = "cuTensorMapEncodeTiled unavailable from the driver";
    return cudaErrorNotSupported;
  }
  const int cpw = (32 / a.pR) * a.pR;
  const int64_t cols = a.m_blk * a.pR;
  CUtensorMap map;
  cuuint64_t gdim[2] = {(cuuint64_t)a.n, (cuuint64_t)cols};
  cuuint64_t gstride[1] = {(cuuint64_t)a.ld8};
  cuuint32_t box[2] = {(cuuint32_t)kKC, 32};
  cuuint32_t estr[2] = {1, 1};
  CUresult r = enc(&map, CU_TENSOR_MAP_DATA_TYPE_UINT8, 2, (void*)a.X8, gdim, gstride, box, estr,
                   CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_128B,
                   CU_TENSOR_MAP_L2_PROMOTION_L2_256B, CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
  if (r != CUDA_SUCCESS) {
    if (msg) {
      char buf[160];
      snprintf(buf, sizeof buf, "cuTensorMapEncodeTiled (int8 X) failed (CUresult %d; n=%lld ld8=%lld)",
               (int)r, (long long)a.n, (long long)a.ld8);
      *msg = buf;
    }
    return cudaErrorInvalidValue;
  }
  OzParams kp;
  kp.T8 = a.T8;
  kp.aux = a.aux;
  kp.G = a.G;
  kp.gate = a.gate;
  kp.ran = a.ran;
  kp.b_out = a.b_out;
  kp.status_out = a.status_out;
  kp.cols = cols;
  kp.m_blk = a.m_blk;
  const int64_t cpt = 4 * (int64_t)cpw;
  kp.num_tiles = (int)((cols + cpt - 1) / cpt);
  kp.NBR = (int)((a.n + kR - 1) / kR);
  kp.pL = a.pL;
  kp.pR = a.pR;
  kp.p = a.pL + a.pR;
  kp.cpw = cpw;
  cudaError_t e;
  if (a.pR == 1 && a.pL + 2 <= 8)
    e = launch_oz_variant<8, true>(s, map, kp, num_sms);
  else if (a.pR == 1)
    e = launch_oz_variant<21, true>(s, map, kp, num_sms);
  else
    e = launch_oz_variant<21, false>(s, map, kp, num_sms);
  if (lc) ++*lc;
  if (e != cudaSuccess && msg) *msg = std::string("ozaki_trsm_gls launch: ") + cudaGetErrorString(e);
  return e;
}

}  // namespace gls
