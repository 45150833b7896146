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
// Kernel layout (CTA pairs, one CTA per SM, persistent over tiles of 256 SNP columns per pair):
//   warp 0      TMA producer: per stage the X tile (128 columns x 128 K per CTA, int8, 4 boxes of 32
//               columns, 128B swizzle) and this CTA's half of the packed digit tiles of TWO row blocks
//               (a "step"), under full/empty mbarriers;
//   warp 1      MMA issuer (leader): per stage and row block, 4 tcgen05.mma.cta_group::2.kind::i8
//               (M=256, N=224, K=32) into that row block's accumulator region of TMEM ([0, 224) and
//               [256, 480)), so each X chunk is staged once for two row blocks; commits free the stage
//               and hand the regions to the epilogue;
//   warps 2-9   epilogue: thread = one SNP column (TMEM lane), half h of the 32 z rows: combine
//               the 7 digit products into z in FP64 (exact int64 partial sums), release the region,
//               then acc_G += z z over the group (Fig. 1 S_BR); S_BL and b_B come exactly from one
//               extra MMA pass against the digits of V = M^-1 [X_L | y] (reading A17) -- X~_R never
//               leaves registers.  After the last step the two halves are summed (through TMEM) in a
//               fixed order and one lane per problem assembles S_i and solves it by Cholesky with the
//               rank rule of reading A4 (Alg. 5 line 11; for p > 8 a separate batched kernel does).
//   warps 10-11 convert-ahead: FP64 -> int8 of the NEXT chunk's X_R through bulk copies into
//               shared memory, concurrently with the tensor-core work.
#include <cuda.h>

#include <cstdio>

#include "gls_internal.cuh"
#include "umma.cuh"

// TMEM round trips per row-block drain in the epilogue: 2 = digits 0-3 then 4-6 (default; integer
// sums, so the same bits as 4 = two digits per load pair).  A/B on one box (tools/gpu_ab_drain.sh,
// config 2): 232.0 vs 233.5 ms per 1e6 SNPs (~0.7 %); config 3: no measurable difference.
#ifndef GLS_OZ_DRAIN_RT
#define GLS_OZ_DRAIN_RT 2
#endif
// pR = 1 variants: drain a row-block half in ONE round trip (all 7 digit loads in flight), so the
// region is released one TMEM latency earlier (A/B: see DESIGN.md §5.4)
#ifndef GLS_OZ_DRAIN_ONE
#define GLS_OZ_DRAIN_ONE 1
#endif

namespace gls {
namespace {

using namespace umma;

constexpr int kR = kOzR;                 // z rows per row block
constexpr int kKC = kOzKC;               // K per stage (one 128-byte swizzle span of int8)
constexpr int kNSL = kOzSlices;          // digits per T element
constexpr int kBN = kNSL * kR;           // MMA N = 224
constexpr int kATile = 128 * kKC;        // 16 KiB
constexpr int kBTile = kBN * kKC;        // 28 KiB (whole packed digit tile)
constexpr int kBHalf = kBTile / 2;       // 14 KiB staged per CTA of a pair
constexpr int kEpiWarps = 8;
constexpr bool kDrainOneTrip = GLS_OZ_DRAIN_ONE != 0;
constexpr int kConvWarps = 2;  // convert-ahead warps: FP64 -> int8 of the NEXT chunk (see the kernel)
constexpr int kThreads = (2 + kEpiWarps + kConvWarps) * 32;
constexpr int kCvBuf = 8192;          // bytes per convert-ahead staging buffer (two per conv warp)
constexpr int kCvRows = kCvBuf / 8;   // X rows per piece
#ifndef GLS_OZ_CV_HINT
#define GLS_OZ_CV_HINT 1
#endif
constexpr bool kCvHint = GLS_OZ_CV_HINT != 0;  // L2 evict_first hints on the convert-ahead traffic
constexpr uint32_t kTmemCols = 512;
// TMEM column pair of double w in the epilogue hand-over scratch: columns MMAs never write
__device__ __forceinline__ uint32_t xcol(int w) { return w < 16 ? 224 + 2 * w : 480 + 2 * (w - 16); }
constexpr uint32_t kIdesc = idesc_i8(256, kBN);  // CTA pair: M = 256
static_assert(kOzTileBytes == kBTile, "packed T tile size");

struct OzParams {
  const int8_t* T8;     // packed digit tiles (oz_tile_offset)
  const double* aux;    // per virtual row: [sigma, W~_0 .. W~_pL], stride pL + 2
  const double* G;      // (pL+1)^2 column-major: S_TL = G[0:pL,0:pL], b_T = G[0:pL,pL]
  const int* gate;      // non-zero: X_R is not int8-representable -> this kernel does nothing
  unsigned long long* ran;
  long long* prof;      // nullable diagnostics: per CTA 8 counters of clock cycles (GLS_OZ_PROF=1)
  double* b_out;
  int32_t* status_out;
  int64_t cols;         // m_blk * pR
  int64_t m_blk;
  int num_tiles;
  int NBR;              // row blocks of 32
  int pL, pR, p;
  int cpw;              // columns per warp quadrant = floor(32 / pR) * pR
  int NC;               // K chunks of 128 rows = ceil(n / 128)
  int NV;               // N of the V block: 8 (pL+1) rounded up to a multiple of 32
  int cpin;             // X chunks c < cpin are loaded L2::evict_last (they are re-read by every row
                        // block of the tile), the others evict_first
  const double* vscale; // pL+1 column scales 2^-(e_w+48) of V = M^{-1} [X_L | y]
  double* s_ws;         // nullable: per problem S_BL (pR x pL), S_BR (pR x pR), b_B (pR) for oz_posv_kernel
  // convert-ahead job (nullable cv_X): FP64 X of the next chunk -> int8 cv_X8, any non-integer or
  // out-of-range value sets *cv_flag
  int64_t n;            // rows of X / T
  const double* cv_X;
  int64_t cv_ldx, cv_cols;
  int8_t* cv_X8;
  int64_t cv_ld8;
  int* cv_flag;
  // per-problem path choice (nullable pflag): pflag[g] != 0 -- problem g holds a value that is not an
  // integer in [-128, 127] and is solved by the FP64 kernel; *gate then counts the flagged problems and
  // this kernel skips only when all gate_all of them are; it stores no result of a flagged problem.
  // cv_pflag: the same flags for the convert-ahead job's chunk (first-time flags add 1 to *cv_flag).
  const int* pflag;
  int64_t gate_all;
  int* cv_pflag;
};

// FP64 value -> int8 code, flagging (bad = 1) anything that is not an integer in [-128, 127]
__device__ __forceinline__ uint32_t to_i8_bits(double v, int& bad) {
  // 32-bit integer tests on the two words of v: an integer 1 <= |v| <= 255 has biased exponent
  // 1023 + k (k <= 7), its integer part in the top k of the high word's 20 mantissa bits and nothing
  // below (the low word and the high word's low 20 - k bits are zero)
  const uint32_t hi = (uint32_t)__double2hiint(v), lo = (uint32_t)__double2loint(v);
  const uint32_t a = hi & 0x7fffffffu;
  const uint32_t k = (a >> 20) - 1023u;  // wraps for |v| < 1
  const bool zero = (a | lo) == 0u;
  const bool ok = k <= 7u && lo == 0u && (a & ((0x100000u >> (k & 7u)) - 1u)) == 0u;
  const uint32_t mag = ((a & 0xfffffu) | 0x100000u) >> (20u - (k & 7u));  // 1 .. 255 when ok
  const bool neg = (hi >> 31) != 0u;
  bad |= !zero && (!ok || mag > (neg ? 128u : 127u));  // 0 < |v| < 1, fractions, |v| >= 128/256, inf, NaN
  return zero ? 0u : ((neg ? (0u - mag) : mag) & 0xffu);
}

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

// Static schedule over CTA pairs: pair `pid` of `np` takes tiles 2 (r np + pid) + {0, 1} in round r
// (rank 0 = pair leader, rank 1 = peer).  A CTA whose tile is past the end still runs the pipeline
// (X reads as zeros, no output) while its partner has a real tile.
struct Sched {
  int pid, np, rank, rounds;
  __device__ Sched(int num_tiles, int rank_) {
    rank = rank_;
    pid = (int)(blockIdx.x >> 1);
    np = (int)(gridDim.x >> 1);
    rounds = (num_tiles + 2 * np - 1) / (2 * np);
  }
  __device__ int tile(int r) const { return 2 * (r * np + pid) + rank; }
  __device__ bool pair_active(int r, int num_tiles) const { return 2 * (r * np + pid) < num_tiles; }
};

__device__ __forceinline__ void timed_wait(uint64_t* bar, uint32_t ph, long long* acc) {
  if (acc) {
    const long long t0 = clock64();
    mbar_wait(bar, ph);
    *acc += clock64() - t0;
  } else {
    mbar_wait(bar, ph);
  }
}

// K chunk order of step i: forward on even, reverse on odd steps (zig-zag), so each pass over the
// X panel starts where the previous one ended and re-reads hit L2.  The digit products are
// exact integers, so the order does not change any bit of the result.
__device__ __forceinline__ int chunk_at(int i, int nc, int k) { return (i & 1) ? nc - 1 - k : k; }

// One CTA pair (cluster of 2, one CTA per SM of a TPC) computes, per step (row blocks 2t and 2t+1, 32
// z rows each) and per 128-row K chunk, D_b[256 SNP columns x 224] += X^T[256 x 128] T_b^T[128 x 224]
// for both row blocks b, as tcgen05.mma.cta_group::2.kind::i8 (M = 256, N = 224, K = 32) issued by
// the leader: each CTA stages its own 128 X columns and half (112 rows) of both packed digit tiles,
// so a stage is 44 KiB per SM and the B operands are shared by the pair.  The two D regions live in
// TMEM ([0, 224) and [256, 480) of 512 columns; CTA r's lanes hold its own 128 columns) and are
// released one by one: the next step's region-0 MMAs start as soon as region 0 is drained, its
// region-1 MMAs are deferred (their stages held) until region 1 is.
// PL1C: pL + 1 when fixed at compile time (0: runtime); NA: accumulators per column
// (>= pL + 1 + pR); PR1: pR == 1 (Gram = z^2, no shuffles); ST: pipeline stages.
template <int PL1C, int NA, bool PR1, int ST>
__global__ void __cluster_dims__(2, 1, 1) __launch_bounds__(kThreads, 1)
    ozaki_trsm_gls_kernel(const __grid_constant__ CUtensorMap xmap, const __grid_constant__ CUtensorMap tmap,
                          const __grid_constant__ CUtensorMap vmap, const OzParams kp) {
  extern __shared__ __align__(1024) uint8_t smem_raw[];
  uint8_t* smem = (uint8_t*)(((uintptr_t)smem_raw + 1023) & ~(uintptr_t)1023);
  uint8_t* sA = smem;
  uint8_t* sB = sA + ST * kATile;                  // per stage: two B halves (two row blocks)
  uint64_t* bars = (uint64_t*)(sB + ST * 2 * kBHalf);
  uint64_t* full = bars;                 // used in the leader: all 60 KiB of a stage landed
  uint64_t* empty = bars + ST;           // both CTAs: the pair's MMAs released the stage
  uint64_t* tfull = bars + 2 * ST;       // both CTAs: accumulator buffer ready for the epilogue
  uint64_t* tempty = bars + 2 * ST + 2;  // used in the leader: both epilogues drained the buffer
  uint64_t* cvbar = bars + 2 * ST + 4;   // 2 per conv warp: its staging buffers landed
  uint32_t* tslot = (uint32_t*)(cvbar + 2 * kConvWarps);
  uint8_t* cvbuf = (uint8_t*)(tslot + 4);  // 2 x kCvBuf per conv warp (16-byte aligned)

  // A gated launch (this chunk is not integer: the FP64 kernel solves it) still runs its
  // convert-ahead job -- the next chunk depends on it -- but no tile.
  const int nflag = kp.gate ? *(volatile const int*)kp.gate : 0;  // uniform across the grid
  const bool gated = kp.pflag ? nflag >= kp.gate_all : nflag != 0;
  const bool masked = kp.pflag && nflag != 0;  // some problems of this launch belong to the FP64 kernel
  if (!gated && kp.ran && blockIdx.x == 0 && threadIdx.x == 0) atomicAdd(kp.ran, 1ull);

  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const uint32_t rank = cluster_ctarank();
  const bool leader = rank == 0;
  if (threadIdx.x == 0) {
    for (int s = 0; s < ST; ++s) {
      mbar_init(&full[s], 1);
      mbar_init(&empty[s], 1);
    }
    for (int b = 0; b < 2; ++b) {
      mbar_init(&tfull[b], 1);
      mbar_init(&tempty[b], 2 * kEpiWarps);
    }
    for (int b = 0; b < 2 * kConvWarps; ++b) mbar_init(&cvbar[b], 1);
    fence_barrier_init();
  }
  if (warp == 1) tmem_alloc_pair(tslot, kTmemCols);
  tc_fence_before();
  __syncthreads();
  cluster_sync_all();  // barriers of both CTAs initialised before any remote arrive / complete_tx
  tc_fence_after();
  const uint32_t tbase = *tslot;
  const int cpt = 4 * kp.cpw;  // columns per tile (per CTA)
  const Sched sc(gated ? 0 : kp.num_tiles, (int)rank);

  // Steps: step t of a tile covers row blocks 2t and 2t+1 (the last one alone when NBR is odd); both
  // have the same K extent, so each X chunk is loaded once and multiplied by both row blocks' digit
  // tiles, into TMEM columns [0, 224) and [256, 480).  The step after the last is the V block.  The
  // accumulator region is single-buffered: the next step's MMAs wait until both epilogues drained it.
  const int nsteps = (kp.NBR + 1) / 2;
  // Split completion: region 0 gets its own tfull commit and the MMAs of region 1's last ST-1 stages
  // are deferred on purpose, so region 0's drain overlaps region 1's tail MMAs and the next step's
  // region-0 MMAs queue behind that tail.  Measured ~+1 % on configs 2 and 3 (for the 21-accumulator
  // variants only since their epilogue stopped being the bottleneck).
  constexpr bool kSplit = true;
#ifndef GLS_OZ_HOLD
#define GLS_OZ_HOLD (ST - 1)
#endif
  // stages the MMA issuer may hold for deferred region-1 MMAs: fewer leave more stages to prefetch into
  // but widen the TMEM hand-over bubbles (A/B: profiles/r02_ab_hold.txt -- ST - 1 is fastest)
  constexpr int kHold = GLS_OZ_HOLD;
  if (warp == 0) {
    // ------------------------------------------------------------ TMA producer (both CTAs)
    if (lane == 0) {
      prefetch_tmap(&xmap);
      prefetch_tmap(&tmap);
      prefetch_tmap(&vmap);
      int stage = 0;
      uint32_t ph = 0;
      long long tw = 0;
      long long* pw = kp.prof ? &tw : nullptr;
      const uint32_t full0 = mapa_shared(smem_u32(full), 0);  // leader's full[0]
      const uint64_t pol_keep = policy_evict_last(), pol_stream = policy_evict_first();
      for (int r = 0; r < sc.rounds; ++r) {
        if (!sc.pair_active(r, kp.num_tiles)) break;
        const int col0 = sc.tile(r) * cpt;
        for (int t = 0; t <= nsteps; ++t) {
          const bool vstep = t == nsteps;
          const int i0 = 2 * t;
          const int nrb = vstep ? 1 : (i0 + 1 < kp.NBR ? 2 : 1);
          const int nc = vstep ? kp.NC : (i0 >> 2) + 1;
#ifdef GLS_OZ_EXP_HALFB
          // EXPERIMENT (wrong results; timing only): one B half per stage, shared by both row blocks
          const uint32_t bbytes = vstep ? (uint32_t)kp.NV * (kKC / 2) : (uint32_t)kBHalf;
#else
          const uint32_t bbytes = vstep ? (uint32_t)kp.NV * (kKC / 2) : (uint32_t)nrb * kBHalf;
#endif
          for (int k = 0; k < nc; ++k) {
            const int c = chunk_at(t, nc, k);
            timed_wait(&empty[stage], ph ^ 1, pw);
            if (leader) mbar_arrive_expect_tx(&full[stage], 2 * (kATile + bbytes));
            const uint32_t fb = full0 + stage * 8;
            const uint64_t pol = c < kp.cpin ? pol_keep : pol_stream;
#pragma unroll
            for (int q = 0; q < 4; ++q)
              tma_2d_g2s_pair_hint(sA + stage * kATile + q * 4096, &xmap, c * kKC, col0 + q * kp.cpw, fb, pol);
            uint8_t* sb = sB + stage * (2 * kBHalf);
            if (vstep) {
              tma_2d_g2s_pair(sb, &vmap, 0, c * kp.NV + (int)rank * (kp.NV / 2), fb);
            } else {
#ifdef GLS_OZ_EXP_HALFB
              for (int sl = 0; sl < 1; ++sl) {
#else
              for (int sl = 0; sl < nrb; ++sl) {
#endif
                const int trow0 = (int)(oz_tile_offset(i0 + sl) * kBN) + (int)rank * (kBN / 2);
                tma_2d_g2s_pair(sb + sl * kBHalf, &tmap, 0, trow0 + c * kBN, fb);
              }
            }
            if (++stage == ST) {
              stage = 0;
              ph ^= 1;
            }
          }
        }
      }
      if (kp.prof) kp.prof[blockIdx.x * 8 + 0] = tw;
    }
  } else if (warp == 1) {
    // ------------------------------------------------------------ MMA issuer (leader only)
    if (leader && lane == 0) {
      int stage = 0;
      uint32_t ph = 0;
      uint32_t u0 = 0, u1 = 0;  // uses of accumulator regions 0 and 1 so far (barrier phases)
      const uint32_t a0 = smem_u32(sA), b0 = smem_u32(sB);
      long long twf = 0, twt = 0;
      long long* pf = kp.prof ? &twf : nullptr;
      long long* pt = kp.prof ? &twt : nullptr;
      const long long tstart = clock64();
      const uint32_t idv = idesc_i8(256, kp.NV);
      // the 4 K=32 MMAs of stage st (K chunk k of the step) into accumulator region sl
      auto issue = [&](int st, int k, int sl, uint32_t idesc) {
        const uint64_t ad = sdesc_k128(a0 + st * kATile);
#ifdef GLS_OZ_EXP_HALFB
        const uint64_t bd = sdesc_k128(b0 + st * (2 * kBHalf));
#else
        const uint64_t bd = sdesc_k128(b0 + st * (2 * kBHalf) + sl * kBHalf);
#endif
#pragma unroll
        for (int kk = 0; kk < kKC / 32; ++kk)
          mma_i8_pair(tbase + sl * 256, ad + (uint64_t)(2 * kk), bd + (uint64_t)(2 * kk), idesc, (k | kk) != 0);
      };
      for (int r = 0; r < sc.rounds; ++r) {
        if (!sc.pair_active(r, kp.num_tiles)) break;
        for (int t = 0; t <= nsteps; ++t) {
          const bool vstep = t == nsteps;
          const int i0 = 2 * t;
          const bool two = !vstep && i0 + 1 < kp.NBR;
          const int nc = vstep ? kp.NC : (i0 >> 2) + 1;
          const uint32_t idesc = vstep ? idv : kIdesc;
          timed_wait(&tempty[0], (u0++ & 1) ^ 1, pt);
          tc_fence_after();
          // Region 1 is drained after region 0 (the epilogue releases them one by one): until it is,
          // its MMAs are deferred -- the stages stay held -- while region 0's go ahead (and, with
          // kSplit, again over the step's last ST-1 stages).
          bool r1 = !two;
          int ndef = 0, dstage = 0, dk = 0;
          for (int k = 0; k < nc; ++k) {
            timed_wait(&full[stage], ph, pf);
            tc_fence_after();
            issue(stage, k, 0, idesc);
            if (k == nc - 1 && (kSplit || !two)) mma_commit_pair_mc(&tfull[0], 3);  // region 0 complete
            const bool hold = two && (!r1 || (kSplit && k >= nc - kHold));
            if (!hold) {
              if (two) issue(stage, k, 1, idesc);
              mma_commit_pair_mc(&empty[stage], 3);
            } else {
              if (ndef++ == 0) {
                dstage = stage;
                dk = k;
              }
              const bool late = kSplit && k >= nc - kHold;  // the tail: flush only when forced
              if (ndef == kHold || k == nc - 1 || (!late && mbar_test(&tempty[1], (u1 & 1) ^ 1))) {
                if (!r1) {
                  timed_wait(&tempty[1], (u1++ & 1) ^ 1, pt);
                  tc_fence_after();
                  r1 = true;
                }
                for (int d = 0, s2 = dstage; d < ndef; ++d, s2 = s2 + 1 == ST ? 0 : s2 + 1) {
                  issue(s2, dk + d, 1, idesc);
                  mma_commit_pair_mc(&empty[s2], 3);
                }
                ndef = 0;
              }
            }
            if (++stage == ST) {
              stage = 0;
              ph ^= 1;
            }
          }
          if (two) mma_commit_pair_mc(&tfull[kSplit ? 1 : 0], 3);  // region 1 (and, unsplit, 0) complete
        }
      }
      if (kp.prof) {
        kp.prof[blockIdx.x * 8 + 1] = twf;
        kp.prof[blockIdx.x * 8 + 2] = twt;
        kp.prof[blockIdx.x * 8 + 3] = clock64() - tstart;
      }
    }
  } else if (warp < 2 + kEpiWarps) {
    // ------------------------------------------------------------ epilogue (both CTAs)
    const int ew = warp - 2;
    const int q = warp & 3;      // TMEM lane quadrant this warp may access
    const int h = ew >> 2;       // which 16 of a row block's 32 z rows
    const int pl1 = PL1C > 0 ? PL1C : kp.pL + 1;
    const int as = pl1 + 1;        // aux row stride
    const int a_in = PR1 ? 0 : lane % kp.pR;  // position inside the group
    const uint32_t tlane = tbase + ((uint32_t)(q * 32) << 16);
    const uint32_t tempty0 = mapa_shared(smem_u32(tempty), 0);  // leader's tempty[0] (tempty[1]: + 8)
    double acc[NA];
    zero_acc(acc);
    uint32_t f0 = 0, f1 = 0;  // completions of tfull[0] / tfull[1] consumed (barrier phases)
    long long twe = 0, prof_drain = 0, prof_busy = 0;
    long long* pe = (kp.prof && ew == 0 && lane == 0) ? &twe : nullptr;
    auto release = [&](int sl) {  // this warp is done reading accumulator region sl
      tc_fence_before();
      __syncwarp();
      if (lane == 0) {
        if (leader)
          mbar_arrive(&tempty[sl]);
        else
          mbar_arrive_cluster(tempty0 + 8 * sl);
      }
    };
    // z rows 16 h .. 16 h + 15 of the row block in TMEM region `sl`: the 7 digit sums combined exactly
    // in int64 (two partial sums), then one FP64 rounding each
    // The region is released right after the last TMEM load completes (before the FP64 rounding), so
    // the MMA issuer's wait for it does not include this warp's arithmetic.
    auto drain = [&](int sl, double (&z)[16]) {
      const uint32_t tr = tlane + sl * 256 + h * 16;
#if defined(GLS_OZ_EXP_NODRAIN)
      // EXPERIMENT (wrong results; timing only): no TMEM traffic or arithmetic in the epilogue
      release(sl);
#pragma unroll
      for (int r = 0; r < 16; ++r) z[r] = 0.0;
#elif GLS_OZ_DRAIN_RT == 2
      if constexpr (PR1 && kDrainOneTrip) {
        // one TMEM round trip: all 7 digit loads in flight, one wait, release, then the arithmetic
        // (the 1-accumulator Gram variants have the registers for it: 148, no spills)
        int32_t d0[16], d1[16], d2[16], d3[16], d4[16], d5[16], d6[16];
        tmem_ld16(tr, d0);
        tmem_ld16(tr + 1 * kR, d1);
        tmem_ld16(tr + 2 * kR, d2);
        tmem_ld16(tr + 3 * kR, d3);
        tmem_ld16(tr + 4 * kR, d4);
        tmem_ld16(tr + 5 * kR, d5);
        tmem_ld16(tr + 6 * kR, d6);
        tmem_wait_ld();
        release(sl);
#pragma unroll
        for (int r = 0; r < 16; ++r) {
          const long long hi = (long long)d0[r] * 16777216LL + (long long)d1[r] * 65536LL +
                               (long long)d2[r] * 256LL + (long long)d3[r];
          const long long lo = (long long)d4[r] * 65536LL + (long long)d5[r] * 256LL + (long long)d6[r];
          z[r] = fma((double)hi, 16777216.0, (double)lo);
        }
        return;
      }
      // two TMEM round trips: digits 0-3 (the high part), then digits 4-6
      long long hi[16];
      {
        int32_t d0[16], d1[16], d2[16], d3[16];
        tmem_ld16(tr, d0);
        tmem_ld16(tr + 1 * kR, d1);
        tmem_ld16(tr + 2 * kR, d2);
        tmem_ld16(tr + 3 * kR, d3);
        tmem_wait_ld();
#pragma unroll
        for (int r = 0; r < 16; ++r)
          hi[r] = (long long)d0[r] * 16777216LL + (long long)d1[r] * 65536LL + (long long)d2[r] * 256LL +
                  (long long)d3[r];
      }
      {
        int32_t d4[16], d5[16], d6[16];
        tmem_ld16(tr + 4 * kR, d4);
        tmem_ld16(tr + 5 * kR, d5);
        tmem_ld16(tr + 6 * kR, d6);
        tmem_wait_ld();
        release(sl);
#pragma unroll
        for (int r = 0; r < 16; ++r) {
          const long long lo = (long long)d4[r] * 65536LL + (long long)d5[r] * 256LL + (long long)d6[r];
          z[r] = fma((double)hi[r], 16777216.0, (double)lo);
        }
      }
#else
      long long hi[16], lo[16];
      int32_t va[16], vb[16];
      // two digits per TMEM round trip (4 waits instead of 7)
      tmem_ld16(tr, va);
      tmem_ld16(tr + 1 * kR, vb);
      tmem_wait_ld();
#pragma unroll
      for (int r = 0; r < 16; ++r) hi[r] = (long long)va[r] * 16777216LL + (long long)vb[r] * 65536LL;
      tmem_ld16(tr + 2 * kR, va);
      tmem_ld16(tr + 3 * kR, vb);
      tmem_wait_ld();
#pragma unroll
      for (int r = 0; r < 16; ++r) hi[r] += (long long)va[r] * 256LL + (long long)vb[r];
      tmem_ld16(tr + 4 * kR, va);
      tmem_ld16(tr + 5 * kR, vb);
      tmem_wait_ld();
#pragma unroll
      for (int r = 0; r < 16; ++r) lo[r] = (long long)va[r] * 65536LL + (long long)vb[r] * 256LL;
      tmem_ld16(tr + 6 * kR, va);
      tmem_wait_ld();
      release(sl);
#pragma unroll
      for (int r = 0; r < 16; ++r) z[r] = fma((double)hi[r], 16777216.0, (double)(lo[r] + (long long)va[r]));
#endif
    };
    // acc layout: the Gram row at the bottom, acc[b] (b < pR), the V block's outputs at the top,
    // acc[NA - 1 - w] (w < pL + 1): static register indices for both whatever pL and pR are.
    // Gram of z rows of row block i: acc[b] += zr z_b over the group's columns (S_BR, row a_in)
    // sigma of the warp's 16 rows of row block i, lane r holding row r: loaded before the step's
    // TMEM wait (a global load from an SM running this kernel takes microseconds), broadcast below
    auto load_sigma = [&](int i) -> double {
      return lane < 16 ? __ldg(kp.aux + (int64_t)(i * kR + h * 16 + lane) * as) : 0.0;
    };
    auto reduce = [&](double sig, double (&z)[16]) {
#pragma unroll
      for (int r = 0; r < 16; ++r) z[r] *= __shfl_sync(0xffffffffu, sig, r);
      if (PR1) {
#pragma unroll
        for (int r = 0; r < 16; ++r) acc[0] = fma(z[r], z[r], acc[0]);
      } else {
        // b outside, rows inside: 16 independent shuffle + FMA chains per b (the rows' order per
        // accumulator is unchanged)
#pragma unroll
        for (int b = 0; b < NA; ++b) {
          if (b >= kp.pR) break;  // uniform
#pragma unroll
          for (int r = 0; r < 16; ++r)
            acc[b] = fma(z[r], __shfl_sync(0xffffffffu, z[r], lane - a_in + b), acc[b]);
        }
      }
    };
    for (int rr = 0; rr < sc.rounds; ++rr) {
      if (!sc.pair_active(rr, kp.num_tiles)) break;
      const int tile = sc.tile(rr);
      for (int t = 0; t < nsteps; ++t) {
        const int i0 = 2 * t;
        const bool two = i0 + 1 < kp.NBR;
        const double sig0 = load_sigma(i0), sig1 = two ? load_sigma(i0 + 1) : 0.0;
        timed_wait(&tfull[0], f0++ & 1, pe);
        const long long tw0 = pe ? clock64() : 0;
        tc_fence_after();
        // one z block live at a time; each region is waited for, drained and released on its own:
        // region 0 completes first and its release lets the next step's MMAs start while region 1's
        // last MMAs still run
        double z[16];
        drain(0, z);
        if (pe) prof_drain += clock64() - tw0;
        reduce(sig0, z);
        if (two) {
          if (kSplit) {
            timed_wait(&tfull[1], f1++ & 1, pe);
            tc_fence_after();
          }
          drain(1, z);
          reduce(sig1, z);
        }
        if (pe) prof_busy += clock64() - tw0;
      }
      {  // V block: S_BL[w] (w < pL) and b_B (w = pL) of this column = 2^-(e_w+48) sum_s 256^(6-s) D[8w+s]
        timed_wait(&tfull[0], f0++ & 1, pe);
        tc_fence_after();
        if (h == 0) {
#pragma unroll
          for (int w = 0; w < NA; ++w) {
            if (w < pl1) {
              int32_t v[8];
              tmem_ld8(tlane + 8 * w, v);
              tmem_wait_ld();
              const long long vh = (long long)v[0] * 16777216LL + (long long)v[1] * 65536LL +
                                   (long long)v[2] * 256LL + (long long)v[3];
              const long long vl = (long long)v[4] * 65536LL + (long long)v[5] * 256LL + (long long)v[6];
              acc[NA - 1 - w] = fma((double)vh, 16777216.0, (double)vl) * __ldg(kp.vscale + w);
            }
          }
        }
        release(0);
      }
      // ---- per-tile finalisation: sum the two row halves, assemble S_i, posv.  The h = 1 warps hand
      // their sums over through TMEM columns no MMA writes ([224, 256) and [480, 512)), same lanes.
      named_bar_sync(1, kEpiWarps * 32);
      if (h == 1) {
#pragma unroll
        for (int w = 0; w < NA; ++w) tmem_st_f64(tlane + xcol(w), acc[w]);
        tmem_wait_st();
        tc_fence_before();
      }
      named_bar_sync(2, kEpiWarps * 32);
      if (h == 0) {
        tc_fence_after();
#pragma unroll
        for (int w = 0; w < NA; ++w) acc[w] += tmem_ld_f64(tlane + xcol(w));
        const int64_t col = (int64_t)tile * cpt + q * kp.cpw + lane;
        const bool owner = lane < kp.cpw && a_in == 0 && col < kp.cols && !(masked && kp.pflag[col / kp.pR]);
        const int p = kp.p, pL = kp.pL, pR = kp.pR;
        double S[400];
        double rhs[20];
        // large p: the record goes to global memory and oz_posv_kernel solves after this kernel (a
        // 20 x 20 Cholesky in local memory here would stall the next tile's first step)
        double* rec = kp.s_ws ? kp.s_ws + (col / pR) * (int64_t)(pR * (pL + pR + 1)) : nullptr;
        if (owner && !rec) {
          for (int a2 = 0; a2 < pL; ++a2) {
            for (int b2 = 0; b2 < pL; ++b2) S[a2 + b2 * 20] = __ldg(kp.G + a2 + b2 * pl1);
            rhs[a2] = __ldg(kp.G + a2 + pL * pl1);
          }
        }
        // the group's columns are lanes lane .. lane + pR - 1 of this warp (groups never straddle warps)
#pragma unroll
        for (int a2 = 0; a2 < (PR1 ? 1 : 20); ++a2) {
          if (a2 < pR) {
#pragma unroll
            for (int w = 0; w < NA; ++w) {
              const double v = PR1 ? acc[w] : __shfl_sync(0xffffffffu, acc[w], lane + a2);
              if (owner && rec) {
                if (w < pR) rec[pR * pL + a2 * pR + w] = v;
                const int wv = NA - 1 - w;
                if (wv < pL) rec[a2 * pL + wv] = v;
                if (wv == pL) rec[pR * pL + pR * pR + a2] = v;
              } else if (owner) {
                if (w < pR) S[(pL + a2) + (pL + w) * 20] = v;  // S_BR
                const int wv = NA - 1 - w;                      // V output wv: S_BL (wv < pL), b_B
                if (wv < pL) {
                  S[(pL + a2) + wv * 20] = v;
                  S[wv + (pL + a2) * 20] = v;
                }
                if (wv == pL) rhs[pL + a2] = v;
              }
            }
          }
        }
        if (owner && !rec)
          posv_store(S, rhs, p, kp.b_out + (col / pR) * p, kp.status_out ? kp.status_out + col / pR : nullptr);
      }
      zero_acc(acc);
    }
    if (pe) {
      kp.prof[blockIdx.x * 8 + 4] = twe;
      kp.prof[blockIdx.x * 8 + 5] = prof_drain;
      kp.prof[blockIdx.x * 8 + 6] = prof_busy;
    }
  } else if (kp.cv_X) {
    // ------------------------------------------------------------ convert-ahead (both CTAs)
    // FP64 X of the next chunk -> int8, piece by piece (kCvRows rows of one column): a bulk copy
    // into shared memory (bytes in flight without registers: plain loads from an SM running this
    // kernel take microseconds), integer bit tests, 2-byte stores.  Pieces are dealt round-robin
    // over all conv warps of the grid; two buffers per warp keep one copy in flight while the other
    // piece is converted.
    const int cw = warp - (2 + kEpiWarps);
    const int64_t gw = (int64_t)blockIdx.x * kConvWarps + cw, nw = (int64_t)gridDim.x * kConvWarps;
    const int64_t n = kp.n, ppc = (n + kCvRows - 1) / kCvRows;
    const int64_t units = kp.cv_cols * ppc;
    uint8_t* const buf0 = cvbuf + (size_t)cw * 2 * kCvBuf;
    uint64_t* const bar0 = cvbar + 2 * cw;
    // the FP64 source is read once and the int8 copy is next read a launch later: both L2::evict_first,
    // so this stream does not push the pinned X panels and the digit tiles out of L2
    const uint64_t pol_once = policy_evict_first();
    auto piece = [&](int64_t u, int64_t& c, int64_t& r0, int& rows) {
      c = u / ppc;
      r0 = (u - c * ppc) * kCvRows;
      rows = (int)(n - r0 < kCvRows ? n - r0 : kCvRows);
    };
    auto issue = [&](int64_t u, int b) {
      int64_t c, r0;
      int rows;
      piece(u, c, r0, rows);
      const uint32_t bytes = (uint32_t)(rows * 8) & ~15u;  // an odd last row is read directly
      if (lane == 0) {
        if (bytes) {
          mbar_arrive_expect_tx(&bar0[b], bytes);
          if (kCvHint)
            bulk_g2s_hint(buf0 + b * kCvBuf, kp.cv_X + c * kp.cv_ldx + r0, bytes, &bar0[b], pol_once);
          else
            bulk_g2s(buf0 + b * kCvBuf, kp.cv_X + c * kp.cv_ldx + r0, bytes, &bar0[b]);
        } else {
          mbar_arrive(&bar0[b]);  // a one-row piece: nothing to copy
        }
      }
    };
    int bad = 0;
    uint32_t ph0 = 0, ph1 = 0;
    if (gw < units) issue(gw, 0);
    if (gw + nw < units) issue(gw + nw, 1);
    int b = 0;
    for (int64_t u = gw; u < units; u += nw, b ^= 1) {
      mbar_wait(&bar0[b], b ? ph1 : ph0);
      if (b) ph1 ^= 1; else ph0 ^= 1;
      int64_t c, r0;
      int rows;
      piece(u, c, r0, rows);
      const double* sv = (const double*)(buf0 + b * kCvBuf);
      int8_t* dst = kp.cv_X8 + c * kp.cv_ld8 + r0;
      int pb = 0;  // this piece holds a value the int8 path cannot take
#pragma unroll 4
      for (int k = 0; k < kCvRows / 64; ++k) {  // lane holds rows 2 lane + 64 k, +1
        const int r = 2 * lane + 64 * k;
        if (r + 2 <= rows) {
          const double2 v = *(const double2*)(sv + r);
          const uint16_t w = (uint16_t)(to_i8_bits(v.x, pb) | to_i8_bits(v.y, pb) << 8);
          if (kCvHint)
            st_u16_hint(dst + r, w, pol_once);
          else
            *(uint16_t*)(dst + r) = w;
        } else if (r < rows) {  // the column's odd last row: not in the bulk copy
          dst[r] = (int8_t)to_i8_bits(__ldg(kp.cv_X + c * kp.cv_ldx + r0 + r), pb);
        }
      }
      if (kp.cv_pflag) {  // flag the piece's problem; its first flag counts it in *cv_flag
        if (__any_sync(0xffffffffu, pb) && lane == 0 && atomicExch(kp.cv_pflag + c / kp.pR, 1) == 0)
          atomicAdd(kp.cv_flag, 1);
      } else {
        bad |= pb;
      }
      __syncwarp();
      fence_proxy_async();  // this warp's reads of the buffer before the copy that overwrites it
      if (u + 2 * nw < units) issue(u + 2 * nw, b);
    }
    if (__any_sync(0xffffffffu, bad) && lane == 0) atomicOr(kp.cv_flag, 1);
  }
  tc_fence_before();
  __syncthreads();
  cluster_sync_all();  // neither CTA leaves while its partner may still signal or fill it
  if (warp == 1) tmem_dealloc_pair(tbase, kTmemCols);
}

// ---------------------------------------------------------------- setup kernels
// Every setup kernel reads T through a column-ownership map (ColOwn, gls_internal.cuh): the single-GPU
// create owns every column (identity map); the distributed create (dist_create.cu) gives each rank the
// column blocks j with j % nranks == rank, stored contiguously, and a kernel only touches owned columns.

// Row maxima over owned columns: rowmax_r = max_{j <= r, j owned} |T_rj|.  One CTA per 32 rows,
// 8 column strands per row (T column-major, so a warp reads 32 consecutive rows of one column).
__global__ void oz_rowmax_kernel(const double* __restrict__ T, int64_t ld, int64_t n, ColOwn own,
                                 double* __restrict__ rowmax) {
  __shared__ double sm[8][32];
  const int rl = threadIdx.x & 31, strand = threadIdx.x >> 5;
  const int64_t r = (int64_t)blockIdx.x * 32 + rl;
  double mx = 0.0;
  if (r < n) {
#pragma unroll 8
    for (int64_t j = strand; j <= r; j += 8)
      if (own.owned(j)) mx = fmax(mx, fabs(T[r + own.local(j) * ld]));
  }
  sm[strand][rl] = mx;
  __syncthreads();
  if (strand == 0) {
    for (int k = 1; k < 8; ++k) mx = fmax(mx, sm[k][rl]);
    rowmax[r] = mx;  // rows >= n: 0
  }
}

// Row scale from the row maximum: e_r with max_j |T_rj| 2^e_r <= 127; sigma_r = 2^-(e_r + 48).
__device__ __forceinline__ void scale_of(double mx, int& e, double& sig) {
  e = 0;
  sig = 0.0;
  if (mx > 0.0) {
    int E;
    const double f = frexp(mx, &E);  // mx = f 2^E, f in [0.5, 1)
    e = (f * 128.0 <= 127.0) ? 7 - E : 6 - E;
    sig = ldexp(1.0, -(e + 48));
  }
}
__global__ void oz_rowscale_kernel(const double* __restrict__ rowmax, int64_t rows, int* __restrict__ escale,
                                   double* __restrict__ aux, int as) {
  for (int64_t r = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; r < rows; r += (int64_t)gridDim.x * blockDim.x) {
    int e;
    double sig;
    scale_of(rowmax[r], e, sig);
    escale[r] = e;
    aux[r * as] = sig;  // rows >= n: sigma = 0 (their T digits are zero too)
  }
}

// Digits of every element of every packed tile whose K chunk is owned: tile (i, c) holds rows
// 32i..32i+31, K columns 128c..128c+127; B row s*32 + rr holds digit s of row 32i + rr (plain
// 128-byte rows; the TMA load applies the 128-byte swizzle).  Tiles of chunks owned by other ranks
// are not written (the distributed create sums the ranks' zero-initialised T8 buffers).
// T is column-major and the digit rows run along K, so the 32 x 128 block goes through shared memory:
// read with a warp on 32 consecutive rows of one column (256 contiguous bytes), then thread (rr, kq)
// converts K 16kq..16kq+15 of row rr and stores 16 bytes per digit -- the 8 threads of a row write its
// 128 contiguous bytes.  Rows are padded to kPackLd doubles (even: 16-byte LDS; 2 extra doubles per
// 16-K group, so a quarter-warp's LDS.128 of 8 groups hit distinct banks).
constexpr int kPackGrp = 18;                 // 16 K + 2 pad doubles per group
constexpr int kPackLd = 8 * kPackGrp + 2;    // 146 doubles per row
__global__ void __launch_bounds__(256) oz_pack_kernel(const double* __restrict__ T, int64_t ld, int64_t n,
                                                      ColOwn own, const int* __restrict__ escale, int NBR,
                                                      int8_t* __restrict__ T8) {
  __shared__ __align__(16) double sT[kR * kPackLd];
  const int64_t tile = blockIdx.x;
  int i = (int)sqrt(2.0 * (double)tile);  // invert oz_tile_offset
  while (i > 0 && oz_tile_offset(i) > tile) --i;
  while (i + 1 <= NBR && oz_tile_offset(i + 1) <= tile) ++i;
  const int c = (int)(tile - oz_tile_offset(i));
  if (!own.owned((int64_t)c * kKC)) return;  // a chunk lies inside one column block (nb % 128 == 0)
  {
    const int rr = threadIdx.x & 31;
    const int64_t r = (int64_t)i * kR + rr;
    double v[kR * kKC / 256];
#pragma unroll
    for (int q = 0; q < kR * kKC / 256; ++q) {  // element (rr, k), k = warp + 8 q
      const int k = (threadIdx.x >> 5) + 8 * q;
      const int64_t j = (int64_t)c * kKC + k;
      v[q] = (r < n && j <= r) ? T[r + own.local(j) * ld] : 0.0;
    }
#pragma unroll
    for (int q = 0; q < kR * kKC / 256; ++q) {
      const int k = (threadIdx.x >> 5) + 8 * q;
      sT[rr * kPackLd + (k >> 4) * kPackGrp + (k & 15)] = v[q];
    }
  }
  __syncthreads();
  const int rr = threadIdx.x >> 3, kq = threadIdx.x & 7;
  const int64_t r = (int64_t)i * kR + rr;
  const int e = (r < n) ? escale[r] : 0;
  const double* src = sT + rr * kPackLd + kq * kPackGrp;
  uint32_t d[kNSL][4];
#pragma unroll
  for (int s = 0; s < kNSL; ++s) d[s][0] = d[s][1] = d[s][2] = d[s][3] = 0;
#pragma unroll
  for (int kk = 0; kk < 16; kk += 2) {
    const double2 x2 = *(const double2*)(src + kk);
#pragma unroll
    for (int h = 0; h < 2; ++h) {
      long long V = llrint(ldexp(h ? x2.y : x2.x, e + 48));
      const int k = kk + h;
#pragma unroll
      for (int s = kNSL - 1; s > 0; --s) {  // signed base-256 digits, least significant first
        const int8_t lo = (int8_t)(V & 0xff);
        d[s][k >> 2] |= (uint32_t)(uint8_t)lo << (8 * (k & 3));
        V = (V - lo) >> 8;
      }
      d[0][k >> 2] |= (uint32_t)(uint8_t)(int8_t)V << (8 * (k & 3));  // |top| <= 127
    }
  }
  int8_t* dst = T8 + tile * (int64_t)kOzTileBytes;
#pragma unroll
  for (int s = 0; s < kNSL; ++s)
    *(uint4*)(dst + (s * kR + rr) * kKC + kq * 16) = make_uint4(d[s][0], d[s][1], d[s][2], d[s][3]);
}

// Column maxima of V = M^{-1} [X_L | y] (n x pl1) over the rows of owned chunks.  One CTA per column.
__global__ void oz_vmax_kernel(const double* __restrict__ V, int64_t n, ColOwn own, double* __restrict__ vmax) {
  __shared__ double sm[256];
  const int w = blockIdx.x;
  double mx = 0.0;
  for (int64_t r = threadIdx.x; r < n; r += blockDim.x)
    if (own.owned(r)) mx = fmax(mx, fabs(V[r + w * n]));
  sm[threadIdx.x] = mx;
  __syncthreads();
  for (int k = 128; k > 0; k >>= 1) {
    if (threadIdx.x < k) sm[threadIdx.x] = fmax(sm[threadIdx.x], sm[threadIdx.x + k]);
    __syncthreads();
  }
  if (threadIdx.x == 0) vmax[w] = sm[0];
}
// Column scales of V: e_w with max_r |V_rw| 2^e_w <= 127.
// vmax and vscale may alias (each thread reads its maximum before writing its scale)
__global__ void oz_vscale_kernel(const double* vmax, int pl1, int* __restrict__ ev, double* vscale) {
  const int w = threadIdx.x;
  if (w < pl1) {
    int e;
    double sig;
    scale_of(vmax[w], e, sig);
    ev[w] = e;
    vscale[w] = sig;
  }
}

// Digit tiles of V for the owned chunks: chunk c holds NV rows of 128 bytes (K = rows 128c..128c+127
// of V); row 8w + s is digit s (most significant first) of column w; rows 8w + 7 and w >= pl1 are
// zero.  Plain layout: the TMA load applies the 128-byte swizzle.
__global__ void oz_vpack_kernel(const double* __restrict__ V, int64_t n, int pl1, ColOwn own,
                                const int* __restrict__ ev, int NV, int8_t* __restrict__ V8) {
  const int c = blockIdx.x;
  if (!own.owned((int64_t)c * kKC)) return;
  int8_t* dst = V8 + (int64_t)c * NV * kKC;
  for (int idx = threadIdx.x; idx < (NV / 8) * kKC; idx += blockDim.x) {
    const int w = idx / kKC, k = idx % kKC;
    const int64_t r = (int64_t)c * kKC + k;
    long long X = 0;
    if (w < pl1 && r < n) X = llrint(ldexp(V[r + w * n], ev[w] + 48));
    int8_t d[8];
    d[7] = 0;
#pragma unroll
    for (int s2 = kNSL - 1; s2 > 0; --s2) {
      const int8_t lo = (int8_t)(X & 0xff);
      d[s2] = lo;
      X = (X - lo) >> 8;
    }
    d[0] = (int8_t)X;
#pragma unroll
    for (int s2 = 0; s2 < 8; ++s2) dst[(8 * w + s2) * kKC + k] = d[s2];
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

// x -> int8 bits for an integer-valued double in [-128, 127], by integer operations on its bits only
// (FP64 arithmetic contends with the tensor core on this part); bad |= any other value.

// X (double, column-major, ld = ldx) -> X8 (int8, column-major, ld = ld8), flagging any value that
// is not an integer in [-128, 127] (NaN included); X8's padding rows [n, ld8) are not written (the
// solve kernel's TMA reads rows < n only).  Integer bit tests only, no FP64 arithmetic.
// A warp converts pieces of 256 rows of one column: lane l holds rows 2l, 2l+1 (+64 k, k < 4), so
// every load instruction reads 512 contiguous bytes and every store writes 64; kInflight pieces are
// in flight per warp.  X columns start 16-byte aligned (ldx even, base 16-byte aligned).
// Work-stealing: blocks claim units of kConvCols columns from an atomic counter (work[0], zeroed
// with the flag).
constexpr int kConvCols = 16;
constexpr int kConvThreads = 256;
constexpr int kInflight = 2;  // 256-row pieces in flight per warp
constexpr int kConvSmem = 8192;

__global__ void __launch_bounds__(kConvThreads, 4) oz_x_to_i8_kernel(const double* __restrict__ X, int64_t ldx,
                                                                     int64_t n, int64_t cols, int8_t* __restrict__ X8,
                                                                     int64_t ld8, int* __restrict__ flag,
                                                                     unsigned long long* __restrict__ work,
                                                                     int* __restrict__ pflag, int pR) {
  __shared__ unsigned long long unit;
  const int64_t nunits = (cols + kConvCols - 1) / kConvCols;
  const uint32_t per_col = (uint32_t)((n + 255) >> 8);  // 256-row pieces per column
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  constexpr int kWarps = kConvThreads / 32;
  int bad = 0;
  for (;;) {
    if (threadIdx.x == 0) unit = atomicAdd(work, 1ull);
    __syncthreads();
    const int64_t u = (int64_t)unit;
    __syncthreads();
    if (u >= nunits) break;
    const int64_t c0 = u * kConvCols;
    const uint32_t nc = (cols - c0 < kConvCols) ? (uint32_t)(cols - c0) : (uint32_t)kConvCols;
    const uint32_t total = per_col * nc;
    for (uint32_t q0 = warp; q0 < total; q0 += kInflight * kWarps) {
      double2 v[kInflight][4];
#pragma unroll
      for (int j = 0; j < kInflight; ++j) {
        const uint32_t q = q0 + j * kWarps;
        const uint32_t c = q / per_col;
        const int64_t r = (int64_t)(q - c * per_col) * 256;
        if (q < total && r + 256 <= n) {
          const double2* src = (const double2*)(X + (c0 + c) * ldx + r) + lane;
#pragma unroll
          for (int k = 0; k < 4; ++k) v[j][k] = __ldcs(src + 32 * k);
        }
      }
#pragma unroll
      for (int j = 0; j < kInflight; ++j) {
        const uint32_t q = q0 + j * kWarps;
        if (q >= total) continue;
        const uint32_t c = q / per_col;
        const int64_t r = (int64_t)(q - c * per_col) * 256;
        const double* src = X + (c0 + c) * ldx + r;
        int8_t* dst = X8 + (c0 + c) * ld8 + r;
        int pb = 0;  // this piece holds a value the int8 path cannot take
        if (r + 256 <= n) {
#pragma unroll
          for (int k = 0; k < 4; ++k)
            *(uint16_t*)(dst + 2 * lane + 64 * k) =
                (uint16_t)(to_i8_bits(v[j][k].x, pb) | to_i8_bits(v[j][k].y, pb) << 8);
        } else {  // the ragged end of the column
          for (int64_t e = lane; r + e < n; e += 32) dst[e] = (int8_t)to_i8_bits(__ldcs(src + e), pb);
        }
        if (pflag) {  // flag the piece's problem; its first flag counts it in *flag
          if (__any_sync(0xffffffffu, pb) && lane == 0 && atomicExch(pflag + (c0 + c) / pR, 1) == 0)
            atomicAdd(flag, 1);
        } else {
          bad |= pb;
        }
      }
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

template <int PL1C, int NA, bool PR1>
cudaError_t launch_oz_variant(cudaStream_t s, const CUtensorMap& xmap, const CUtensorMap& tmap,
                              const CUtensorMap& vmap, const OzParams& kp, int num_sms) {
  constexpr int kFixed = 1024 + 512 + 2 * kConvWarps * kCvBuf;  // alignment, barriers, conv staging
  constexpr int kStage = kATile + 2 * kBHalf;  // X chunk + the digit halves of two row blocks
  constexpr int ST = (232448 - kFixed) / kStage < 8 ? (232448 - kFixed) / kStage : 8;
  static_assert(ST >= 4, "shared memory budget");
  constexpr int smem = ST * kStage + kFixed;
  auto kern = ozaki_trsm_gls_kernel<PL1C, NA, PR1, ST>;
  static int max_pairs_dev[64];  // per device: cluster occupancy of this variant
  int dev = 0;
  cudaGetDevice(&dev);
  if (dev < 0 || dev >= 64) dev = 0;
  if (first_use_on_device((const void*)kern)) {
    cudaError_t e = cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, smem);
    if (e != cudaSuccess) return e;
    int mp = num_sms / 2;
    cudaLaunchConfig_t cfg = {};
    cfg.gridDim = dim3((unsigned)(2 * mp));
    cfg.blockDim = dim3(kThreads);
    cfg.dynamicSmemBytes = smem;
    int nc = 0;
    if (cudaOccupancyMaxActiveClusters(&nc, (void*)kern, &cfg) == cudaSuccess && nc > 0 && nc < mp) mp = nc;
    cudaGetLastError();
    max_pairs_dev[dev] = mp;
  }
  int max_pairs = max_pairs_dev[dev] > 0 ? max_pairs_dev[dev] : num_sms / 2;
  // GLS_OZ_PAIRS (tests): fewer CTA pairs than the machine holds -- a different tile-to-pair schedule and
  // different timing, under which the results must not change by a bit
  static const int pairs_cap = getenv("GLS_OZ_PAIRS") ? atoi(getenv("GLS_OZ_PAIRS")) : 0;
  if (pairs_cap > 0 && pairs_cap < max_pairs) max_pairs = pairs_cap;
  const int need = (kp.num_tiles + 1) / 2;
  const int np = need < max_pairs ? need : max_pairs;
  kern<<<2 * np, kThreads, smem, s>>>(xmap, tmap, vmap, kp);
  return cudaGetLastError();
}

// Alg. 5 line 11 for the records the int8 kernel left in s_ws (large p): S_i = [[S_TL, S_BL^T],
// [S_BL, S_BR]], [b_T; b_B] with S_TL, b_T from G, then the same posv_store as in the kernel.
__global__ void __launch_bounds__(128) oz_posv_kernel(const double* __restrict__ rec, const double* __restrict__ G,
                                                      int pL, int pR, int64_t m_blk, const int* gate,
                                                      const int* __restrict__ pflag, int64_t gate_all,
                                                      double* __restrict__ b_out, int32_t* __restrict__ st) {
  const int nflag = gate ? *(volatile const int*)gate : 0;
  if (pflag ? nflag >= gate_all : nflag != 0) return;
  const bool masked = pflag && nflag != 0;
  const int p = pL + pR, pl1 = pL + 1;
  const int64_t rs = (int64_t)pR * (pL + pR + 1);
  for (int64_t g = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; g < m_blk; g += (int64_t)gridDim.x * blockDim.x) {
    if (masked && pflag[g]) continue;  // the FP64 kernel solves this problem
    double S[400];
    double rhs[20];
    for (int a2 = 0; a2 < pL; ++a2) {
      for (int b2 = 0; b2 < pL; ++b2) S[a2 + b2 * 20] = G[a2 + b2 * pl1];
      rhs[a2] = G[a2 + pL * pl1];
    }
    const double* r = rec + g * rs;
    for (int a2 = 0; a2 < pR; ++a2) {
      for (int w = 0; w < pL; ++w) {
        S[(pL + a2) + w * 20] = r[a2 * pL + w];
        S[w + (pL + a2) * 20] = r[a2 * pL + w];
      }
      for (int b2 = 0; b2 < pR; ++b2) S[(pL + a2) + (pL + b2) * 20] = r[pR * pL + a2 * pR + b2];
      rhs[pL + a2] = r[pR * pL + pR * pR + a2];
    }
    posv_store(S, rhs, p, b_out + g * p, st ? st + g : nullptr);
  }
}

__global__ void __launch_bounds__(256) oz_repack_kernel(const int8_t* __restrict__ src, int64_t n, int64_t rows,
                                                        int8_t* __restrict__ dst, int64_t ld8) {
  for (int64_t r = blockIdx.x; r < rows; r += gridDim.x)
    for (int64_t j = threadIdx.x; j < n; j += blockDim.x) dst[r * ld8 + j] = src[r * n + j];
}

}  // namespace

int64_t oz_total_tiles(int64_t NBR) { return oz_tile_offset(NBR); }

void oz_rowmax(cudaStream_t s, const double* T, int64_t ld, int64_t n, ColOwn own, double* rowmax, int64_t* lc) {
  const int NBR = (int)((n + kR - 1) / kR);
  oz_rowmax_kernel<<<NBR, 256, 0, s>>>(T, ld, n, own, rowmax);
  if (lc) ++*lc;
}
void oz_rowscale(cudaStream_t s, const double* rowmax, int64_t n, int* escale, double* aux, int pl1, int64_t* lc) {
  const int64_t rows = (n + kR - 1) / kR * kR;
  oz_rowscale_kernel<<<(unsigned)((rows + 255) / 256), 256, 0, s>>>(rowmax, rows, escale, aux, pl1 + 1);
  if (lc) ++*lc;
}
void oz_pack(cudaStream_t s, const double* T, int64_t ld, int64_t n, ColOwn own, const int* escale, int8_t* T8,
             int64_t* lc) {
  const int NBR = (int)((n + kR - 1) / kR);
  oz_pack_kernel<<<(unsigned)oz_total_tiles(NBR), 256, 0, s>>>(T, ld, n, own, escale, NBR, T8);
  if (lc) ++*lc;
}
void oz_aux_from_w(cudaStream_t s, const double* W, int64_t n, int pl1, double* aux, int64_t* lc) {
  const int64_t rows = (n + kR - 1) / kR * kR;
  const int64_t tot = rows * pl1;
  oz_aux_w_kernel<<<(unsigned)((tot + 255) / 256 < 2048 ? (tot + 255) / 256 : 2048), 256, 0, s>>>(W, n, n, pl1, rows,
                                                                                                   aux);
  if (lc) ++*lc;
}
void oz_vmax(cudaStream_t s, const double* V, int64_t n, int pl1, ColOwn own, double* vmax, int64_t* lc) {
  oz_vmax_kernel<<<pl1, 256, 0, s>>>(V, n, own, vmax);
  if (lc) ++*lc;
}
void oz_vdigits(cudaStream_t s, const double* V, int64_t n, int pl1, ColOwn own, const double* vmax, int* ev,
                double* vscale, int8_t* V8, int64_t* lc) {
  oz_vscale_kernel<<<1, 32, 0, s>>>(vmax, pl1, ev, vscale);
  oz_vpack_kernel<<<(unsigned)oz_nchunks(n), 256, 0, s>>>(V, n, pl1, own, ev, oz_nv(pl1), V8);
  if (lc) *lc += 2;
}

// Single-GPU setup of the int8 path (every column owned).  scratch: (n + 31) / 32 * 32 doubles.
void oz_setup(cudaStream_t s, const double* T, int64_t ld, int64_t n, const double* W, int pl1,
              int8_t* T8, double* aux, int* escale, const double* V, int8_t* V8, double* vscale,
              double* scratch, int64_t* lc) {
  const ColOwn all;
  oz_rowmax(s, T, ld, n, all, scratch, lc);
  oz_rowscale(s, scratch, n, escale, aux, pl1, lc);
  oz_pack(s, T, ld, n, all, escale, T8, lc);
  oz_aux_from_w(s, W, n, pl1, aux, lc);
  // V digits (the row-exponent scratch is free again once oz_pack_kernel has run: same stream); the
  // column maxima of V land in vscale and are turned into the scales in place
  oz_vmax(s, V, n, pl1, all, vscale, lc);
  oz_vdigits(s, V, n, pl1, all, vscale, escale, vscale, V8, lc);
}

void oz_repack_rows(cudaStream_t s, const int8_t* src, int64_t n, int64_t rows, int8_t* dst, int64_t ld8,
                    int64_t* lc) {
  if (rows <= 0) return;
  const int64_t blocks = rows < 148 * 16 ? rows : 148 * 16;
  oz_repack_kernel<<<(unsigned)blocks, 256, 0, s>>>(src, n, rows, dst, ld8);
  if (lc) ++*lc;
}

void oz_convert(cudaStream_t s, const double* X, int64_t ldx, int64_t n, int64_t cols, int8_t* X8,
                int64_t ld8, int* flag, unsigned long long* work, int num_sms, int64_t* lc, int* pflag, int pR) {
  const int64_t nunits = (cols + kConvCols - 1) / kConvCols;
  int64_t blocks = (int64_t)num_sms * 4;
  if (blocks > nunits) blocks = nunits;
  if (blocks < 1) blocks = 1;
  // Used for the first chunk of a block (later chunks are converted by the solve kernel's
  // convert-ahead warps).  kConvSmem of (unused) dynamic shared memory keeps these blocks off SMs
  // that hold an int8 solve CTA: placed beside one, plain loads convert at ~1 GB/s per SM.
  oz_x_to_i8_kernel<<<(unsigned)blocks, kConvThreads, kConvSmem, s>>>(X, ldx, n, cols, X8, ld8, flag, work,
                                                                      pflag, pR);
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
  kp.prof = nullptr;
  static long long* prof_buf = nullptr;
  static bool prof_on = getenv("GLS_OZ_PROF") != nullptr;
  if (prof_on) {
    if (!prof_buf) cudaMalloc(&prof_buf, 8 * 1024 * sizeof(long long));
    cudaMemsetAsync(prof_buf, 0, 8 * 1024 * sizeof(long long), s);
    kp.prof = prof_buf;
  }
  kp.b_out = a.b_out;
  kp.status_out = a.status_out;
  kp.s_ws = a.s_ws;
  kp.n = a.n;
  kp.cv_X = a.cv_X;
  kp.cv_ldx = a.cv_ldx;
  kp.cv_cols = a.cv_cols;
  kp.cv_X8 = a.cv_X8;
  kp.cv_ld8 = a.cv_ld8;
  kp.cv_flag = a.cv_flag;
  kp.pflag = a.pflag;
  kp.gate_all = a.gate_all;
  kp.cv_pflag = a.cv_pflag;
  kp.cols = cols;
  kp.m_blk = a.m_blk;
  const int64_t cpt = 4 * (int64_t)cpw;
  kp.num_tiles = (int)((cols + cpt - 1) / cpt);
  kp.NBR = (int)((a.n + kR - 1) / kR);
  kp.pL = a.pL;
  kp.pR = a.pR;
  kp.p = a.pL + a.pR;
  kp.cpw = cpw;
  // packed digit tiles as a 2D byte tensor [tiles * 224 rows][128]: TMA boxes of 112 rows (half a
  // tile, one per CTA of the pair) with the 128-byte swizzle the smem descriptors expect
  CUtensorMap tmap;
  const int64_t trows = oz_total_tiles(kp.NBR) * kBN;
  cuuint64_t tdim[2] = {(cuuint64_t)kKC, (cuuint64_t)trows};
  cuuint64_t tstride[1] = {(cuuint64_t)kKC};
  cuuint32_t tbox[2] = {(cuuint32_t)kKC, (cuuint32_t)(kBN / 2)};
  r = enc(&tmap, CU_TENSOR_MAP_DATA_TYPE_UINT8, 2, (void*)a.T8, tdim, tstride, tbox, estr,
          CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_128B, CU_TENSOR_MAP_L2_PROMOTION_L2_256B,
          CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
  if (r != CUDA_SUCCESS) {
    if (msg) *msg = "cuTensorMapEncodeTiled (packed T digits) failed";
    return cudaErrorInvalidValue;
  }
  // digits of V = M^{-1} [X_L | y]: [NC * NV rows][128], boxes of NV/2 rows (one per CTA of a pair)
  kp.NC = (int)oz_nchunks(a.n);
  // pin about 85 MB of X panels in L2 (of 126 MB): cpin chunks x 16 KiB x (CTAs in flight)
  static int pin_mb = -1;
  if (pin_mb < 0) {
    pin_mb = 85;
    if (const char* e = getenv("GLS_OZ_PIN_MB")) pin_mb = atoi(e);
  }
  kp.cpin = (int)((int64_t)pin_mb * 1000000 / ((int64_t)kATile * num_sms));
  kp.NV = oz_nv(a.pL + 1);
  kp.vscale = a.vscale;
  CUtensorMap vmap;
  cuuint64_t vdim[2] = {(cuuint64_t)kKC, (cuuint64_t)kp.NC * kp.NV};
  cuuint32_t vbox[2] = {(cuuint32_t)kKC, (cuuint32_t)(kp.NV / 2)};
  r = enc(&vmap, CU_TENSOR_MAP_DATA_TYPE_UINT8, 2, (void*)a.V8, vdim, tstride, vbox, estr,
          CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_128B, CU_TENSOR_MAP_L2_PROMOTION_L2_256B,
          CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
  if (r != CUDA_SUCCESS) {
    if (msg) *msg = "cuTensorMapEncodeTiled (packed V digits) failed";
    return cudaErrorInvalidValue;
  }
  cudaError_t e;
  if (a.pR == 1 && a.pL == 3)  // the configurations' covariate set: intercept, covariate, sex
    e = launch_oz_variant<4, 5, true>(s, map, tmap, vmap, kp, num_sms);
  else if (a.pR == 1 && a.pL + 2 <= 8)
    e = launch_oz_variant<0, 8, true>(s, map, tmap, vmap, kp, num_sms);
  else if (a.pR == 1)
    e = launch_oz_variant<0, 21, true>(s, map, tmap, vmap, kp, num_sms);
  else
    e = launch_oz_variant<0, 21, false>(s, map, tmap, vmap, kp, num_sms);
  if (lc) ++*lc;
  if (e == cudaSuccess && a.s_ws) {
    const int64_t blocks = (a.m_blk + 127) / 128 < 4 * num_sms ? (a.m_blk + 127) / 128 : 4 * num_sms;
    oz_posv_kernel<<<(unsigned)blocks, 128, 0, s>>>(a.s_ws, a.G, a.pL, a.pR, a.m_blk, a.gate, a.pflag, a.gate_all,
                                                    a.b_out,
                                                    a.status_out);
    e = cudaGetLastError();
    if (lc) ++*lc;
  }
  if (e != cudaSuccess && msg) *msg = std::string("ozaki_trsm_gls launch: ") + cudaGetErrorString(e);
  if (prof_on && e == cudaSuccess) {
    long long h[8 * 1024];
    cudaStreamSynchronize(s);
    cudaMemcpy(h, prof_buf, sizeof h, cudaMemcpyDeviceToHost);
    double sum[7] = {0, 0, 0, 0, 0, 0, 0};
    int nb = 0;
    for (int b = 0; b < 1024; b += 2)
      if (h[b * 8 + 3] > 0) {
        ++nb;
        for (int k = 0; k < 7; ++k) sum[k] += (double)h[b * 8 + k];
      }
    if (nb)
      fprintf(stderr, "[oz prof] ctas %d  total %.3e cyc  mma wait full %.1f%%  wait tmem-empty %.1f%%  "
              "producer wait empty %.1f%%  epilogue wait tmem-full %.1f%%  drain %.1f%%  busy %.1f%%\n", nb,
              sum[3] / nb, 100 * sum[1] / sum[3], 100 * sum[2] / sum[3], 100 * sum[0] / sum[3],
              100 * sum[4] / sum[3], 100 * sum[5] / sum[3], 100 * sum[6] / sum[3]);
  }
  return e;
}

}  // namespace gls
