// gls_internal.cuh -- internal declarations shared by the libgls.so translation units.
// Nothing here is visible through the C ABI (include/gls.h).
#pragma once

#include <cuda_runtime.h>
#include <stdint.h>

#include <string>

namespace gls {

// Per-device "done once" flags for kernel attribute setup (a process may drive several GPUs):
// returns true the first time it is called for (key, current device).
bool first_use_on_device(const void* key);

// The library's private stream-ordered device pool (one per device, created on first use) and an
// allocation from it on stream s (gls_api.cu).  Every device buffer of the library comes from here.
cudaMemPool_t gls_device_pool(int device);
cudaError_t gls_pool_alloc(void** p, size_t bytes, int device, cudaStream_t s);

// ---------------------------------------------------------------- hot-kernel tiling constants
// Row block of T / z handled per epilogue ("nb" in DESIGN.md), K extent per pipeline stage.
constexpr int kNB = 128;         // z rows per row block (4 warp slices x 32)
constexpr int kKT = 16;          // K per stage (one 128-byte TMA swizzle span of doubles)
constexpr int kKTPerRB = kNB / kKT;
constexpr int kTileDoubles = kNB * kKT;  // packed T tile: 2048 doubles = 16 KiB
constexpr int kMaxPanelCols = 64;        // 2 warps x 32 columns

// Packed-T tile index of (row block i, K tile kt): row block i holds K tiles 0..8(i+1)-1.
__host__ __device__ inline int64_t tpk_tile_offset(int64_t i) { return 4 * i * (i + 1); }
inline int64_t tpk_total_tiles(int64_t NB) { return 4 * NB * (NB + 1); }
// Zero rows placed ABOVE the data so that the last row block ends at row n:
// real row r sits at virtual row r + pad.  Kept even so every TMA box starts on a 16-byte boundary
// (an odd start row faults the TMA unit); for odd n one zero row is left below the data instead.
__host__ __device__ inline int64_t row_pad(int64_t n, int64_t NB) { return (NB * kNB - n) & ~(int64_t)1; }
// Packed W per row block: 4 slices x NW x 4 subtiles x 32 lanes x 2 doubles.
inline int64_t wpk_rb_doubles(int NW) { return 1024 * (int64_t)NW; }

// Hot-kernel geometry for a given pR: groups never straddle a warp.
struct PanelGeom {
  int gw;   // problems (groups) per warp
  int cpw;  // columns per warp = gw * pR (<= 32)
  int cpp;  // columns per panel = 2 * cpw
  int gpp;  // groups per panel = 2 * gw
  bool full_gram;  // groups straddle 8-column MMA tiles (pR does not divide 8)
};
inline PanelGeom panel_geom(int pR) {
  PanelGeom g;
  g.gw = 32 / pR;
  g.cpw = g.gw * pR;
  g.cpp = 2 * g.cpw;
  g.gpp = 2 * g.gw;
  g.full_gram = (8 % pR) != 0;
  return g;
}

// ---------------------------------------------------------------- generic FP64 DMMA GEMM
enum GemmFlags : int {
  GEMM_KMAX_ROW = 1,   // op(A) lower triangular: k < r0 + BM
  GEMM_KMAX_COL = 2,   // op(B) upper triangular: k < c0 + BN
  GEMM_KMIN_COL = 4,   // op(B) lower triangular: k >= c0
  GEMM_LOWER_C = 8,    // only tiles intersecting the lower triangle of C
};
// C[M x N] = alpha * op(A) * op(B) + beta * C, column-major.  op = 'N' or 'T'.
// ws (nullable, device, kSplitKWsDoubles doubles, private to the stream s): when given, GEMMs with
// few output tiles and a long K are split over K (partial tiles in ws, then a fixed-order reduction).
constexpr size_t kSplitKWsDoubles = (size_t)2 << 20;  // 16 MiB: (148 + 74) tiles x 128 x 64 doubles
void dgemm(cudaStream_t s, int64_t M, int64_t N, int64_t K, double alpha, const double* A,
           int64_t lda, char opA, const double* B, int64_t ldb, char opB, double beta, double* C,
           int64_t ldc, int flags, int64_t* launch_counter, double* ws = nullptr, int max_ctas = 0);

// Skinny products with a lower-triangular T (k <= 21 columns; memory-bound, deterministic):
// W = T B (part: scratch of 32 * n * k doubles) and V = T^T W.
void trmm_lower_skinny(cudaStream_t s, int64_t n, int k, const double* T, int64_t ldt, const double* B,
                       int64_t ldb, double* W, int64_t ldw, double* part, int64_t* launch_counter);
void trmm_lower_t_skinny(cudaStream_t s, int64_t n, int k, const double* T, int64_t ldt, const double* W,
                         int64_t ldw, double* V, int64_t ldv, int64_t* launch_counter);

// ---------------------------------------------------------------- setup: Cholesky + inverse
// In place: on return T (n x n, lower, ld) holds L^{-1} of M = L L^T; A (M on entry) is destroyed.
// T must be zero-initialised.  tol_fail: device {double tol; unsigned long long fail_pivot}.
struct CholStatus {
  double tol;
  unsigned long long fail;  // ULLONG_MAX when no pivot failed
};
// Columns of A still arriving (host M uploaded in column chunks on another stream): columns
// [k cols, (k+1) cols) are in place once ready[k] has fired.  chol_inv makes every stream wait for
// the chunks a kernel touches before launching it.
struct ColsReady {
  int64_t cols = 0;
  const cudaEvent_t* ready = nullptr;
  int64_t nchunks = 0;
};
void chol_inv(cudaStream_t s, int64_t n, double* A, double* T, int64_t ld, CholStatus* st,
              int64_t* launch_counter, const ColsReady* arriving = nullptr);
void chol_prepare(cudaStream_t s, int64_t n, const double* A, int64_t ld, CholStatus* st,
                  int64_t* launch_counter);

// ---------------------------------------------------------------- packing + hot kernel
void pack_T(cudaStream_t s, const double* T, int64_t ld, int64_t n, int64_t NB, double* Tpk,
            int64_t* launch_counter);
void pack_W(cudaStream_t s, const double* W, int64_t ld, int64_t n, int ncolsW, int64_t NB, int NW,
            double* Wpk, int64_t* launch_counter);

struct SolveArgs {
  const double* X;      // X_R block, column-major, leading dimension ldx (device)
  int64_t ldx;          // >= n, even
  int64_t n;
  int64_t NB;
  int pL, pR;
  int64_t m_blk;
  const double* Tpk;
  const double* Wpk;
  const double* G;      // (pL+1) x (pL+1): S_TL = G[0:pL,0:pL], b_T = G[0:pL, pL]
  double* b_out;        // device
  int32_t* status_out;  // device or nullptr
  // nullable per-problem path flags (int8 conversion): when set, only problems g with pflag[g] != 0 are
  // solved and stored (the int8 kernel stores the others), and panels without one are skipped
  const int* pflag = nullptr;
  // nullable: only the first min(m_blk, *m_dev) problems exist (a compacted block, fb_compact)
  const int* m_dev = nullptr;
  // with a gate: run only if gate_lo < *gate <= gate_hi (default: *gate != 0 for counts)
  int gate_lo = 0, gate_hi = 0x7fffffff;
};
// Compacted FP64 fallback (reading A16): fb_compact writes the block's flagged count (the sum of the
// chunks' counts ccount[0, nchunks)) to *count and, when 0 < *count <= cap, the flagged problems'
// indices (ascending) to idx and their columns gathered into Xc (leading dimension ldx); after the FP64
// kernel has solved Xc (m_dev = count), fb_scatter writes its records / statuses back to b / st.
void fb_compact(cudaStream_t s, const int* pflag, int64_t groups, const int* ccount, int nchunks, int cap, int* idx,
                int* count, const double* X, int64_t ldx, int pR, double* Xc, int num_sms, int64_t* lc);
void fb_scatter(cudaStream_t s, const double* bc, const int32_t* sc, const int* idx, const int* count, int cap,
                int p, double* b, int32_t* st, int num_sms, int64_t* lc);
// Returns cudaSuccess or the launch error; msg receives a description on failure.
// gate (nullable, device): when non-null the kernel returns at once unless *gate != 0 (it is the
// fallback for blocks the int8 path rejected).
cudaError_t launch_fused_trsm_gls(cudaStream_t s, const SolveArgs& a, int num_sms, std::string* msg,
                                  int64_t* launch_counter, const int* gate = nullptr,
                                  unsigned long long* ran = nullptr);

// ---------------------------------------------------------------- int8 (Ozaki-split) hot path
constexpr int kOzR = 32;          // z rows per row block
constexpr int kOzKC = 128;        // K per stage
constexpr int kOzSlices = 7;      // base-256 digits per element of T (55-bit fixed point per row)
constexpr int kOzTileBytes = kOzSlices * kOzR * kOzKC;  // 28 KiB packed digit tile
// Largest n for which every digit product sum fits int32: 128 * 128 * n < 2^31.
constexpr int64_t kOzMaxN = 131071;
// Packed tile index of (row block i, K chunk 0); row block i holds i/4 + 1 chunks.
__host__ __device__ inline int64_t oz_tile_offset(int64_t i) {
  const int64_t q = i >> 2, r = i & 3;
  return (q + 1) * (2 * q + r);
}
int64_t oz_total_tiles(int64_t NBR);
inline int64_t oz_nchunks(int64_t n) { return (n + kOzKC - 1) / kOzKC; }
// N of the V block (digits of V = M^{-1} [X_L | y], 8 rows per column): multiple of 32
inline int oz_nv(int pl1) { return ((8 * pl1 + 31) / 32) * 32; }
// T (n x n lower, column-major) and W = [X~_L | y~] (n x pl1) -> digit tiles T8 and the per-row
// aux table [sigma_r, W~_r,0 .. W~_r,pL] (stride pl1 + 1, ceil(n/32)*32 rows).  escale: int[rows].
// V = T^T W = M^{-1} [X_L | y] (n x pl1, column-major) -> column scales vscale[pl1] and digit tiles
// V8 (oz_nchunks(n) x oz_nv(pl1) x 128 bytes): S_BL and b_B of a column x are x^T V (§5.4).
// Column ownership of T for the setup kernels: global column j is owned when (j / nb) % nranks == rank,
// and lives at local column ((j / nb) / nranks) nb + j % nb of the rank's array.  The default owns
// every column at its own index (single-GPU create).
struct ColOwn {
  int64_t nb = (int64_t)1 << 40;
  int nranks = 1, rank = 0;
  // (nranks == 1: no 64-bit divisions -- the setup kernels of the single-GPU create run at full speed)
  __host__ __device__ bool owned(int64_t j) const { return nranks == 1 || (j / nb) % nranks == rank; }
  __host__ __device__ int64_t local(int64_t j) const {
    return nranks == 1 ? j : ((j / nb) / nranks) * nb + j % nb;
  }
};
// Setup of the int8 path from T = L^{-1} (dense, column-major, ld) and W = [X~_L | y~], V = M^{-1}[X_L|y]:
// row scales + aux, digit tiles T8, V digits.  scratch: (n + 31) / 32 * 32 doubles.
void oz_setup(cudaStream_t s, const double* T, int64_t ld, int64_t n, const double* W, int pl1,
              int8_t* T8, double* aux, int* escale, const double* V, int8_t* V8, double* vscale,
              double* scratch, int64_t* lc);
// Its steps, for the distributed create (dist_create.cu), each touching owned columns / chunks only:
void oz_rowmax(cudaStream_t s, const double* T, int64_t ld, int64_t n, ColOwn own, double* rowmax, int64_t* lc);
void oz_rowscale(cudaStream_t s, const double* rowmax, int64_t n, int* escale, double* aux, int pl1, int64_t* lc);
void oz_pack(cudaStream_t s, const double* T, int64_t ld, int64_t n, ColOwn own, const int* escale, int8_t* T8,
             int64_t* lc);
void oz_aux_from_w(cudaStream_t s, const double* W, int64_t n, int pl1, double* aux, int64_t* lc);
void oz_vmax(cudaStream_t s, const double* V, int64_t n, int pl1, ColOwn own, double* vmax, int64_t* lc);
void oz_vdigits(cudaStream_t s, const double* V, int64_t n, int pl1, ColOwn own, const double* vmax, int* ev,
                double* vscale, int8_t* V8, int64_t* lc);
// X (double) -> X8 (int8, ld8 % 16 == 0); *flag |= 1 if some value is not an integer in [-128,127].
// With pflag (zeroed, one int per problem of pR columns): pflag[g] = 1 for every problem holding such
// a value and *flag counts those problems instead.
// work: a zeroed unsigned long long (the pass's work-stealing counter).
void oz_convert(cudaStream_t s, const double* X, int64_t ldx, int64_t n, int64_t cols, int8_t* X8,
                int64_t ld8, int* flag, unsigned long long* work, int num_sms, int64_t* launch_counter,
                int* pflag = nullptr, int pR = 1);
struct OzArgs {
  const int8_t* X8;     // column-major, ld8 (multiple of 16), device
  int64_t ld8;
  int64_t n;
  int pL, pR;
  int64_t m_blk;
  const int8_t* T8;
  const double* aux;
  const double* G;
  const int* gate;      // nullable; the kernel does nothing when *gate != 0
  unsigned long long* ran;  // nullable; block 0 adds 1 when the kernel does its work
  const int8_t* V8;     // digit tiles of V (oz_setup)
  const double* vscale;
  double* b_out;
  int32_t* status_out;
  double* s_ws;         // nullable: m_blk records of pR (pL + pR + 1) doubles; when set, the kernel
                        // stores S_BL, S_BR, b_B there and a batched posv kernel solves (large p)
  // nullable convert-ahead job run by the kernel's conv warps (also when gated): FP64 X (ld cv_ldx,
  // even, 16-byte aligned, cv_cols columns of n) -> int8 cv_X8 (ld cv_ld8); non-integers set *cv_flag
  const double* cv_X = nullptr;
  int64_t cv_ldx = 0, cv_cols = 0;
  int8_t* cv_X8 = nullptr;
  int64_t cv_ld8 = 0;
  int* cv_flag = nullptr;
  // nullable per-problem path flags (see oz_convert): with pflag, *gate counts the launch's flagged
  // problems, the kernel runs unless all gate_all are flagged and stores none of the flagged ones;
  // cv_pflag receives the convert-ahead chunk's flags (first-time flags counted in *cv_flag)
  const int* pflag = nullptr;
  int64_t gate_all = 0;
  int* cv_pflag = nullptr;
};
constexpr int kOzPosvInKernelMaxP = 8;  // p above this: posv in a separate kernel (oz s_ws)
constexpr int64_t kConvertAheadMinN = 4096;  // n below this: standalone FP64 -> int8 pass per chunk
constexpr int64_t kSerialChunkBytes = 1ll << 30;  // int8 workspace per chunk when the passes are standalone
constexpr int64_t kUploadChunkCols = 512;  // host M reaches the device in chunks of this many columns
// rows of n int8 codes packed back to back -> the same rows at pitch ld8 (>= n); padding untouched
void oz_repack_rows(cudaStream_t s, const int8_t* src, int64_t n, int64_t rows, int8_t* dst, int64_t ld8,
                    int64_t* launch_counter);
cudaError_t launch_ozaki_gls(cudaStream_t s, const OzArgs& a, int num_sms, std::string* msg,
                             int64_t* launch_counter);

}  // namespace gls
