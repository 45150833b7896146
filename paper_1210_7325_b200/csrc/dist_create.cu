// dist_create.cu -- NEXT-3 of SURVEY §8(f), the in-scope half: the once-per-job factorisation of an M
// that one GPU cannot hold, split across the GPUs of the node (§6: "for problems
// in which M does not fit ... algorithms-by-blocks ... ScaLAPACK ... Elemental").
//
// The single-GPU gls_create needs the dense M and T = L^{-1} at once (2 n^2 8 bytes: 275 GB at the
// int8 path's limit n = 131071).  Here rank r of G holds only the column blocks j of width nb with
// j % G == r (1D block-cyclic, as ScaLAPACK's column distribution), for both M (becoming L) and T, and
// the ranks run a right-looking blocked Cholesky with a panel broadcast per block column -- Alg. 5
// line 1 -- fused with the forward substitution that turns the identity into T (line 2's L^{-1} applied
// to the identity; design A, reading A13):
//
//   for k = 0 .. K-1 (owner o = k mod G):
//     o:   L_kk L_kk^T = A_kk, T_kk = L_kk^{-1}           (chol_inv.cu, one block)
//          panel P_k = [T_kk ; A_{>k,k} T_kk^T]           (= [T_kk ; L_{>k,k}])       -> broadcast
//     all: for owned j <  k:  R_j[k]  := T_kk R_j[k]       (T_kj = L_kk^{-1} (E - sum_{l<k} L_kl T_lj))
//          for owned j <= k:  R_j[>k] -= L_{>k,k} R_j[k]   (right-looking substitution)
//          for owned j >  k:  A_{>=j,j} -= L_{>=j,k} L_{j,k}^T   (trailing update, lower part)
//   (R_j starts as the identity block E_j; after step K-1 it is column block j of T.)
//
// Then the int8 path's shared state from the distributed T:
//   W = T [X_L | y] = sum_r T_{:,owned r} [X_L | y]_{owned r}    (partials all-gathered, summed in rank order)
//   row scales from max_j |T_rj| (partial maxima, all-reduce MAX: exact), G = W^T W, aux;
//   digit tiles of T and V = T^T W for the owned K chunks (column scales of V by all-reduce MAX),
//   assembled by an all-reduce SUM of the zero-initialised int8 buffers (every byte has one writer).
// The collectives run in the caller (multi.dist_create: torch.distributed over NCCL, or gloo);
// this file only computes.  Every rank ends with bit-identical T8 / V8 / aux / G (the same inputs
// reach the same deterministic kernels), and an int8-only context (gls_create_adopt_int8) receives them.
#include <climits>
#include <cmath>
#include <cstring>
#include <string>

#include "../../include/gls.h"
#include "gls_internal.cuh"

using namespace gls;

struct gls_dist {
  int device = 0;
  int64_t n = 0, nb = 0, K = 0, nloc = 0;
  int pL = 0, pR = 0, pl1 = 0, G = 1, r = 0;
  cudaStream_t s = nullptr;
  double* A = nullptr;       // n x nloc: owned column blocks of M (lower part), becoming L; ld = n
  double* R = nullptr;       // n x nloc: owned column blocks of T; ld = n
  double* panel = nullptr;   // (n - k nb) x nb, ld = n - k nb
  double* tmp = nullptr;     // nb x nloc scratch
  double* B = nullptr;       // n x pl1: [X_L | y]
  double* Bloc = nullptr;    // nloc x pl1: the rows of B at owned columns
  double* Wpart = nullptr;   // n x pl1
  double* W = nullptr;       // n x pl1 (the summed W, written by the caller)
  double* V = nullptr;       // n x pl1 (rows of owned columns)
  double* rowmax = nullptr;  // NBR x 32
  double* vmax = nullptr;    // pl1
  int* esc = nullptr;        // NBR x 32
  double* ws = nullptr;      // split-K workspace of dgemm
  CholStatus* st = nullptr;
  double tol = 0.0;
  gls_ctx* ctx = nullptr;    // int8-only adopt context receiving T8, aux, V8, vscale, G
  void* sh[8] = {};          // its shared buffers: G, T8, aux, V8, vscale
  int64_t shb[8] = {};
  int64_t launches = 0;
  int64_t failed_pivot = -1;
  int64_t width(int64_t j) const { return std::min(nb, n - j * nb); }
  int64_t lcol(int64_t j) const { return (j / G) * nb; }                       // local column of block j
  int64_t owned_upto(int64_t k) const { return k >= r ? (k - r) / G + 1 : 0; }  // owned blocks j <= k
  int64_t loc_cols(int64_t blocks) const { return std::min(blocks * nb, nloc); }
};

namespace {

void dist_free(gls_dist* d) {
  if (!d) return;
  // the buffers are also read and written by the caller's collectives on other streams
  cudaDeviceSynchronize();
  for (void* p : {(void*)d->A, (void*)d->R, (void*)d->panel, (void*)d->tmp, (void*)d->B, (void*)d->Bloc,
                  (void*)d->Wpart, (void*)d->W, (void*)d->V, (void*)d->rowmax, (void*)d->vmax, (void*)d->esc,
                  (void*)d->ws, (void*)d->st})
    if (p) cudaFreeAsync(p, d->s);  // back to the library's stream-ordered pool (no unmapping)
  if (d->s) cudaStreamSynchronize(d->s);
  if (d->ctx) gls_destroy(d->ctx);
  if (d->s) cudaStreamDestroy(d->s);
  cudaGetLastError();
  delete d;
}

bool on_device(const void* p) {
  cudaPointerAttributes at;
  if (cudaPointerGetAttributes(&at, p) != cudaSuccess) {
    cudaGetLastError();
    return false;
  }
  return at.type == cudaMemoryTypeDevice || at.type == cudaMemoryTypeManaged;
}

__global__ void dist_maxdiag_kernel(int64_t n, const double* M, double* out) {
  __shared__ double red[256];
  double m = 0.0;
  for (int64_t k = threadIdx.x; k < n; k += blockDim.x) m = fmax(m, M[k + k * n]);
  red[threadIdx.x] = m;
  __syncthreads();
  for (int w = 128; w > 0; w >>= 1) {
    if (threadIdx.x < w) red[threadIdx.x] = fmax(red[threadIdx.x], red[threadIdx.x + w]);
    __syncthreads();
  }
  if (threadIdx.x == 0) *out = red[0];
}

}  // namespace

extern "C" int gls_dist_create(int64_t n, int32_t pL, int32_t pR, int64_t nb, int32_t nranks, int32_t rank,
                               const double* M, const double* X_L, const double* y, gls_dist** out) {
  if (!out) return GLS_ERR_ARG;
  *out = nullptr;
  if (!M || !y || (pL > 0 && !X_L) || nranks < 1 || rank < 0 || rank >= nranks || nb < kOzKC || nb % kOzKC)
    return GLS_ERR_ARG;
  if (pL < 0 || pR < 1 || pL + pR > 20 || n <= pL + pR || n > kOzMaxN) return GLS_ERR_DIM;
  gls_dist* d = new gls_dist();
  d->n = n;
  d->nb = nb;
  d->K = (n + nb - 1) / nb;
  d->pL = pL;
  d->pR = pR;
  d->pl1 = pL + 1;
  d->G = nranks;
  d->r = rank;
  for (int64_t j = rank; j < d->K; j += nranks) d->nloc += d->width(j);
  auto fail = [&](int rc) {
    dist_free(d);
    return rc;
  };
  if (cudaGetDevice(&d->device) != cudaSuccess || cudaStreamCreateWithFlags(&d->s, cudaStreamNonBlocking) != cudaSuccess)
    return fail(GLS_ERR_CUDA);
  int rc = gls_create_adopt_int8(n, pL, pR, &d->ctx);
  if (rc) return fail(rc);
  int32_t cnt = 0;
  rc = gls_shared_view_ex(d->ctx, GLS_SHARE_INT8_ONLY, d->sh, d->shb, &cnt);
  if (rc || cnt != 5) return fail(rc ? rc : GLS_ERR_STATE);
  const int64_t NBR = (n + kOzR - 1) / kOzR;
  const size_t nl = (size_t)(d->nloc > 0 ? d->nloc : 1);
  const int pl1 = d->pl1;
  // from the library's stream-ordered pool (cached across creates: cudaMalloc / cudaFree of these
  // ~2 n^2 / G * 8 bytes mapped and unmapped pages on every create), usable from any stream after
  // the synchronisation below
  auto palloc = [&](auto** p, size_t bytes) { return gls_pool_alloc((void**)p, bytes, d->device, d->s); };
  if (palloc(&d->A, (size_t)n * nl * 8) || palloc(&d->R, (size_t)n * nl * 8) ||
      palloc(&d->panel, (size_t)n * nb * 8) || palloc(&d->tmp, (size_t)nb * nl * 8) ||
      palloc(&d->B, (size_t)n * pl1 * 8) || palloc(&d->Bloc, nl * pl1 * 8) ||
      palloc(&d->Wpart, (size_t)n * pl1 * 8) || palloc(&d->W, (size_t)n * pl1 * 8) ||
      palloc(&d->V, (size_t)n * pl1 * 8) || palloc(&d->rowmax, (size_t)NBR * kOzR * 8) ||
      palloc(&d->vmax, (size_t)pl1 * 8) || palloc(&d->esc, (size_t)NBR * kOzR * sizeof(int)) ||
      palloc(&d->ws, kSplitKWsDoubles * 8) || palloc(&d->st, sizeof(CholStatus)) ||
      cudaStreamSynchronize(d->s))
    return fail(GLS_ERR_OOM);
  cudaStream_t s = d->s;
  // owned column blocks of M (contiguous n x w column ranges of the column-major M)
  for (int64_t j = rank; j < d->K; j += nranks)
    if (cudaMemcpyAsync(d->A + d->lcol(j) * n, M + j * nb * n, (size_t)n * d->width(j) * 8, cudaMemcpyDefault, s))
      return fail(GLS_ERR_CUDA);
  if (cudaMemsetAsync(d->R, 0, (size_t)n * nl * 8, s) || cudaMemsetAsync(d->V, 0, (size_t)n * pl1 * 8, s) ||
      cudaMemsetAsync(d->sh[1], 0, (size_t)d->shb[1], s) || cudaMemsetAsync(d->sh[3], 0, (size_t)d->shb[3], s))
    return fail(GLS_ERR_CUDA);
  if ((pL > 0 && cudaMemcpyAsync(d->B, X_L, (size_t)n * pL * 8, cudaMemcpyDefault, s)) ||
      cudaMemcpyAsync(d->B + (size_t)n * pL, y, (size_t)n * 8, cudaMemcpyDefault, s))
    return fail(GLS_ERR_CUDA);
  // NotSPD tolerance (reading A5) from the whole diagonal of M, on every rank
  double mx = 0.0;
  if (on_device(M)) {
    dist_maxdiag_kernel<<<1, 256, 0, s>>>(n, M, d->vmax);
    if (cudaMemcpyAsync(&mx, d->vmax, 8, cudaMemcpyDeviceToHost, s) || cudaStreamSynchronize(s)) return fail(GLS_ERR_CUDA);
  } else {
    for (int64_t k = 0; k < n; ++k) mx = std::fmax(mx, M[k + k * n]);
  }
  d->tol = std::ldexp(1.0, -52) * mx;
  if (cudaStreamSynchronize(s) || cudaGetLastError()) return fail(GLS_ERR_CUDA);
  *out = d;
  return GLS_OK;
}

extern "C" int gls_dist_info(const gls_dist* d, int64_t* nb, int64_t* nblocks, int64_t* nloc) {
  if (!d || !nb || !nblocks || !nloc) return GLS_ERR_ARG;
  *nb = d->nb;
  *nblocks = d->K;
  *nloc = d->nloc;
  return GLS_OK;
}

extern "C" int gls_dist_buffer(gls_dist* d, int32_t which, int64_t k, void** ptr, int64_t* bytes) {
  if (!d || !ptr || !bytes) return GLS_ERR_ARG;
  const int64_t n = d->n;
  switch (which) {
    case GLS_DIST_PANEL:
      if (k < 0 || k >= d->K) return GLS_ERR_ARG;
      *ptr = d->panel;
      *bytes = (n - k * d->nb) * d->width(k) * 8;
      return GLS_OK;
    case GLS_DIST_WPART: *ptr = d->Wpart; *bytes = n * d->pl1 * 8; return GLS_OK;
    case GLS_DIST_W: *ptr = d->W; *bytes = n * d->pl1 * 8; return GLS_OK;
    case GLS_DIST_ROWMAX: *ptr = d->rowmax; *bytes = (n + kOzR - 1) / kOzR * kOzR * 8; return GLS_OK;
    case GLS_DIST_VMAX: *ptr = d->vmax; *bytes = d->pl1 * 8; return GLS_OK;
    case GLS_DIST_T8: *ptr = d->sh[1]; *bytes = d->shb[1]; return GLS_OK;
    case GLS_DIST_V8: *ptr = d->sh[3]; *bytes = d->shb[3]; return GLS_OK;
    default: return GLS_ERR_ARG;
  }
}

extern "C" int gls_dist_step(gls_dist* d, int32_t phase, int64_t k) {
  if (!d || !d->ctx) return GLS_ERR_ARG;
  const int64_t n = d->n, nb = d->nb;
  const int pl1 = d->pl1;
  cudaStream_t s = d->s;
  int64_t* lc = &d->launches;
  const ColOwn own{nb, d->G, d->r};
  switch (phase) {
    case GLS_DIST_FACTOR: {  // owner of block k: diagonal block and panel
      if (k < 0 || k >= d->K || k % d->G != d->r) return GLS_ERR_ARG;
      const int64_t j0 = k * nb, w = d->width(k), lc0 = d->lcol(k), ldp = n - j0, mb = n - j0 - w;
      double* Akk = d->A + j0 + lc0 * n;
      double* Tkk = d->R + j0 + lc0 * n;
      CholStatus h{d->tol, ULLONG_MAX};
      if (cudaMemcpyAsync(d->st, &h, sizeof h, cudaMemcpyHostToDevice, s)) return GLS_ERR_CUDA;
      chol_inv(s, w, Akk, Tkk, n, d->st, lc);
      if (cudaMemcpyAsync(&h, d->st, sizeof h, cudaMemcpyDeviceToHost, s) || cudaStreamSynchronize(s))
        return GLS_ERR_CUDA;
      if (h.fail != ULLONG_MAX) {
        d->failed_pivot = j0 + (int64_t)h.fail;
        return GLS_ERR_NOT_SPD;
      }
      // P_k = [T_kk ; A_{>k,k} T_kk^T]
      if (cudaMemcpy2DAsync(d->panel, ldp * 8, Tkk, n * 8, w * 8, w, cudaMemcpyDeviceToDevice, s))
        return GLS_ERR_CUDA;
      if (mb > 0)
        dgemm(s, mb, w, w, 1.0, Akk + w, n, 'N', Tkk, n, 'T', 0.0, d->panel + w, ldp, GEMM_KMAX_COL, lc, d->ws);
      break;
    }
    case GLS_DIST_UPDATE: {  // every rank, once P_k is in d->panel
      if (k < 0 || k >= d->K) return GLS_ERR_ARG;
      const int64_t j0 = k * nb, w = d->width(k), ldp = n - j0, mb = n - j0 - w;
      const double* Tkk = d->panel;
      const double* Lb = d->panel + w;
      const int64_t cb = d->loc_cols(d->owned_upto(k - 1));  // owned j < k
      const int64_t cle = d->loc_cols(d->owned_upto(k));     // owned j <= k
      if (cb > 0) {  // R_j[k] := T_kk R_j[k]
        dgemm(s, w, cb, w, 1.0, Tkk, ldp, 'N', d->R + j0, n, 'N', 0.0, d->tmp, w, GEMM_KMAX_ROW, lc, d->ws);
        if (cudaMemcpy2DAsync(d->R + j0, n * 8, d->tmp, w * 8, w * 8, cb, cudaMemcpyDeviceToDevice, s))
          return GLS_ERR_CUDA;
      }
      if (mb > 0 && cle > 0)  // R_j[>k] -= L_{>k,k} R_j[k]
        dgemm(s, mb, cle, w, -1.0, Lb, ldp, 'N', d->R + j0, n, 'N', 1.0, d->R + j0 + w, n, 0, lc, d->ws);
      for (int64_t j = k + 1; j < d->K; ++j) {  // trailing update of the owned blocks right of k
        if (j % d->G != d->r) continue;
        const int64_t j1 = j * nb, wj = d->width(j);
        const double* Lj = d->panel + (j1 - j0);
        dgemm(s, n - j1, wj, w, -1.0, Lj, ldp, 'N', Lj, ldp, 'T', 1.0, d->A + j1 + d->lcol(j) * n, n, GEMM_LOWER_C,
              lc, d->ws);
      }
      break;
    }
    case GLS_DIST_PARTIALS: {  // W partial and row maxima of the owned columns of T
      for (int64_t j = d->r; j < d->K; j += d->G)
        if (cudaMemcpy2DAsync(d->Bloc + d->lcol(j), d->nloc * 8, d->B + j * nb, n * 8, d->width(j) * 8, pl1,
                              cudaMemcpyDeviceToDevice, s))
          return GLS_ERR_CUDA;
      if (d->nloc > 0)
        dgemm(s, n, pl1, d->nloc, 1.0, d->R, n, 'N', d->Bloc, d->nloc, 'N', 0.0, d->Wpart, n, 0, lc, d->ws);
      else if (cudaMemsetAsync(d->Wpart, 0, (size_t)n * pl1 * 8, s))
        return GLS_ERR_CUDA;
      oz_rowmax(s, d->R, n, n, own, d->rowmax, lc);
      break;
    }
    case GLS_DIST_PACK: {  // after W (summed) and the row maxima (all-reduce MAX) are in place
      double* Gm = (double*)d->sh[0];
      double* aux = (double*)d->sh[2];
      oz_rowscale(s, d->rowmax, n, d->esc, aux, pl1, lc);
      oz_aux_from_w(s, d->W, n, pl1, aux, lc);
      dgemm(s, pl1, pl1, n, 1.0, d->W, n, 'T', d->W, n, 'N', 0.0, Gm, pl1, 0, lc, d->ws);
      oz_pack(s, d->R, n, n, own, d->esc, (int8_t*)d->sh[1], lc);
      for (int64_t j = d->r; j < d->K; j += d->G) {  // V rows of the owned columns: T_{:,j}^T W
        const int64_t j1 = j * nb;
        dgemm(s, d->width(j), pl1, n - j1, 1.0, d->R + j1 + d->lcol(j) * n, n, 'T', d->W + j1, n, 'N', 0.0,
              d->V + j1, n, 0, lc, d->ws);
      }
      oz_vmax(s, d->V, n, pl1, own, d->vmax, lc);
      break;
    }
    case GLS_DIST_PACK2:  // after the column maxima of V (all-reduce MAX)
      oz_vdigits(s, d->V, n, pl1, own, d->vmax, d->esc, (double*)d->sh[4], (int8_t*)d->sh[3], lc);
      break;
    default:
      return GLS_ERR_ARG;
  }
  if (cudaStreamSynchronize(s) || cudaGetLastError()) return GLS_ERR_CUDA;
  return GLS_OK;
}

extern "C" int gls_dist_finish(gls_dist* d, gls_ctx** out) {
  if (!d || !out || !d->ctx) return GLS_ERR_ARG;
  int rc = gls_commit_shared(d->ctx);
  if (rc) return rc;
  *out = d->ctx;
  d->ctx = nullptr;
  return GLS_OK;
}

extern "C" int64_t gls_dist_failed_pivot(const gls_dist* d) { return d ? d->failed_pivot : -1; }

extern "C" int64_t gls_dist_launches(const gls_dist* d) { return d ? d->launches : -1; }

extern "C" void gls_dist_destroy(gls_dist* d) { dist_free(d); }
