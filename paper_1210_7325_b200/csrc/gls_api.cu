// gls_api.cu -- the C ABI (include/gls.h) and the host runtime around the kernels:
// context lifetime, pointer-kind dispatch, the once-per-context setup (Alg. 5 lines 1,2,4,5,6;
// PAPER.md:311-317) and the double-buffered host->device stream of X_R blocks
// (Alg. 8 ooc-hp-gwas; workspaces fig:workspaces PAPER.md:633-653).
#include <cuda_runtime.h>

#include <chrono>
#include <climits>
#include <cstdio>
#include <cstdlib>
#include <cstring>
#include <algorithm>
#include <mutex>
#include <set>
#include <string>
#include <vector>

#include <nvtx3/nvToolsExt.h>
#include <nvtx3/nvToolsExtCudaRt.h>

#include "../../include/gls.h"
#include "gls_internal.cuh"

using namespace gls;

namespace gls {
bool first_use_on_device(const void* key) {
  static std::mutex mu;
  static std::set<std::pair<const void*, int>> done;
  int dev = 0;
  cudaGetDevice(&dev);
  std::lock_guard<std::mutex> lk(mu);
  return done.insert({key, dev}).second;
}
}  // namespace gls

namespace {
enum CtxState { ST_OK = 0, ST_FAILED = 1, ST_ADOPT = 2 };
}

// The streams and fixed events a context owns; taken from / given back to a per-device cache
// (res_take / res_give) instead of being created and destroyed with every context.
struct CtxRes {
  cudaStream_t own = nullptr, h2d = nullptr, d2h = nullptr, fb = nullptr, alloc = nullptr;
  cudaEvent_t ev[12] = {};  // ev_oz[2], ev_fb[2], ev_h2d[2], ev_comp[2], ev_d2h[2], ev_create, misc
};

struct gls_ctx {
  int device = 0;
  CtxRes res;
  int64_t n = 0;
  int pL = 0, pR = 0, p = 0, NW = 1;
  int64_t NB = 0;
  int state = ST_FAILED;
  int64_t failed_pivot = -1;
  std::string err;
  int num_sms = 148;
  cudaStream_t own_stream = nullptr, stream = nullptr, h2d = nullptr, d2h = nullptr;
  // shared state (replicated across GPUs)
  double* Tpk = nullptr;
  size_t Tpk_bytes = 0;
  double* Wpk = nullptr;
  size_t Wpk_bytes = 0;
  double* G = nullptr;
  size_t G_bytes = 0;
  // int8 (Ozaki-split) path, ozaki_gls.cu: digit tiles of T and the per-row [sigma | W~] table
  int8_t* T8 = nullptr;
  size_t T8_bytes = 0;
  double* aux = nullptr;
  size_t aux_bytes = 0;
  int8_t* V8 = nullptr;      // digits of V = M^{-1} [X_L | y]
  size_t V8_bytes = 0;
  double* vscale = nullptr;  // their column scales
  size_t vscale_bytes = 0;
  int path = GLS_PATH_AUTO;
  bool oz_ok = false;  // n small enough for exact int32 digit products
  bool fp64_ok = true;  // false: an int8-only context (no packed T for the FP64 kernel; gls_create_adopt_int8)
  // int8 conversion workspaces (two, swapping roles) and their rejection flags
  int64_t x8_cols = 0, ld8 = 0;
  double* sws = nullptr;     // per-problem records for the separate posv of large p (OzArgs::s_ws)
  int64_t sws_groups = 0;
  int8_t* x8[2] = {nullptr, nullptr};
  int* flags = nullptr;                  // 2 ints, then (8-byte aligned) 2 work counters
  int* cflags = nullptr;                 // per conversion chunk of a block: its problems on the FP64 path
  int64_t cflags_cap = 0;
  int* pflags = nullptr;                 // per problem of a block: 1 = holds a value int8 cannot take
  int64_t pflags_cap = 0;
  // compacted FP64 fallback of a chunk's few flagged problems (fb_compact): indices, gathered columns
  // (leading dimension fb_ldx), their records and statuses; fb_cap problems
  int* fb_idx = nullptr;
  double* fb_X = nullptr;
  double* fb_b = nullptr;
  int32_t* fb_s = nullptr;
  int64_t fb_cap = 0, fb_ldx = 0;
  unsigned long long* ran = nullptr;     // [0] int8 kernel launches that ran, [1] FP64 ones
  cudaEvent_t ev_oz[2] = {}, ev_fb[2] = {};
  cudaStream_t fb = nullptr;  // gated FP64 fallback launches (off the int8 kernel's stream)
  // host int8 staging (gls_solve_block_i8 with a host or unaligned source)
  int8_t* stage8[2] = {nullptr, nullptr};
  int8_t* raw8[2] = {nullptr, nullptr};  // when ld8 != n: rows of n bytes as they arrive, repacked to ld8
  int64_t stage8_cols = 0;
  // optional per-launch timing of the hot kernels (gls_set_timing): event pairs on the launch stream
  bool timing = false;
  struct TimedLaunch {
    cudaEvent_t a, b;
    int kind;  // 0 int8 kernel, 1 FP64 kernel, 2 int8 conversion
  };
  std::vector<TimedLaunch> tl;
  std::vector<cudaEvent_t> ev_pool;
  // optional overlap accounting of the host->HBM stream (gls_set_stream_report): per chunk, timing
  // events around its H2D copy, its compute (recorded after Alg. 8's two waits have cleared) and its
  // D2H copy, on the streams that run them
  bool srep = false;
  struct ChunkRec {
    cudaEvent_t h0, h1, c0, c1, d0, d1;
    cudaEvent_t cr;  // first chunk of a call: the compute stream done with its earlier work (e.g. an
                     // asynchronous gls_create), before it waits for the chunk's data
    int64_t hbytes, dbytes;
  };
  std::vector<ChunkRec> srec;
  // host-streaming workspaces (two, swapping roles -- fig:workspaces)
  int64_t block_cols = 0;
  int64_t stage_cols = 0, ld_stage = 0;
  double* stage[2] = {nullptr, nullptr};
  double* bstage[2] = {nullptr, nullptr};
  int32_t* sstage[2] = {nullptr, nullptr};
  int64_t bstage_groups = 0;
  cudaEvent_t ev_h2d[2] = {}, ev_comp[2] = {}, ev_d2h[2] = {};
  uint64_t seq = 0;
  // device scratch for host outputs of device-resident X_R
  double* bscratch = nullptr;
  int32_t* sscratch = nullptr;
  int64_t scratch_groups = 0;
  int64_t launches = 0;
  // gls_create_async: the factorisation is enqueued, not waited for; its NotSPD outcome (the device
  // status, copied into the pinned hst by the stream) is resolved at the first synchronising call
  bool create_pending = false;
  CholStatus* hst = nullptr;            // pinned
  cudaEvent_t ev_create = nullptr;      // after the whole setup and the status copy
  // first-time workspace allocations: a stream with nothing queued, so allocating does not wait for
  // the (possibly still running) factorisation on the context's stream
  cudaStream_t alloc_stream = nullptr;
};

namespace {

struct DeviceGuard {
  int prev = -1;
  explicit DeviceGuard(int dev) {
    if (cudaGetDevice(&prev) != cudaSuccess) prev = -1;
    if (prev != dev) cudaSetDevice(dev);
  }
  ~DeviceGuard() {
    int cur = -1;
    if (prev >= 0 && cudaGetDevice(&cur) == cudaSuccess && cur != prev) cudaSetDevice(prev);
  }
};

// NVTX (header-only v3; a no-op unless a tool such as Nsight Systems is attached): ranges in the "gls"
// domain around the API calls and, in the Alg. 8 streams, around each chunk's H2D / compute / D2H
// enqueue, and names on the context's streams, so a timeline shows Alg. 8's overlap directly.
nvtxDomainHandle_t nvtx_domain() {
  static nvtxDomainHandle_t d = nvtxDomainCreateA("gls");
  return d;
}
struct NvtxRange {
  explicit NvtxRange(const char* name) {
    nvtxEventAttributes_t a = {};
    a.version = NVTX_VERSION;
    a.size = NVTX_EVENT_ATTRIB_STRUCT_SIZE;
    a.messageType = NVTX_MESSAGE_TYPE_ASCII;
    a.message.ascii = name;
    nvtxDomainRangePushEx(nvtx_domain(), &a);
  }
  void end() {
    if (open_) nvtxDomainRangePop(nvtx_domain());
    open_ = false;
  }
  ~NvtxRange() { end(); }
  bool open_ = true;
};

int fail_cuda(gls_ctx* c, cudaError_t e, const char* what) {
  if (c) {
    c->err = std::string(what) + ": " + cudaGetErrorString(e);
  }
  cudaGetLastError();
  return e == cudaErrorMemoryAllocation ? GLS_ERR_OOM : GLS_ERR_CUDA;
}

#define CK(ctx, call)                                          \
  do {                                                         \
    cudaError_t e_ = (call);                                   \
    if (e_ != cudaSuccess) return fail_cuda((ctx), e_, #call); \
  } while (0)

bool is_device_ptr(const void* p) {
  cudaPointerAttributes at;
  if (cudaPointerGetAttributes(&at, p) != cudaSuccess) {
    cudaGetLastError();
    return false;
  }
  return at.type == cudaMemoryTypeDevice || at.type == cudaMemoryTypeManaged;
}

// Device memory comes from a private stream-ordered pool per device (cudaMemPoolCreate, created
// on first use; cudaMallocFromPoolAsync on the context's own stream).  Freed blocks stay cached in
// it (release threshold GLS_POOL_KEEP_BYTES, default 32 GiB -- the two FP64 host staging buffers
// alone are 12 GB at n = 1e4) so a create/destroy cycle does not pay page unmapping and remapping
// every time (measured: with 8 GiB, destroying a context after a FP64 host-input solve took
// 0.3-3.6 s and the next solve's first touch ~0.7 s more).  Being private, the cache never raises
// the threshold of the device's default pool that PyTorch and other allocators rely on, and
// gls_release_cached_memory hands it back to the driver.
constexpr int kMaxDevices = 64;
std::mutex g_pool_mu;
cudaMemPool_t g_pool[kMaxDevices] = {};

}  // namespace

namespace gls {
cudaMemPool_t gls_device_pool(int device) {
  if (device < 0 || device >= kMaxDevices) return nullptr;
  std::lock_guard<std::mutex> lk(g_pool_mu);
  if (g_pool[device]) return g_pool[device];
  cudaMemPoolProps props;
  memset(&props, 0, sizeof props);
  props.allocType = cudaMemAllocationTypePinned;
  props.handleTypes = cudaMemHandleTypeNone;
  props.location.type = cudaMemLocationTypeDevice;
  props.location.id = device;
  cudaMemPool_t pool = nullptr;
  if (cudaMemPoolCreate(&pool, &props) != cudaSuccess) {
    cudaGetLastError();
    return nullptr;
  }
  uint64_t keep = 32ull << 30;
  if (const char* e = getenv("GLS_POOL_KEEP_BYTES")) keep = strtoull(e, nullptr, 10);
  cudaMemPoolSetAttribute(pool, cudaMemPoolAttrReleaseThreshold, &keep);
  // no hidden cross-stream waits: a workspace allocated on the idle alloc_stream while an
  // asynchronous gls_create still runs must not be handed memory whose free is still pending on the
  // context's stream (the allocation would then wait for the whole factorisation)
  int no = 0;
  cudaMemPoolSetAttribute(pool, cudaMemPoolReuseAllowInternalDependencies, &no);
  cudaGetLastError();
  g_pool[device] = pool;
  return pool;
}

// Pinned host slots for the contexts' Cholesky status (CholStatus, 16 bytes each): cudaMallocHost
// once per block of slots and never freed -- a cudaMallocHost / cudaFreeHost pair per context costs
// driver round trips (cudaFreeHost may wait for the device) on every create / destroy.
std::mutex g_slot_mu;
std::vector<CholStatus*> g_free_slots;
CholStatus* status_slot_get() {
  std::lock_guard<std::mutex> lk(g_slot_mu);
  if (g_free_slots.empty()) {
    constexpr int kSlots = 256;
    CholStatus* blk = nullptr;
    if (cudaMallocHost((void**)&blk, kSlots * sizeof(CholStatus)) != cudaSuccess) {
      cudaGetLastError();
      return nullptr;
    }
    for (int k = kSlots - 1; k >= 0; --k) g_free_slots.push_back(blk + k);
  }
  CholStatus* s = g_free_slots.back();
  g_free_slots.pop_back();
  return s;
}
void status_slot_put(CholStatus* s) {
  if (!s) return;
  std::lock_guard<std::mutex> lk(g_slot_mu);
  g_free_slots.push_back(s);
}

// Per-device cache of context streams / events.  Creating and destroying five streams and ~40
// events per context made the driver stall the host for 25-90 ms every ~9 create / destroy cycles
// once the process had seen heavy pinned-memory traffic (bench steps: a 27-63 ms gls_destroy, then
// a 53-93 ms gls_create whose traced phases were normal; profiles/r02_step_outliers.txt).  A
// context now takes its streams and fixed events from here and gives them back idle (every stream
// synchronised) on destroy; timing events likewise.  GLS_RES_CACHE=0 restores create / destroy.
std::mutex g_res_mu;
std::vector<CtxRes> g_res[kMaxDevices];
std::vector<cudaEvent_t> g_tev[kMaxDevices];  // timing-enabled events (gls_set_timing, stream reports)
bool res_cache_on() {
  static const bool v = !(getenv("GLS_RES_CACHE") && atoi(getenv("GLS_RES_CACHE")) == 0);
  return v;
}
bool res_take(int dev, CtxRes* r) {
  if (!res_cache_on() || dev < 0 || dev >= kMaxDevices) return false;
  std::lock_guard<std::mutex> lk(g_res_mu);
  if (g_res[dev].empty()) return false;
  *r = g_res[dev].back();
  g_res[dev].pop_back();
  return true;
}
void res_give(int dev, CtxRes& r) {
  for (cudaStream_t st : {r.own, r.h2d, r.d2h, r.fb, r.alloc})
    if (st) cudaStreamSynchronize(st);
  const bool whole = r.own && r.h2d && r.d2h && r.fb && r.alloc &&
                     std::all_of(std::begin(r.ev), std::end(r.ev), [](cudaEvent_t e) { return e != nullptr; });
  if (res_cache_on() && whole && dev >= 0 && dev < kMaxDevices) {
    std::lock_guard<std::mutex> lk(g_res_mu);
    g_res[dev].push_back(r);
  } else {
    for (cudaEvent_t e : r.ev)
      if (e) cudaEventDestroy(e);
    for (cudaStream_t st : {r.own, r.h2d, r.d2h, r.fb, r.alloc})
      if (st) cudaStreamDestroy(st);
  }
  r = CtxRes{};
}
cudaEvent_t tev_take(int dev) {
  if (res_cache_on() && dev >= 0 && dev < kMaxDevices) {
    std::lock_guard<std::mutex> lk(g_res_mu);
    if (!g_tev[dev].empty()) {
      cudaEvent_t e = g_tev[dev].back();
      g_tev[dev].pop_back();
      return e;
    }
  }
  cudaEvent_t e = nullptr;
  if (cudaEventCreate(&e) != cudaSuccess) {
    cudaGetLastError();
    return nullptr;
  }
  return e;
}
void tev_give(int dev, cudaEvent_t e) {
  if (!e) return;
  if (res_cache_on() && dev >= 0 && dev < kMaxDevices) {
    std::lock_guard<std::mutex> lk(g_res_mu);
    g_tev[dev].push_back(e);
  } else {
    cudaEventDestroy(e);
  }
}

// ordering-only events (no timing) for the host-M upload of a create; every wait on one is enqueued
// within the create that recorded it, so handing it to the next create is safe
std::vector<cudaEvent_t> g_sev[kMaxDevices];
cudaError_t sev_take(int dev, cudaEvent_t* e) {
  if (res_cache_on() && dev >= 0 && dev < kMaxDevices) {
    std::lock_guard<std::mutex> lk(g_res_mu);
    if (!g_sev[dev].empty()) {
      *e = g_sev[dev].back();
      g_sev[dev].pop_back();
      return cudaSuccess;
    }
  }
  return cudaEventCreateWithFlags(e, cudaEventDisableTiming);
}
void sev_give(int dev, cudaEvent_t e) {
  if (!e) return;
  if (res_cache_on() && dev >= 0 && dev < kMaxDevices) {
    std::lock_guard<std::mutex> lk(g_res_mu);
    g_sev[dev].push_back(e);
  } else {
    cudaEventDestroy(e);
  }
}

cudaError_t gls_pool_alloc(void** p, size_t bytes, int device, cudaStream_t s) {
  cudaMemPool_t pool = gls_device_pool(device);
  if (!pool) return cudaErrorMemoryAllocation;
  return cudaMallocFromPoolAsync(p, bytes, pool, s);
}
}  // namespace gls

namespace {

template <typename T>
cudaError_t dalloc(gls_ctx* c, T** p, size_t bytes) {
  return gls_pool_alloc((void**)p, bytes, c->device, c->own_stream);
}
template <typename T>
void dfree(gls_ctx* c, T*& p) {
  if (p) cudaFreeAsync(p, c->own_stream);
  p = nullptr;
}
// Workspace allocation usable from every stream on return, without waiting for work queued on the
// context's streams (an asynchronous gls_create may still be running there): made on alloc_stream,
// which carries nothing else.  Callers that replace an existing buffer synchronise the device first.
template <typename T>
cudaError_t walloc(gls_ctx* c, T** p, size_t bytes) {
  cudaError_t e = gls_pool_alloc((void**)p, bytes, c->device, c->alloc_stream);
  if (e == cudaSuccess) e = cudaStreamSynchronize(c->alloc_stream);
  return e;
}

int check_dims(int64_t n, int32_t pL, int32_t pR) {
  if (pL < 0 || pR < 1) return GLS_ERR_DIM;
  const int64_t p = (int64_t)pL + pR;
  if (p > 20 || n <= p || n > (int64_t)INT32_MAX / 2) return GLS_ERR_DIM;
  return GLS_OK;
}

int ctx_init(gls_ctx* c, int64_t n, int32_t pL, int32_t pR, bool fp64_state = true) {
  c->n = n;
  c->pL = pL;
  c->pR = pR;
  c->p = pL + pR;
  c->NW = (pL + 1 + 7) / 8;
  c->NB = (n + kNB - 1) / kNB;
  CK(c, cudaGetDevice(&c->device));
  CK(c, cudaDeviceGetAttribute(&c->num_sms, cudaDevAttrMultiProcessorCount, c->device));
  int prio_lo = 0, prio_hi = 0;  // the context's stream is high priority: in gls_create it carries the
  cudaDeviceGetStreamPriorityRange(&prio_lo, &prio_hi);  // critical path of the factorisation
  CtxRes& r = c->res;
  if (!res_take(c->device, &r)) {
    CK(c, cudaStreamCreateWithPriority(&r.own, cudaStreamNonBlocking, prio_hi));
    CK(c, cudaStreamCreateWithFlags(&r.h2d, cudaStreamNonBlocking));
    CK(c, cudaStreamCreateWithFlags(&r.d2h, cudaStreamNonBlocking));
    CK(c, cudaStreamCreateWithFlags(&r.fb, cudaStreamNonBlocking));
    CK(c, cudaStreamCreateWithFlags(&r.alloc, cudaStreamNonBlocking));
    for (cudaEvent_t& e : r.ev) CK(c, cudaEventCreateWithFlags(&e, cudaEventDisableTiming));
    nvtxNameCudaStreamA(r.own, "gls compute");
    nvtxNameCudaStreamA(r.h2d, "gls h2d (Alg. 8 async_read)");
    nvtxNameCudaStreamA(r.d2h, "gls d2h (Alg. 8 async_write)");
    nvtxNameCudaStreamA(r.fb, "gls fp64 fallback");
    nvtxNameCudaStreamA(r.alloc, "gls alloc");
  }
  c->own_stream = r.own;
  c->h2d = r.h2d;
  c->d2h = r.d2h;
  c->fb = r.fb;
  c->alloc_stream = r.alloc;
  c->stream = c->own_stream;
  for (int k = 0; k < 2; ++k) {
    c->ev_oz[k] = r.ev[0 + k];
    c->ev_fb[k] = r.ev[2 + k];
    c->ev_h2d[k] = r.ev[4 + k];
    c->ev_comp[k] = r.ev[6 + k];
    c->ev_d2h[k] = r.ev[8 + k];
    CK(c, cudaEventRecord(c->ev_fb[k], c->own_stream));
  }
  const PanelGeom pg = panel_geom(pR);
  c->oz_ok = n <= kOzMaxN;
  if (const char* e = getenv("GLS_PATH")) c->path = (strcmp(e, "fp64") == 0) ? GLS_PATH_FP64 : GLS_PATH_AUTO;
  // host-streamed chunks: one wave of FP64 panels, or 4 waves of 128-column int8 tiles
  c->block_cols = c->oz_ok ? (int64_t)c->num_sms * 4 * 4 * (32 / pR) * pR
                           : (int64_t)c->num_sms * pg.cpp;
  c->Tpk_bytes = (size_t)tpk_total_tiles(c->NB) * kTileDoubles * sizeof(double);
  c->Wpk_bytes = (size_t)c->NB * wpk_rb_doubles(c->NW) * sizeof(double);
  c->G_bytes = (size_t)(pL + 1) * (pL + 1) * sizeof(double);
  c->fp64_ok = fp64_state;
  if (fp64_state) {
    CK(c, dalloc(c, &c->Tpk, c->Tpk_bytes));
    CK(c, dalloc(c, &c->Wpk, c->Wpk_bytes));
  } else {
    c->Tpk_bytes = c->Wpk_bytes = 0;
  }
  CK(c, dalloc(c, &c->G, c->G_bytes));
  CK(c, dalloc(c, &c->flags, 2 * sizeof(int) + 2 * sizeof(unsigned long long)));
  CK(c, dalloc(c, &c->ran, 2 * sizeof(unsigned long long)));
  CK(c, cudaMemsetAsync(c->ran, 0, 2 * sizeof(unsigned long long), c->own_stream));
  if (c->oz_ok) {
    const int64_t NBR = (n + kOzR - 1) / kOzR;
    c->T8_bytes = (size_t)oz_total_tiles(NBR) * kOzTileBytes;
    c->aux_bytes = (size_t)NBR * kOzR * (pL + 2) * sizeof(double);
    CK(c, dalloc(c, &c->T8, c->T8_bytes));
    CK(c, dalloc(c, &c->aux, c->aux_bytes));
    c->V8_bytes = (size_t)oz_nchunks(n) * oz_nv(pL + 1) * kOzKC;
    c->vscale_bytes = (size_t)(pL + 1) * sizeof(double);
    CK(c, dalloc(c, &c->V8, c->V8_bytes));
    CK(c, dalloc(c, &c->vscale, c->vscale_bytes));
  }
  CK(c, cudaStreamSynchronize(c->own_stream));  // buffers are used from other streams too
  return GLS_OK;
}

void free_staging(gls_ctx* c) {
  for (int k = 0; k < 2; ++k) {
    dfree(c, c->stage[k]);
    dfree(c, c->bstage[k]);
    dfree(c, c->sstage[k]);
  }
  c->stage_cols = 0;
  c->bstage_groups = 0;
}

// Setup: Alg. 5 lines 1 (potrf), 2 + 4 (X~_L, y~), 5 (S_TL), 6 (b_T).
void set_not_spd(gls_ctx* c, unsigned long long fail) {
  c->failed_pivot = (int64_t)fail;
  char buf[128];
  snprintf(buf, sizeof buf, "M is not SPD: Cholesky pivot %lld <= 2^-52 * max diag", (long long)fail);
  c->err = buf;
}

// async (gls_create_async): everything is enqueued on the context's stream and nothing is waited
// for; the NotSPD outcome is resolved later by resolve_create.
int ctx_setup(gls_ctx* c, const double* M, const double* X_L, const double* y, bool async = false) {
  const int64_t n = c->n;
  const int pL = c->pL;
  cudaStream_t s = c->stream;
  double *A = nullptr, *T = nullptr, *B = nullptr, *W = nullptr;
  int* esc = nullptr;
  double* rmax = nullptr;  // row maxima of T (int8 setup scratch)
  CholStatus* st = nullptr;
  int rc = GLS_OK;
  auto cleanup = [&]() {
    dfree(c, rmax);
    dfree(c, A);
    dfree(c, T);
    dfree(c, B);
    dfree(c, W);
    dfree(c, esc);
    dfree(c, st);
  };
#define CKS(call)                              \
  do {                                         \
    cudaError_t e_ = (call);                   \
    if (e_ != cudaSuccess) {                   \
      rc = fail_cuda(c, e_, #call);            \
      cudaStreamSynchronize(s);                \
      cleanup();                               \
      return rc;                               \
    }                                          \
  } while (0)
  // GLS_TRACE=1 prints host-side phase times of the setup (diagnostics only)
  static const bool trace = getenv("GLS_TRACE") != nullptr;
  auto t0 = std::chrono::steady_clock::now();
  auto mark = [&](const char* what) {
    if (!trace) return;
    cudaStreamSynchronize(s);
    auto t1 = std::chrono::steady_clock::now();
    fprintf(stderr, "[gls] setup %-10s %8.3f ms\n", what,
            std::chrono::duration<double, std::milli>(t1 - t0).count());
    t0 = t1;
  };
  const size_t nn = (size_t)n * (size_t)n * sizeof(double);
  CKS(dalloc(c, &A, nn));
  CKS(dalloc(c, &T, nn));
  CKS(dalloc(c, &B, (size_t)n * (pL + 1) * sizeof(double)));
  CKS(dalloc(c, &W, (size_t)n * (pL + 1) * sizeof(double)));
  CKS(dalloc(c, &st, sizeof(CholStatus)));
  if (!c->hst && !(c->hst = status_slot_get())) CKS(cudaErrorMemoryAllocation);  // status in and out
  if (c->oz_ok) {
    CKS(dalloc(c, &esc, (size_t)((n + kOzR - 1) / kOzR) * kOzR * sizeof(int)));
    CKS(dalloc(c, &rmax, (size_t)((n + kOzR - 1) / kOzR) * kOzR * sizeof(double)));
  }
  mark("alloc");
  if (trace) {  // the private pool's footprint: growth here means the allocations above mapped memory
    uint64_t res = 0, used = 0;
    if (cudaMemPool_t pool = gls::gls_device_pool(c->device)) {
      cudaMemPoolGetAttribute(pool, cudaMemPoolAttrReservedMemCurrent, &res);
      cudaMemPoolGetAttribute(pool, cudaMemPoolAttrUsedMemCurrent, &used);
    }
    fprintf(stderr, "[gls] pool reserved %.3f GB used %.3f GB\n", res / 1e9, used / 1e9);
  }
  // A host M is uploaded in column chunks on the h2d stream while the factorisation runs: the
  // recursion works left to right and waits for the chunks each kernel touches, so only the first
  // chunk's copy is exposed.  The NotSPD tolerance (max of the diagonal) is then taken on the host.
  ColsReady arriving;
  std::vector<cudaEvent_t> col_ev;
  const bool m_host = !is_device_ptr(M) && n >= kUploadChunkCols * 2;
  if (m_host) {
    double mx = 0.0;
    for (int64_t k = 0; k < n; ++k) mx = std::fmax(mx, M[k + k * n]);
    c->hst->tol = std::ldexp(1.0, -52) * mx;
    c->hst->fail = ULLONG_MAX;
    CKS(cudaMemcpyAsync(st, c->hst, sizeof(CholStatus), cudaMemcpyHostToDevice, s));
    {  // the h2d stream writes A: after its (stream-ordered) allocation
      cudaEvent_t ea = nullptr;
      CKS(sev_take(c->device, &ea));
      col_ev.push_back(ea);
      CKS(cudaEventRecord(ea, s));
      CKS(cudaStreamWaitEvent(c->h2d, ea, 0));
    }
    const size_t ev0 = col_ev.size();
    const int64_t nch = (n + kUploadChunkCols - 1) / kUploadChunkCols;
    col_ev.resize(ev0 + (size_t)nch);
    for (int64_t k = 0; k < nch; ++k) {
      const int64_t c0 = k * kUploadChunkCols, c1 = std::min(n, c0 + kUploadChunkCols);
      CKS(sev_take(c->device, &col_ev[ev0 + (size_t)k]));
      CKS(cudaMemcpyAsync(A + c0 * n, M + c0 * n, (size_t)(c1 - c0) * n * sizeof(double), cudaMemcpyHostToDevice,
                          c->h2d));
      CKS(cudaEventRecord(col_ev[ev0 + (size_t)k], c->h2d));
    }
    arriving.cols = kUploadChunkCols;
    arriving.ready = col_ev.data() + ev0;
    arriving.nchunks = nch;
    CKS(cudaMemsetAsync(T, 0, nn, s));
  } else {
    CKS(cudaMemcpyAsync(A, M, nn, cudaMemcpyDefault, s));
    CKS(cudaMemsetAsync(T, 0, nn, s));
  }
  mark("copy+zero");
  if (!m_host) chol_prepare(s, n, A, n, st, &c->launches);
  chol_inv(s, n, A, T, n, st, &c->launches, m_host ? &arriving : nullptr);
  if (m_host) CKS(cudaStreamWaitEvent(s, col_ev.back(), 0));  // M is the caller's again after return
  CKS(cudaGetLastError());
  mark("chol_inv");
  CKS(cudaMemcpyAsync(c->hst, st, sizeof(CholStatus), cudaMemcpyDeviceToHost, s));
  if (!async) {
    CKS(cudaStreamSynchronize(s));
    if (c->hst->fail != ULLONG_MAX) {
      set_not_spd(c, c->hst->fail);
      for (auto e : col_ev) sev_give(c->device, e);
      cleanup();
      return GLS_ERR_NOT_SPD;
    }
  }
  // (async: a failed factorisation leaves NaN / garbage in T; the setup below and any solve enqueued
  // before resolve_create only compute on it -- no address depends on its values -- and their
  // results are discarded when resolve_create reports GLS_ERR_NOT_SPD)
  // B = [X_L | y];  W = T B = [X~_L | y~];  G = W^T W  (S_TL and b_T)
  if (pL > 0) CKS(cudaMemcpyAsync(B, X_L, (size_t)n * pL * sizeof(double), cudaMemcpyDefault, s));
  CKS(cudaMemcpyAsync(B + (size_t)n * pL, y, (size_t)n * sizeof(double), cudaMemcpyDefault, s));
  // W = T B: memory-bound skinny product (the dense A, free after chol_inv, holds its 32 (pL+1) n
  // partial sums when n >= 32 (pL+1); small n takes the tiled GEMM)
  if (n >= 32 * (int64_t)(pL + 1))
    trmm_lower_skinny(s, n, pL + 1, T, n, B, n, W, n, A, &c->launches);
  else
    dgemm(s, n, pL + 1, n, 1.0, T, n, 'N', B, n, 'N', 0.0, W, n, GEMM_KMAX_ROW, &c->launches);
  // G: a (pL+1)^2 output with K = n -- split K over the machine, partial tiles in A (free again once
  // W is formed; it holds the at most 16 (pL+1)^2 partials whenever n^2 does)
  dgemm(s, pL + 1, pL + 1, n, 1.0, W, n, 'T', W, n, 'N', 0.0, c->G, pL + 1, 0, &c->launches,
        n * n >= 16 * (int64_t)(pL + 1) * (pL + 1) ? A : nullptr);
  mark("W,G");
  pack_T(s, T, n, n, c->NB, c->Tpk, &c->launches);
  pack_W(s, W, n, n, pL + 1, c->NB, c->NW, c->Wpk, &c->launches);
  if (c->oz_ok) {
    // V = T^T W = M^{-1} [X_L | y] into B (free again: W = T B is formed)
    trmm_lower_t_skinny(s, n, pL + 1, T, n, W, n, B, n, &c->launches);
    oz_setup(s, T, n, n, W, pL + 1, c->T8, c->aux, esc, B, c->V8, c->vscale, rmax, &c->launches);
  }
  CKS(cudaGetLastError());
  if (async) {
    c->ev_create = c->res.ev[10];
    CKS(cudaEventRecord(c->ev_create, s));
    c->create_pending = true;
  } else {
    CKS(cudaStreamSynchronize(s));
  }
  for (auto e : col_ev) sev_give(c->device, e);  // (a pending event may be re-recorded: waits already enqueued keep their record)
  mark("pack");
  cleanup();  // stream-ordered frees on the context's stream
  mark("free");
#undef CKS
  return GLS_OK;
}

// gls_create_async: wait for the enqueued setup; a failed factorisation puts the context in the
// failed state and returns GLS_ERR_NOT_SPD (once -- later calls see GLS_ERR_STATE).
int resolve_create(gls_ctx* c) {
  if (!c->create_pending) return GLS_OK;
  c->create_pending = false;
  CK(c, cudaEventSynchronize(c->ev_create));
  if (c->hst->fail != ULLONG_MAX) {
    set_not_spd(c, c->hst->fail);
    c->state = ST_FAILED;
    return GLS_ERR_NOT_SPD;
  }
  return GLS_OK;
}

int ensure_scratch(gls_ctx* c, int64_t groups) {
  if (groups <= c->scratch_groups) return GLS_OK;
  if (c->bscratch) CK(c, cudaStreamSynchronize(c->stream));  // the old scratch may still be in use there
  dfree(c, c->bscratch);
  dfree(c, c->sscratch);
  c->scratch_groups = 0;
  CK(c, walloc(c, &c->bscratch, (size_t)groups * c->p * sizeof(double)));
  CK(c, walloc(c, &c->sscratch, (size_t)groups * sizeof(int32_t)));
  c->scratch_groups = groups;
  return GLS_OK;
}

int ensure_staging(gls_ctx* c, int64_t chunk_groups) {
  const int64_t cols = chunk_groups * c->pR;
  const int64_t ld = c->n + (c->n & 1);
  if (c->stage_cols >= cols && c->ld_stage == ld && c->bstage_groups >= chunk_groups) return GLS_OK;
  if (c->stage[0] || c->bstage[0]) CK(c, cudaDeviceSynchronize());  // old buffers may still be in use
  free_staging(c);
  for (int k = 0; k < 2; ++k) {
    CK(c, walloc(c, &c->stage[k], (size_t)ld * cols * sizeof(double)));
    if (ld != c->n) {  // the pad row of the odd-n staged copy must read as zero
      CK(c, cudaMemsetAsync(c->stage[k], 0, (size_t)ld * cols * sizeof(double), c->alloc_stream));
      CK(c, cudaStreamSynchronize(c->alloc_stream));
    }
    CK(c, walloc(c, &c->bstage[k], (size_t)chunk_groups * c->p * sizeof(double)));
    CK(c, walloc(c, &c->sstage[k], (size_t)chunk_groups * sizeof(int32_t)));
  }
  c->stage_cols = cols;
  c->ld_stage = ld;
  c->bstage_groups = chunk_groups;
  return GLS_OK;
}

cudaEvent_t pool_event(gls_ctx* c) {
  if (!c->ev_pool.empty()) {
    cudaEvent_t e = c->ev_pool.back();
    c->ev_pool.pop_back();
    return e;
  }
  return tev_take(c->device);
}
// Brackets one launch on `s` with an event pair when timing is on (diagnostics for bench.py).
struct LaunchTimer {
  gls_ctx* c;
  cudaStream_t s;
  int kind;
  cudaEvent_t a = nullptr;
  LaunchTimer(gls_ctx* c_, cudaStream_t s_, int k) : c(c_), s(s_), kind(k) {
    if (c->timing && (a = pool_event(c))) cudaEventRecord(a, s);
  }
  ~LaunchTimer() {
    if (!a) return;
    cudaEvent_t b = pool_event(c);
    if (!b) return;
    cudaEventRecord(b, s);
    c->tl.push_back({a, b, kind});
  }
};

// A timing event on `s` when stream accounting is on (else nullptr).
cudaEvent_t srep_mark(gls_ctx* c, cudaStream_t s) {
  if (!c->srep) return nullptr;
  cudaEvent_t e = pool_event(c);
  if (e) cudaEventRecord(e, s);
  return e;
}

int run_fp64(gls_ctx* c, const double* X, int64_t ldx, int64_t groups, double* b, int32_t* stt,
             const int* gate, cudaStream_t strm = nullptr, const int* pflag = nullptr, const int* m_dev = nullptr,
             int gate_lo = 0, int gate_hi = INT_MAX) {
  if (!strm) strm = c->stream;
  LaunchTimer lt(c, strm, 1);
  SolveArgs a;
  a.X = X;
  a.ldx = ldx;
  a.n = c->n;
  a.NB = c->NB;
  a.pL = c->pL;
  a.pR = c->pR;
  a.m_blk = groups;
  a.Tpk = c->Tpk;
  a.Wpk = c->Wpk;
  a.G = c->G;
  a.b_out = b;
  a.status_out = stt;
  a.pflag = pflag;
  a.m_dev = m_dev;
  a.gate_lo = gate_lo;
  a.gate_hi = gate_hi;
  std::string msg;
  cudaError_t e = launch_fused_trsm_gls(strm, a, c->num_sms, &msg, &c->launches, gate, c->ran + 1);
  if (e != cudaSuccess) {
    c->err = msg;
    cudaGetLastError();
    return GLS_ERR_CUDA;
  }
  return GLS_OK;
}

int ensure_x8(gls_ctx* c, int64_t cols) {
  const int64_t ld8 = (c->n + 15) & ~(int64_t)15;
  if (c->x8_cols >= cols && c->ld8 == ld8) return GLS_OK;
  if (c->x8[0]) CK(c, cudaDeviceSynchronize());
  dfree(c, c->x8[0]);
  dfree(c, c->x8[1]);
  c->x8_cols = 0;
  for (int k = 0; k < 2; ++k) CK(c, walloc(c, &c->x8[k], (size_t)ld8 * cols));
  c->x8_cols = cols;
  c->ld8 = ld8;
  return GLS_OK;
}

int run_int8(gls_ctx* c, const int8_t* X8, int64_t ld8, int64_t groups, double* b, int32_t* stt,
             const int* gate, const double* cv_X = nullptr, int64_t cv_ldx = 0, int64_t cv_cols = 0,
             int8_t* cv_X8 = nullptr, int* cv_flag = nullptr, const int* pflag = nullptr,
             int* cv_pflag = nullptr) {
  if (c->p > kOzPosvInKernelMaxP && c->sws_groups < groups) {
    if (c->sws) CK(c, cudaDeviceSynchronize());
    dfree(c, c->sws);
    c->sws_groups = 0;
    CK(c, walloc(c, &c->sws, (size_t)groups * c->pR * (c->p + 1) * sizeof(double)));
    c->sws_groups = groups;
  }
  LaunchTimer lt(c, c->stream, 0);
  OzArgs a;
  a.X8 = X8;
  a.ld8 = ld8;
  a.n = c->n;
  a.pL = c->pL;
  a.pR = c->pR;
  a.m_blk = groups;
  a.T8 = c->T8;
  a.aux = c->aux;
  a.G = c->G;
  a.gate = gate;
  a.ran = c->ran;
  a.V8 = c->V8;
  a.vscale = c->vscale;
  a.b_out = b;
  a.status_out = stt;
  a.s_ws = c->p > kOzPosvInKernelMaxP ? c->sws : nullptr;
  a.cv_X = cv_X;
  a.cv_ldx = cv_ldx;
  a.cv_cols = cv_cols;
  a.cv_X8 = cv_X8;
  a.cv_ld8 = ld8;
  a.cv_flag = cv_flag;
  a.pflag = pflag;
  a.gate_all = groups;
  a.cv_pflag = cv_pflag;
  std::string msg;
  cudaError_t e = launch_ozaki_gls(c->stream, a, c->num_sms, &msg, &c->launches);
  if (e != cudaSuccess) {
    c->err = msg;
    cudaGetLastError();
    return GLS_ERR_CUDA;
  }
  return GLS_OK;
}

// An int8-only context (no packed T for the FP64 kernel): a double X block is converted chunk by chunk
// by standalone passes and solved on the int8 path; a chunk that is not integer-valued cannot fall back
// to the FP64 kernel, so the block fails with GLS_ERR_ARG (checked on the host after the block: this
// entry point synchronises).
int run_kernel_int8_only(gls_ctx* c, const double* X, int64_t ldx, int64_t groups, double* b, int32_t* stt) {
  const int pR = c->pR, p = c->p;
  const int64_t cpt = 4 * (int64_t)((32 / pR) * pR);
  const int64_t wave_groups = (int64_t)c->num_sms * cpt / pR;
  const int64_t ld8 = (c->n + 15) & ~(int64_t)15;
  int64_t cap = std::min<int64_t>(8 * wave_groups, kSerialChunkBytes / (ld8 * pR)) / wave_groups * wave_groups;
  if (cap < wave_groups) cap = wave_groups;
  const int64_t chunk = std::min(cap, groups);
  int rc = ensure_x8(c, chunk * pR);
  if (rc) return rc;
  unsigned long long* work = (unsigned long long*)(c->flags + 2);
  CK(c, cudaMemsetAsync(c->flags, 0, sizeof(int), c->stream));
  for (int64_t g0 = 0; g0 < groups; g0 += chunk) {
    const int64_t gc = std::min(chunk, groups - g0);
    CK(c, cudaMemsetAsync(work, 0, sizeof(unsigned long long), c->stream));
    {
      LaunchTimer lt(c, c->stream, 2);
      oz_convert(c->stream, X + (size_t)g0 * pR * ldx, ldx, c->n, gc * pR, c->x8[0], c->ld8, c->flags, work,
                 c->num_sms, &c->launches);
      CK(c, cudaGetLastError());
    }
    rc = run_int8(c, c->x8[0], c->ld8, gc, b + (size_t)g0 * p, stt ? stt + g0 : nullptr, nullptr);
    if (rc) return rc;
  }
  int bad = 0;
  CK(c, cudaMemcpyAsync(&bad, c->flags, sizeof(int), cudaMemcpyDeviceToHost, c->stream));
  CK(c, cudaStreamSynchronize(c->stream));
  if (bad) {
    c->err = "int8-only context: X_R holds a value that is not an integer in [-128, 127] (no FP64 fallback)";
    return GLS_ERR_ARG;
  }
  return GLS_OK;
}

// One block of device-resident double X (column-major, ld = ldx, even, 16-byte aligned).
// Path AUTO: chunks of up to 8 waves of int8 tiles (1, 2, .. 8, 8, ..).  Chunk 0 is converted to int8
// by a standalone pass; every later chunk j+1 is converted by the convert-ahead warps of the int8
// kernel of chunk j, concurrently with its tensor-core work, into the other of the two int8
// workspaces.  The path is chosen per problem: a problem whose pR columns hold a value that is not an
// integer in [-128, 127] is flagged (pflags[g] = 1, counted in cflags[j]) and solved by the FP64 kernel,
// every other problem by the int8 kernel -- so a problem's bits depend on its own values only, not on
// its neighbours or the block partition.  Each chunk's int8 launch is gated on the device by the chunk's
// count (skipped when every problem is flagged) and stores no flagged problem; after the last chunk the
// FP64 kernel solves the block's flagged problems (compacted into a dense block when they fit, else in
// place on the panels holding one), also gated on the device, and the host never waits.
int run_kernel(gls_ctx* c, const double* X, int64_t ldx, int64_t groups, double* b, int32_t* stt) {
  if (!c->fp64_ok) return run_kernel_int8_only(c, X, ldx, groups, b, stt);
  if (c->path == GLS_PATH_FP64 || !c->oz_ok) return run_fp64(c, X, ldx, groups, b, stt, nullptr);
  const int pR = c->pR, p = c->p;
  const int64_t cpt = 4 * (int64_t)((32 / pR) * pR);
  const int64_t wave_groups = (int64_t)c->num_sms * cpt / pR;
  // convert-ahead needs the kernel's tensor work per column (~n^2) to cover the conversion of the
  // next chunk's column (8n bytes): at small n the convert-ahead warps would become the bottleneck
  // (n = 1500: kernel 1.8 -> 3.5 ms), and the conversion runs as standalone passes instead
  const bool ahead = c->n >= kConvertAheadMinN;
  std::vector<int64_t> bnd{0};
  if (ahead) {
    for (int64_t j = 1; bnd.back() < groups; ++j)
      bnd.push_back(std::min(groups, bnd.back() + std::min<int64_t>(j, 8) * wave_groups));
  } else {
    // nothing to hide the passes behind: chunks of 8 waves (one pass and one solve launch each; the
    // int8/FP64 path is decided per chunk) within the workspace budget
    const int64_t ld8 = (c->n + 15) & ~(int64_t)15;
    int64_t cap = std::min<int64_t>(8 * wave_groups, kSerialChunkBytes / (ld8 * pR)) / wave_groups * wave_groups;
    if (cap < wave_groups) cap = wave_groups;
    for (int64_t g = 0; g < groups; g += cap) bnd.push_back(std::min(groups, g + cap));
  }
  const int64_t nchunks = (int64_t)bnd.size() - 1;
  int64_t chunk_groups = 0;
  for (int64_t j = 0; j < nchunks; ++j) chunk_groups = std::max(chunk_groups, bnd[j + 1] - bnd[j]);
  int rc = ensure_x8(c, chunk_groups * pR);
  if (rc) return rc;
  if (c->cflags_cap < nchunks) {
    if (c->cflags) CK(c, cudaDeviceSynchronize());
    dfree(c, c->cflags);
    c->cflags_cap = 0;
    const int64_t cap = std::max<int64_t>(nchunks, 256);
    CK(c, walloc(c, &c->cflags, (size_t)cap * sizeof(int)));
    c->cflags_cap = cap;
  }
  if (c->pflags_cap < groups) {
    if (c->pflags) CK(c, cudaDeviceSynchronize());
    dfree(c, c->pflags);
    c->pflags_cap = 0;
    const int64_t cap = std::max<int64_t>(groups, 65536);
    CK(c, walloc(c, &c->pflags, (size_t)cap * sizeof(int)));
    c->pflags_cap = cap;
  }
  int* const pf = c->pflags;
  // the FP64 fallback of the block's flagged problems runs after its int8 launches: up to fcap of them
  // gathered into a dense block (kFbCompactBytes of columns), more in place on the panels holding one
  constexpr size_t kFbCompactBytes = (size_t)512 << 20;
  const int64_t gpp = panel_geom(pR).gpp;
  int64_t fcap = std::min<int64_t>(groups, (int64_t)(kFbCompactBytes / ((size_t)pR * ldx * sizeof(double))));
  fcap = std::max<int64_t>(fcap / gpp * gpp, gpp);
  if (c->fb_cap < fcap || c->fb_ldx != ldx) {
    if (c->fb_X) CK(c, cudaDeviceSynchronize());
    dfree(c, c->fb_idx);
    dfree(c, c->fb_X);
    dfree(c, c->fb_b);
    dfree(c, c->fb_s);
    c->fb_cap = 0;
    CK(c, walloc(c, &c->fb_idx, (size_t)(fcap + 1) * sizeof(int)));  // + the block's flagged count
    CK(c, walloc(c, &c->fb_X, (size_t)fcap * pR * ldx * sizeof(double)));
    CK(c, walloc(c, &c->fb_b, (size_t)fcap * p * sizeof(double)));
    CK(c, walloc(c, &c->fb_s, (size_t)fcap * sizeof(int32_t)));
    c->fb_cap = fcap;
    c->fb_ldx = ldx;
  }
  // the flags of the previous block were last read by its FP64 launches on this stream
  CK(c, cudaMemsetAsync(c->cflags, 0, (size_t)nchunks * sizeof(int), c->stream));
  CK(c, cudaMemsetAsync(pf, 0, (size_t)groups * sizeof(int), c->stream));
  unsigned long long* work = (unsigned long long*)(c->flags + 2);
  CK(c, cudaMemsetAsync(work, 0, sizeof(unsigned long long), c->stream));
  {
    LaunchTimer lt(c, c->stream, 2);
    oz_convert(c->stream, X, ldx, c->n, (bnd[1] - bnd[0]) * pR, c->x8[0], c->ld8, c->cflags, work, c->num_sms,
               &c->launches, pf, pR);
    CK(c, cudaGetLastError());
  }
  for (int64_t j = 0; j < nchunks; ++j) {
    const int buf = (int)(j & 1);
    const int64_t g0 = bnd[j], gc = bnd[j + 1] - bnd[j];
    if (!ahead && j > 0) {
      CK(c, cudaMemsetAsync(work, 0, sizeof(unsigned long long), c->stream));
      LaunchTimer lt(c, c->stream, 2);
      oz_convert(c->stream, X + (size_t)g0 * pR * ldx, ldx, c->n, gc * pR, c->x8[buf], c->ld8, c->cflags + j,
                 work, c->num_sms, &c->launches, pf + g0, pR);
      CK(c, cudaGetLastError());
    }
    // cflags[j] is final here (written by chunk j-1's kernel or a standalone pass)
    double* bj = b + (size_t)g0 * p;
    int32_t* sj = stt ? stt + g0 : nullptr;
    if (ahead && j + 1 < nchunks)
      rc = run_int8(c, c->x8[buf], c->ld8, gc, bj, sj, c->cflags + j, X + (size_t)bnd[j + 1] * pR * ldx, ldx,
                    (bnd[j + 2] - bnd[j + 1]) * pR, c->x8[buf ^ 1], c->cflags + j + 1, pf + g0, pf + bnd[j + 1]);
    else
      rc = run_int8(c, c->x8[buf], c->ld8, gc, bj, sj, c->cflags + j, nullptr, 0, 0, nullptr, nullptr, pf + g0);
    if (rc) return rc;
  }
  // FP64 for the block's flagged problems, after every int8 launch (an FP64 panel is a long one-CTA
  // trsm: beside a persistent int8 kernel it would hold back that kernel's last CTA pair), each launch
  // gated on the device by the flagged count (all of them return at once for genotype blocks)
  int* const fcount = c->fb_idx + fcap;
  fb_compact(c->stream, pf, groups, c->cflags, (int)nchunks, (int)fcap, c->fb_idx, fcount, X, ldx, pR, c->fb_X,
             c->num_sms, &c->launches);
  rc = run_fp64(c, c->fb_X, ldx, fcap, c->fb_b, c->fb_s, fcount, c->stream, nullptr, fcount, 0, (int)fcap);
  if (rc) return rc;
  fb_scatter(c->stream, c->fb_b, c->fb_s, c->fb_idx, fcount, (int)fcap, p, b, stt, c->num_sms, &c->launches);
  CK(c, cudaGetLastError());
  return run_fp64(c, X, ldx, groups, b, stt, fcount, c->stream, pf, nullptr, (int)fcap, INT_MAX);
}

// Alg. 8 with host DRAM -> HBM in place of disk -> RAM: chunk j+1 is copied
// into workspace (j+1)%2 on the h2d stream while chunk j is computed from workspace j%2; b of
// chunk j is copied back on the d2h stream.  Event waits reproduce the algorithm's two waits:
// "wait(current X_blk)" (compute waits ev_h2d) and "wait(previous b_blk)" (workspace reuse waits
// ev_comp / ev_d2h of the chunk that used it two iterations ago).
int solve_streamed(gls_ctx* c, const double* X_R, int64_t m_blk, double* b_out, bool b_dev,
                   int32_t* status_out, bool s_dev) {
  const int pR = c->pR, p = c->p;
  const int64_t n = c->n;
  int64_t chunk_groups = c->block_cols / pR;
  if (chunk_groups < 1) chunk_groups = 1;
  if (chunk_groups > m_blk) chunk_groups = m_blk;
  int rc = ensure_staging(c, chunk_groups);
  if (rc) return rc;
  const int64_t ld = c->ld_stage;
  for (int64_t g0 = 0; g0 < m_blk; g0 += chunk_groups) {
    const int64_t gc = (m_blk - g0 < chunk_groups) ? m_blk - g0 : chunk_groups;
    const int buf = (int)(c->seq++ & 1);
    const double* src = X_R + (size_t)g0 * pR * n;
    gls_ctx::ChunkRec rec{};
    NvtxRange nr_read("Alg. 8 async_read(X_blk)");
    CK(c, cudaStreamWaitEvent(c->h2d, c->ev_comp[buf], 0));
    rec.h0 = srep_mark(c, c->h2d);
    if (ld == n)
      CK(c, cudaMemcpyAsync(c->stage[buf], src, (size_t)n * gc * pR * sizeof(double), cudaMemcpyDefault,
                            c->h2d));
    else
      CK(c, cudaMemcpy2DAsync(c->stage[buf], ld * sizeof(double), src, n * sizeof(double),
                              n * sizeof(double), gc * pR, cudaMemcpyDefault, c->h2d));
    rec.h1 = srep_mark(c, c->h2d);
    rec.hbytes = (int64_t)n * gc * pR * (int64_t)sizeof(double);
    CK(c, cudaEventRecord(c->ev_h2d[buf], c->h2d));
    nr_read.end();
    NvtxRange nr_comp("Alg. 8 wait(X_blk), trsm + assembly + posv");
    if (g0 == 0) rec.cr = srep_mark(c, c->stream);
    CK(c, cudaStreamWaitEvent(c->stream, c->ev_h2d[buf], 0));  // wait(current X_blk)
    CK(c, cudaStreamWaitEvent(c->stream, c->ev_d2h[buf], 0));  // wait(previous b_blk) of this workspace
    rec.c0 = srep_mark(c, c->stream);
    double* bdst = b_dev ? b_out + (size_t)g0 * p : c->bstage[buf];
    int32_t* sdst = status_out ? (s_dev ? status_out + g0 : c->sstage[buf]) : nullptr;
    rc = run_kernel(c, c->stage[buf], ld, gc, bdst, sdst);
    if (rc) return rc;
    rec.c1 = srep_mark(c, c->stream);
    CK(c, cudaEventRecord(c->ev_comp[buf], c->stream));
    nr_comp.end();
    NvtxRange nr_write("Alg. 8 async_write(b_blk)");
    if (!b_dev || (status_out && !s_dev)) {
      CK(c, cudaStreamWaitEvent(c->d2h, c->ev_comp[buf], 0));
      rec.d0 = srep_mark(c, c->d2h);
      if (!b_dev)
        CK(c, cudaMemcpyAsync(b_out + (size_t)g0 * p, c->bstage[buf], (size_t)gc * p * sizeof(double),
                              cudaMemcpyDeviceToHost, c->d2h));
      if (status_out && !s_dev)
        CK(c, cudaMemcpyAsync(status_out + g0, c->sstage[buf], (size_t)gc * sizeof(int32_t),
                              cudaMemcpyDeviceToHost, c->d2h));
      rec.d1 = srep_mark(c, c->d2h);
      rec.dbytes = (int64_t)gc * ((b_dev ? 0 : p * (int64_t)sizeof(double)) +
                                  ((status_out && !s_dev) ? (int64_t)sizeof(int32_t) : 0));
      CK(c, cudaEventRecord(c->ev_d2h[buf], c->d2h));
    }
    if (c->srep) c->srec.push_back(rec);
  }
  return GLS_OK;
}

int ensure_stage8(gls_ctx* c, int64_t cols) {
  const int64_t ld8 = (c->n + 15) & ~(int64_t)15;
  if (c->stage8_cols >= cols && c->ld8 == ld8) return GLS_OK;
  if (c->stage8[0]) CK(c, cudaDeviceSynchronize());
  for (int k = 0; k < 2; ++k) {
    dfree(c, c->stage8[k]);
    dfree(c, c->raw8[k]);
  }
  c->stage8_cols = 0;
  for (int k = 0; k < 2; ++k) {
    CK(c, walloc(c, &c->stage8[k], (size_t)ld8 * cols));
    if (ld8 != c->n) CK(c, walloc(c, &c->raw8[k], (size_t)c->n * cols));
  }
  c->stage8_cols = cols;
  c->ld8 = ld8;
  return GLS_OK;
}

// Genotype codes (int8) from host memory, or from device memory with an unaligned layout:
// the same double-buffered stream as solve_streamed (Alg. 8), one byte per genotype on the link.
int solve_streamed_i8(gls_ctx* c, const int8_t* G, int64_t ldg, int64_t m_blk, double* b_out, bool b_dev,
                      int32_t* status_out, bool s_dev) {
  const int pR = c->pR, p = c->p;
  const int64_t n = c->n;
  int64_t chunk_groups = c->block_cols / pR;
  if (chunk_groups < 1) chunk_groups = 1;
  if (chunk_groups > m_blk) chunk_groups = m_blk;
  int rc = ensure_stage8(c, chunk_groups * pR);
  if (rc) return rc;
  if (!b_dev || (status_out && !s_dev)) {
    // the b / status staging of the double path, sized for these chunks
    if (c->bstage_groups < chunk_groups) {
      if (c->bstage[0]) CK(c, cudaDeviceSynchronize());
      for (int k = 0; k < 2; ++k) {
        dfree(c, c->bstage[k]);
        dfree(c, c->sstage[k]);
        CK(c, walloc(c, &c->bstage[k], (size_t)chunk_groups * p * sizeof(double)));
        CK(c, walloc(c, &c->sstage[k], (size_t)chunk_groups * sizeof(int32_t)));
      }
      c->bstage_groups = chunk_groups;
    }
  }
  // a quarter-size first chunk (the warm-up block of §4.3): the first copy is the
  // one nothing hides
  const int64_t first = (m_blk > chunk_groups && chunk_groups >= 4) ? chunk_groups / 4 : chunk_groups;
  for (int64_t g0 = 0, gc = 0; g0 < m_blk; g0 += gc) {
    gc = std::min<int64_t>(m_blk - g0, g0 == 0 ? first : chunk_groups);
    const int buf = (int)(c->seq++ & 1);
    NvtxRange nr_read("Alg. 8 async_read(X_blk)");
    CK(c, cudaStreamWaitEvent(c->h2d, c->ev_comp[buf], 0));
    // contiguous rows whose length is not a multiple of 16 bytes (the TMA row pitch): one linear copy
    // (a pitched copy of short rows runs at a fraction of the link rate), repacked on the device
    const bool repack = ldg == n && c->ld8 != n;
    gls_ctx::ChunkRec rec{};
    rec.h0 = srep_mark(c, c->h2d);
    if (repack)
      CK(c, cudaMemcpyAsync(c->raw8[buf], G + (size_t)g0 * pR * ldg, (size_t)gc * pR * n, cudaMemcpyDefault,
                            c->h2d));
    else
      CK(c, cudaMemcpy2DAsync(c->stage8[buf], c->ld8, G + (size_t)g0 * pR * ldg, ldg, n, gc * pR,
                              cudaMemcpyDefault, c->h2d));
    rec.h1 = srep_mark(c, c->h2d);
    rec.hbytes = (int64_t)n * gc * pR;
    CK(c, cudaEventRecord(c->ev_h2d[buf], c->h2d));
    nr_read.end();
    NvtxRange nr_comp("Alg. 8 wait(X_blk), trsm + assembly + posv");
    if (g0 == 0) rec.cr = srep_mark(c, c->stream);
    CK(c, cudaStreamWaitEvent(c->stream, c->ev_h2d[buf], 0));  // wait(current X_blk)
    CK(c, cudaStreamWaitEvent(c->stream, c->ev_d2h[buf], 0));  // wait(previous b_blk) of this workspace
    rec.c0 = srep_mark(c, c->stream);
    if (repack) {
      oz_repack_rows(c->stream, c->raw8[buf], n, gc * pR, c->stage8[buf], c->ld8, &c->launches);
      CK(c, cudaGetLastError());
    }
    double* bdst = b_dev ? b_out + (size_t)g0 * p : c->bstage[buf];
    int32_t* sdst = status_out ? (s_dev ? status_out + g0 : c->sstage[buf]) : nullptr;
    rc = run_int8(c, c->stage8[buf], c->ld8, gc, bdst, sdst, nullptr);
    if (rc) return rc;
    rec.c1 = srep_mark(c, c->stream);
    CK(c, cudaEventRecord(c->ev_comp[buf], c->stream));
    nr_comp.end();
    NvtxRange nr_write("Alg. 8 async_write(b_blk)");
    if (!b_dev || (status_out && !s_dev)) {
      CK(c, cudaStreamWaitEvent(c->d2h, c->ev_comp[buf], 0));
      rec.d0 = srep_mark(c, c->d2h);
      if (!b_dev)
        CK(c, cudaMemcpyAsync(b_out + (size_t)g0 * p, c->bstage[buf], (size_t)gc * p * sizeof(double),
                              cudaMemcpyDeviceToHost, c->d2h));
      if (status_out && !s_dev)
        CK(c, cudaMemcpyAsync(status_out + g0, c->sstage[buf], (size_t)gc * sizeof(int32_t),
                              cudaMemcpyDeviceToHost, c->d2h));
      rec.d1 = srep_mark(c, c->d2h);
      rec.dbytes = (int64_t)gc * ((b_dev ? 0 : p * (int64_t)sizeof(double)) +
                                  ((status_out && !s_dev) ? (int64_t)sizeof(int32_t) : 0));
      CK(c, cudaEventRecord(c->ev_d2h[buf], c->d2h));
    }
    if (c->srep) c->srec.push_back(rec);
  }
  return GLS_OK;
}

// Every synchronising entry point ends here: all of the context's streams drained, and the outcome
// of an asynchronous gls_create resolved (GLS_ERR_NOT_SPD once if the factorisation failed).
int sync_all(gls_ctx* c) {
  CK(c, cudaStreamSynchronize(c->h2d));
  CK(c, cudaStreamSynchronize(c->fb));
  CK(c, cudaStreamSynchronize(c->stream));
  CK(c, cudaStreamSynchronize(c->d2h));
  return resolve_create(c);
}

}  // namespace

extern "C" {

const char* gls_error_string(int code) {
  switch (code) {
    case GLS_OK: return "GLS_OK: success";
    case GLS_ERR_ARG: return "GLS_ERR_ARG: invalid argument (NULL pointer or bad flag)";
    case GLS_ERR_DIM: return "GLS_ERR_DIM: dimensions must satisfy n > pL+pR, pL >= 0, pR >= 1, pL+pR <= 20, m_blk >= 1";
    case GLS_ERR_NOT_SPD: return "GLS_ERR_NOT_SPD: M is not symmetric positive definite";
    case GLS_ERR_CUDA: return "GLS_ERR_CUDA: CUDA error (see gls_last_error)";
    case GLS_ERR_OOM: return "GLS_ERR_OOM: out of device or pinned memory";
    case GLS_ERR_STATE: return "GLS_ERR_STATE: context failed or not committed";
    default: return "unknown gls error code";
  }
}

int gls_create(int64_t n, int32_t pL, int32_t pR, const double* M, const double* X_L,
               const double* y, gls_ctx** out) {
  if (!out) return GLS_ERR_ARG;
  *out = nullptr;
  if (!M || !y || (pL > 0 && !X_L)) return GLS_ERR_ARG;
  int rc = check_dims(n, pL, pR);
  if (rc) return rc;
  NvtxRange nr("gls_create");
  gls_ctx* c = new gls_ctx();
  *out = c;
  rc = ctx_init(c, n, pL, pR);
  if (rc) return rc;
  DeviceGuard g(c->device);
  rc = ctx_setup(c, M, X_L, y);
  if (rc) return rc;
  c->state = ST_OK;
  return GLS_OK;
}

int gls_create_async(int64_t n, int32_t pL, int32_t pR, const double* M, const double* X_L,
                     const double* y, gls_ctx** out) {
  if (!out) return GLS_ERR_ARG;
  *out = nullptr;
  if (!M || !y || (pL > 0 && !X_L)) return GLS_ERR_ARG;
  int rc = check_dims(n, pL, pR);
  if (rc) return rc;
  NvtxRange nr("gls_create_async");
  gls_ctx* c = new gls_ctx();
  *out = c;
  rc = ctx_init(c, n, pL, pR);
  if (rc) return rc;
  DeviceGuard g(c->device);
  rc = ctx_setup(c, M, X_L, y, true);
  if (rc) return rc;
  c->state = ST_OK;  // tentatively: resolve_create (any synchronising call) may still fail it
  return GLS_OK;
}

int gls_create_adopt(int64_t n, int32_t pL, int32_t pR, gls_ctx** out) {
  if (!out) return GLS_ERR_ARG;
  *out = nullptr;
  int rc = check_dims(n, pL, pR);
  if (rc) return rc;
  gls_ctx* c = new gls_ctx();
  *out = c;
  rc = ctx_init(c, n, pL, pR);
  if (rc) return rc;
  c->state = ST_ADOPT;
  return GLS_OK;
}

int gls_create_adopt_int8(int64_t n, int32_t pL, int32_t pR, gls_ctx** out) {
  if (!out) return GLS_ERR_ARG;
  *out = nullptr;
  int rc = check_dims(n, pL, pR);
  if (rc) return rc;
  if (n > kOzMaxN) return GLS_ERR_DIM;
  gls_ctx* c = new gls_ctx();
  *out = c;
  rc = ctx_init(c, n, pL, pR, false);
  if (rc) return rc;
  c->state = ST_ADOPT;
  return GLS_OK;
}

int gls_shared_view_ex(gls_ctx* c, int32_t flags, void** ptrs, int64_t* bytes, int32_t* count) {
  if (!c || !ptrs || !bytes || !count || (flags & ~GLS_SHARE_INT8_ONLY)) return GLS_ERR_ARG;
  if (c->state == ST_FAILED) return GLS_ERR_STATE;
  const bool fp64 = c->fp64_ok && !(flags & GLS_SHARE_INT8_ONLY);
  if (!fp64 && !c->oz_ok) return GLS_ERR_STATE;
  if (c->create_pending) {  // the views are read by the caller's collectives: the setup must be done
    DeviceGuard g(c->device);
    const int rc = sync_all(c);
    if (rc) return rc;
  }
  int k = 0;
  if (fp64) {
    ptrs[k] = c->Tpk;
    bytes[k++] = (int64_t)c->Tpk_bytes;
    ptrs[k] = c->Wpk;
    bytes[k++] = (int64_t)c->Wpk_bytes;
  }
  ptrs[k] = c->G;
  bytes[k++] = (int64_t)c->G_bytes;
  if (c->oz_ok) {
    ptrs[k] = c->T8;
    bytes[k++] = (int64_t)c->T8_bytes;
    ptrs[k] = c->aux;
    bytes[k++] = (int64_t)c->aux_bytes;
    ptrs[k] = c->V8;
    bytes[k++] = (int64_t)c->V8_bytes;
    ptrs[k] = c->vscale;
    bytes[k++] = (int64_t)c->vscale_bytes;
  }
  *count = k;
  return GLS_OK;
}

int gls_shared_view(gls_ctx* c, void** ptrs, int64_t* bytes, int32_t* count) {
  return gls_shared_view_ex(c, 0, ptrs, bytes, count);
}

int gls_commit_shared(gls_ctx* c) {
  if (!c) return GLS_ERR_ARG;
  if (c->state == ST_FAILED) return GLS_ERR_STATE;
  DeviceGuard g(c->device);
  CK(c, cudaDeviceSynchronize());
  c->state = ST_OK;
  return GLS_OK;
}

int gls_solve_block_ex(gls_ctx* c, const double* X_R, int64_t m_blk, double* b_out,
                       int32_t* status_out, int async) {
  if (!c) return GLS_ERR_ARG;
  if (c->state != ST_OK) return GLS_ERR_STATE;
  if (!X_R || !b_out || (async != 0 && async != 1)) return GLS_ERR_ARG;
  if (m_blk < 1) return GLS_ERR_DIM;
  NvtxRange nr("gls_solve_block");
  DeviceGuard g(c->device);
  c->err.clear();
  const bool x_dev = is_device_ptr(X_R);
  const bool b_dev = is_device_ptr(b_out);
  const bool s_dev = status_out ? is_device_ptr(status_out) : false;
  int rc;
  const bool direct = x_dev && (c->n % 2 == 0) && (((uintptr_t)X_R & 15) == 0);
  if (direct) {
    double* bdst = b_out;
    int32_t* sdst = status_out;
    if (!b_dev || (status_out && !s_dev)) {
      rc = ensure_scratch(c, m_blk);
      if (rc) return rc;
      if (!b_dev) bdst = c->bscratch;
      if (status_out && !s_dev) sdst = c->sscratch;
    }
    rc = run_kernel(c, X_R, c->n, m_blk, bdst, sdst);
    if (rc) return rc;
    if (!b_dev)
      CK(c, cudaMemcpyAsync(b_out, bdst, (size_t)m_blk * c->p * sizeof(double), cudaMemcpyDeviceToHost,
                            c->stream));
    if (status_out && !s_dev)
      CK(c, cudaMemcpyAsync(status_out, sdst, (size_t)m_blk * sizeof(int32_t), cudaMemcpyDeviceToHost,
                            c->stream));
  } else {
    rc = solve_streamed(c, X_R, m_blk, b_out, b_dev, status_out, s_dev);
    if (rc) return rc;
  }
  if (!async) return sync_all(c);
  return GLS_OK;
}

int gls_solve_block_i8(gls_ctx* c, const int8_t* G, int64_t ldg, int64_t m_blk, double* b_out,
                       int32_t* status_out, int async) {
  if (!c) return GLS_ERR_ARG;
  if (c->state != ST_OK) return GLS_ERR_STATE;
  if (!G || !b_out || (async != 0 && async != 1) || ldg < c->n) return GLS_ERR_ARG;
  if (m_blk < 1) return GLS_ERR_DIM;
  if (!c->oz_ok) {
    c->err = "gls_solve_block_i8 needs n <= 131071 (exact int32 digit products)";
    return GLS_ERR_DIM;
  }
  NvtxRange nr("gls_solve_block_i8");
  DeviceGuard g(c->device);
  c->err.clear();
  const bool x_dev = is_device_ptr(G);
  const bool b_dev = is_device_ptr(b_out);
  const bool s_dev = status_out ? is_device_ptr(status_out) : false;
  int rc;
  if (x_dev && ldg % 16 == 0 && ((uintptr_t)G & 15) == 0) {
    double* bdst = b_out;
    int32_t* sdst = status_out;
    if (!b_dev || (status_out && !s_dev)) {
      rc = ensure_scratch(c, m_blk);
      if (rc) return rc;
      if (!b_dev) bdst = c->bscratch;
      if (status_out && !s_dev) sdst = c->sscratch;
    }
    // one launch covers at most 2^31 - 1 columns (TMA coordinates are int32)
    const int64_t max_groups = ((int64_t)1 << 30) / c->pR;
    for (int64_t g0 = 0; g0 < m_blk; g0 += max_groups) {
      const int64_t gc = (m_blk - g0 < max_groups) ? m_blk - g0 : max_groups;
      rc = run_int8(c, G + (size_t)g0 * c->pR * ldg, ldg, gc, bdst + (size_t)g0 * c->p,
                    sdst ? sdst + g0 : nullptr, nullptr);
      if (rc) return rc;
    }
    if (!b_dev)
      CK(c, cudaMemcpyAsync(b_out, bdst, (size_t)m_blk * c->p * sizeof(double), cudaMemcpyDeviceToHost,
                            c->stream));
    if (status_out && !s_dev)
      CK(c, cudaMemcpyAsync(status_out, sdst, (size_t)m_blk * sizeof(int32_t), cudaMemcpyDeviceToHost,
                            c->stream));
  } else {
    rc = solve_streamed_i8(c, G, ldg, m_blk, b_out, b_dev, status_out, s_dev);
    if (rc) return rc;
  }
  if (!async) return sync_all(c);
  return GLS_OK;
}

int gls_set_timing(gls_ctx* c, int32_t enable) {
  if (!c) return GLS_ERR_ARG;
  c->timing = enable != 0;
  return GLS_OK;
}

int gls_read_timing(gls_ctx* c, double* ms_int8, double* ms_fp64, double* ms_conv, int64_t* launches) {
  if (!c || !ms_int8 || !ms_fp64 || !ms_conv || !launches) return GLS_ERR_ARG;
  DeviceGuard g(c->device);
  int rc = sync_all(c);
  if (rc) return rc;
  double t[3] = {0, 0, 0};
  static const bool trace = getenv("GLS_TRACE_LAUNCHES") != nullptr;  // diagnostics: the timeline
  for (auto& x : c->tl) {
    float ms = 0.f;
    CK(c, cudaEventElapsedTime(&ms, x.a, x.b));
    t[x.kind] += ms;
    if (trace) {
      float t0 = 0.f;
      cudaEventElapsedTime(&t0, c->tl.front().a, x.a);
      static const char* kinds[3] = {"int8", "fp64", "conv"};
      fprintf(stderr, "[gls] launch %-4s start %9.3f ms  dur %8.3f ms\n", kinds[x.kind], t0, ms);
    }
    c->ev_pool.push_back(x.a);
    c->ev_pool.push_back(x.b);
  }
  *launches = (int64_t)c->tl.size();
  c->tl.clear();
  *ms_int8 = t[0];
  *ms_fp64 = t[1];
  *ms_conv = t[2];
  return GLS_OK;
}

int gls_set_stream_report(gls_ctx* c, int32_t enable) {
  if (!c) return GLS_ERR_ARG;
  c->srep = enable != 0;
  return GLS_OK;
}

int gls_read_stream_report(gls_ctx* c, gls_stream_report* r) {
  if (!c || !r) return GLS_ERR_ARG;
  DeviceGuard g(c->device);
  int rc = sync_all(c);
  if (rc) return rc;
  memset(r, 0, sizeof *r);
  if (!c->srec.empty()) {
    const cudaEvent_t t0 = c->srec.front().h0;
    auto at = [&](cudaEvent_t e) -> double {  // ms since the first chunk's H2D start
      float ms = 0.f;
      if (!e || !t0 || cudaEventElapsedTime(&ms, t0, e) != cudaSuccess) {
        cudaGetLastError();
        return 0.0;
      }
      return (double)ms;
    };
    double end = 0.0, prev_c1 = 0.0;
    for (size_t j = 0; j < c->srec.size(); ++j) {
      const gls_ctx::ChunkRec& x = c->srec[j];
      const double h0 = at(x.h0), h1 = at(x.h1), c0 = at(x.c0), c1 = at(x.c1);
      r->h2d_ms += h1 - h0;
      r->compute_ms += c1 - c0;
      r->h2d_bytes += x.hbytes;
      r->d2h_bytes += x.dbytes;
      end = std::max(end, c1);
      if (x.d0) {
        const double d1 = at(x.d1);
        r->d2h_ms += d1 - at(x.d0);
        end = std::max(end, d1);
      }
      if (j == 0) {
        // the part of the first load the compute stream waited for: from when it was free (after
        // the work queued before this call, e.g. an asynchronous gls_create) or the copy's start
        r->first_load_ms = std::max(0.0, c0 - std::max(h0, x.cr ? at(x.cr) : h0));
      } else {
        // the compute stream's idle time between chunk j-1 and chunk j: the part before chunk j's
        // data had arrived waited at wait(current X_blk), the rest at wait(previous b_blk)
        const double stall = std::max(0.0, c0 - prev_c1);
        const double on_h2d = std::min(stall, std::max(0.0, h1 - prev_c1));
        r->exposed_h2d_ms += on_h2d;
        r->exposed_other_ms += stall - on_h2d;
      }
      prev_c1 = c1;
    }
    r->tail_ms = std::max(0.0, end - prev_c1);
    r->wall_ms = end;
    r->chunks = (int64_t)c->srec.size();
    for (auto& x : c->srec)
      for (cudaEvent_t e : {x.h0, x.h1, x.c0, x.c1, x.d0, x.d1, x.cr})
        if (e) c->ev_pool.push_back(e);
    c->srec.clear();
  }
  return GLS_OK;
}

int gls_solve_block(gls_ctx* c, const double* X_R, int64_t m_blk, double* b_out) {
  return gls_solve_block_ex(c, X_R, m_blk, b_out, nullptr, 0);
}

int gls_sync(gls_ctx* c) {
  if (!c) return GLS_ERR_ARG;
  DeviceGuard g(c->device);
  return sync_all(c);
}

int gls_set_stream(gls_ctx* c, void* stream) {
  if (!c) return GLS_ERR_ARG;
  cudaStream_t next = stream ? (cudaStream_t)stream : c->own_stream;
  if (next == c->stream) return GLS_OK;
  // work still pending on the old stream uses the context's scratch buffers (x8, cflags, bscratch,
  // staging): order the new stream after it, so reuse on the new stream cannot race with it
  DeviceGuard g(c->device);
  cudaEvent_t e = c->res.ev[11];
  cudaError_t err = cudaEventRecord(e, c->stream);
  if (err == cudaSuccess) err = cudaStreamWaitEvent(next, e, 0);
  if (err != cudaSuccess) return fail_cuda(c, err, "gls_set_stream");
  c->stream = next;
  return GLS_OK;
}

int gls_set_block_cols(gls_ctx* c, int64_t cols) {
  if (!c) return GLS_ERR_ARG;
  if (cols < 1) return GLS_ERR_DIM;
  c->block_cols = cols;
  return GLS_OK;
}

int gls_release_cached_memory(void) {
  int dev = 0;
  cudaMemPool_t pool = nullptr;
  if (cudaGetDevice(&dev) != cudaSuccess || cudaDeviceSynchronize() != cudaSuccess ||
      !(pool = gls_device_pool(dev)) || cudaMemPoolTrimTo(pool, 0) != cudaSuccess) {
    cudaGetLastError();
    return GLS_ERR_CUDA;
  }
  return GLS_OK;
}

void gls_destroy(gls_ctx* c) {
  if (!c) return;
  DeviceGuard g(c->device);
  // every stream that may still read or write context buffers, before the stream-ordered frees
  if (c->h2d) cudaStreamSynchronize(c->h2d);
  if (c->fb) cudaStreamSynchronize(c->fb);
  if (c->stream) cudaStreamSynchronize(c->stream);
  if (c->d2h) cudaStreamSynchronize(c->d2h);
  free_staging(c);
  dfree(c, c->bscratch);
  dfree(c, c->sscratch);
  dfree(c, c->Tpk);
  dfree(c, c->Wpk);
  dfree(c, c->G);
  dfree(c, c->T8);
  dfree(c, c->aux);
  dfree(c, c->V8);
  dfree(c, c->vscale);
  dfree(c, c->x8[0]);
  dfree(c, c->x8[1]);
  dfree(c, c->sws);
  dfree(c, c->flags);
  dfree(c, c->cflags);
  dfree(c, c->pflags);
  dfree(c, c->fb_idx);
  dfree(c, c->fb_X);
  dfree(c, c->fb_b);
  dfree(c, c->fb_s);
  dfree(c, c->ran);
  for (int k = 0; k < 2; ++k) {
    dfree(c, c->stage8[k]);
    dfree(c, c->raw8[k]);
  }
  if (c->own_stream) cudaStreamSynchronize(c->own_stream);
  for (auto& x : c->tl) {
    tev_give(c->device, x.a);
    tev_give(c->device, x.b);
  }
  for (auto e : c->ev_pool) tev_give(c->device, e);
  for (auto& x : c->srec)
    for (cudaEvent_t e : {x.h0, x.h1, x.c0, x.c1, x.d0, x.d1, x.cr}) tev_give(c->device, e);
  status_slot_put(c->hst);
  res_give(c->device, c->res);  // idle streams and events back to the device's cache
  cudaGetLastError();
  delete c;
}

int gls_set_path(gls_ctx* c, int32_t path) {
  if (!c) return GLS_ERR_ARG;
  if (path != GLS_PATH_AUTO && path != GLS_PATH_FP64) return GLS_ERR_ARG;
  if (path == GLS_PATH_FP64 && !c->fp64_ok) return GLS_ERR_STATE;
  c->path = path;
  return GLS_OK;
}

int gls_path_counts(gls_ctx* c, int64_t* int8_launches, int64_t* fp64_launches) {
  if (!c || !int8_launches || !fp64_launches) return GLS_ERR_ARG;
  if (!c->ran) return GLS_ERR_STATE;
  DeviceGuard g(c->device);
  int rc = sync_all(c);
  if (rc) return rc;
  unsigned long long h[2];
  CK(c, cudaMemcpy(h, c->ran, sizeof h, cudaMemcpyDeviceToHost));
  *int8_launches = (int64_t)h[0];
  *fp64_launches = (int64_t)h[1];
  return GLS_OK;
}

int gls_get_dims(const gls_ctx* c, int64_t* n, int32_t* pL, int32_t* pR) {
  if (!c || !n || !pL || !pR) return GLS_ERR_ARG;
  *n = c->n;
  *pL = c->pL;
  *pR = c->pR;
  return GLS_OK;
}

int64_t gls_failed_pivot(const gls_ctx* c) { return c ? c->failed_pivot : -1; }

const char* gls_last_error(const gls_ctx* c) { return c ? c->err.c_str() : ""; }

int64_t gls_kernel_launches(const gls_ctx* c) { return c ? c->launches : 0; }

}  // extern "C"
