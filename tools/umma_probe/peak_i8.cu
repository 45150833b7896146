// Dense tcgen05 kind::i8 throughput microbenchmark (the denominator of bench.py's int8 roofline).
//
// One CTA pair per TPC (74 clusters of 2 on a 148-SM B200), 1 CTA per SM.  Each CTA holds a
// 128 x 128-byte A tile and an N/2 x 128-byte B half-tile in shared memory (128B swizzle, filled
// with pseudo-random bytes so the datapath toggles as with real digits), and the pair leader issues
// back-to-back tcgen05.mma.cta_group::2.kind::i8 (M = 256, N, K = 32), four per K = 128 chunk,
// alternating between two TMEM accumulators, with a commit + wait every `batch` chunks so the
// issue queue never overflows.  No global-memory traffic in the timed loop: this is the tensor
// pipe's rate at the clock the part sustains under that load.
//
//   burst:     one launch of ~20 ms (after a warm-up launch), CUDA events
//   sustained: back-to-back launches for 4 s, total ops / total event time
// Ops = 2 * 256 * N * 32 per MMA.  Output: one JSON line.
//
//   nvcc -gencode arch=compute_100a,code=sm_100a -O3 -std=c++17 -o peak_i8 peak_i8.cu -lcuda
#include <cuda.h>
#include <cuda_runtime.h>

#include <cstdio>
#include <cstdlib>

#include "../../paper_1210_7325_b200/csrc/umma.cuh"
using namespace gls::umma;

#define CK(x)                                                                              \
  do {                                                                                     \
    cudaError_t e = (x);                                                                   \
    if (e != cudaSuccess) {                                                                \
      printf("{\"error\": \"%s at %d: %s\"}\n", #x, __LINE__, cudaGetErrorString(e));      \
      exit(1);                                                                             \
    }                                                                                      \
  } while (0)

template <int N>
__global__ void __cluster_dims__(2, 1, 1) __launch_bounds__(128, 1) peak_kernel(long long chunks, int batch,
                                                                              int* sink) {
  extern __shared__ __align__(1024) uint8_t smem_raw[];
  uint8_t* smem = (uint8_t*)(((uintptr_t)smem_raw + 1023) & ~(uintptr_t)1023);
  uint8_t* sA = smem;                 // 128 rows x 128 bytes
  uint8_t* sB = smem + 128 * 128;     // N/2 rows x 128 bytes
  uint64_t* bar = (uint64_t*)(sB + (N / 2) * 128);
  uint32_t* tbase = (uint32_t*)(bar + 2);  // bar[0], bar[1]
  const int warp = threadIdx.x / 32;
  const uint32_t rank = cluster_ctarank();
  // pseudo-random operand bytes (a hash of the position): realistic toggling of the datapath
  for (int i = threadIdx.x; i < (128 + N / 2) * 128 / 4; i += blockDim.x) {
    uint32_t h = (uint32_t)i * 2654435761u ^ (rank * 40503u + blockIdx.x * 97u);
    h ^= h >> 13;
    h *= 0x5bd1e995u;
    h ^= h >> 15;
    ((uint32_t*)smem)[i] = h;
  }
  fence_proxy_async();
  if (threadIdx.x == 0) {
    mbar_init(&bar[0], 1);
    mbar_init(&bar[1], 1);
    fence_barrier_init();
  }
  if (warp == 1) tmem_alloc_pair(tbase, 512);
  tc_fence_before();
  __syncthreads();
  cluster_sync_all();
  tc_fence_after();
  const uint32_t tm = *tbase;
  const long long nbatch = (chunks + batch - 1) / batch;
  if (rank == 0 && threadIdx.x == 0) {
    // batch b commits to bar[b & 1]; the issuer then waits for batch b - 1, so one batch of MMAs is
    // always queued behind the one executing (no drain bubble)
    constexpr uint32_t idesc = idesc_i8(256, N);
    for (long long b = 0; b < nbatch; ++b) {
      const long long c1 = (b + 1) * batch < chunks ? (b + 1) * batch : chunks;
      for (long long c = b * batch; c < c1; ++c) {
        const uint32_t d = tm + (uint32_t)(c & 1) * 256;
#pragma unroll
        for (int k = 0; k < 4; ++k)
          mma_i8_pair(d, sdesc_k128(smem_u32(sA) + 32 * k), sdesc_k128(smem_u32(sB) + 32 * k), idesc,
                      (c > 1 || k > 0) ? 1u : 0u);
      }
      mma_commit_pair_mc(&bar[b & 1], 0x3);
      if (b >= 1) mbar_wait(&bar[(b - 1) & 1], (uint32_t)(((b - 1) >> 1) & 1));
    }
    mbar_wait(&bar[(nbatch - 1) & 1], (uint32_t)(((nbatch - 1) >> 1) & 1));
  } else if (rank == 1 && threadIdx.x == 0) {
    // the peer's barriers receive the multicast commits: consume them so the phases stay in step
    for (long long b = 0; b < nbatch; ++b) mbar_wait(&bar[b & 1], (uint32_t)((b >> 1) & 1));
  }
  tc_fence_before();
  __syncthreads();
  cluster_sync_all();
  tc_fence_after();
  if (threadIdx.x < 32 && warp == 0) {
    int32_t v[8];
    tmem_ld8(tm, v);
    tmem_wait_ld();
    if (v[0] == 0x7fffffff) sink[0] = v[1];  // keep the accumulators live
  }
  tc_fence_before();
  __syncthreads();
  cluster_sync_all();
  if (warp == 1) tmem_dealloc_pair(tm, 512);
}

template <int N>
void run(int sms) {
  // 128 KB (more than the operands need) so that exactly one CTA -- one 512-column TMEM owner -- fits per SM
  const size_t smem = 128 * 1024;
  CK(cudaFuncSetAttribute(peak_kernel<N>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem));
  int* sink;
  CK(cudaMalloc(&sink, 4));
  const int grid = (sms / 2) * 2;
  const double ops_per_chunk = 4.0 * 2.0 * 256.0 * N * 32.0 * (grid / 2);
  cudaEvent_t e0, e1;
  CK(cudaEventCreate(&e0));
  CK(cudaEventCreate(&e1));
  // calibrate: ~20 ms per launch
  long long chunks = 20000;
  peak_kernel<N><<<grid, 128, smem>>>(chunks, 8, sink);
  CK(cudaDeviceSynchronize());
  CK(cudaEventRecord(e0));
  peak_kernel<N><<<grid, 128, smem>>>(chunks, 8, sink);
  CK(cudaEventRecord(e1));
  CK(cudaEventSynchronize(e1));
  float ms = 0;
  CK(cudaEventElapsedTime(&ms, e0, e1));
  chunks = (long long)(chunks * 20.0 / ms);
  CK(cudaEventRecord(e0));
  peak_kernel<N><<<grid, 128, smem>>>(chunks, 8, sink);
  CK(cudaEventRecord(e1));
  CK(cudaEventSynchronize(e1));
  CK(cudaEventElapsedTime(&ms, e0, e1));
  const double burst = ops_per_chunk * chunks / (ms * 1e-3) / 1e12;
  // sustained: back-to-back launches for ~4 s
  const int launches = (int)(4000.0 / ms) + 1;
  CK(cudaEventRecord(e0));
  for (int i = 0; i < launches; ++i) peak_kernel<N><<<grid, 128, smem>>>(chunks, 8, sink);
  CK(cudaEventRecord(e1));
  CK(cudaEventSynchronize(e1));
  float ms_s = 0;
  CK(cudaEventElapsedTime(&ms_s, e0, e1));
  const double sustained = ops_per_chunk * chunks * launches / (ms_s * 1e-3) / 1e12;
  printf("{\"probe\": \"tcgen05.mma.cta_group::2.kind::i8 dense\", \"M\": 256, \"N\": %d, \"K\": 32, "
         "\"ctas\": %d, \"burst_tops\": %.1f, \"burst_ms\": %.2f, \"sustained_tops\": %.1f, "
         "\"sustained_s\": %.2f}\n",
         N, grid, burst, ms, sustained, ms_s * 1e-3);
  CK(cudaFree(sink));
}

int main() {
  int dev = 0, sms = 0;
  CK(cudaGetDevice(&dev));
  CK(cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev));
  run<256>(sms);
  run<224>(sms);
  return 0;
}
