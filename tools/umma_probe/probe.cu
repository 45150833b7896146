// Standalone check of the tcgen05 kind::i8 building blocks (descriptors, TMA swizzle, TMEM
// layout) used by csrc/ozaki_gls.cu: one CTA computes D[128 x 224] = A[128 x K] B[224 x K]^T in
// int32 with K = 256 and compares with a CPU product.  Diagnostics only.
#include <cuda.h>
#include <cuda_runtime.h>
#include <cstdio>
#include <cstdlib>
#include <vector>
#include "../../paper_1210_7325_b200/csrc/umma.cuh"
using namespace gls::umma;

constexpr int M = 128, N = 224, K = 256, KC = K / 128;

__global__ void __launch_bounds__(192, 1) probe_kernel(const __grid_constant__ CUtensorMap amap,
                                                       const int8_t* Bpk, int32_t* D) {
  extern __shared__ __align__(1024) uint8_t smem_raw[];
  uint8_t* smem = (uint8_t*)(((uintptr_t)smem_raw + 1023) & ~(uintptr_t)1023);
  uint8_t* sA = smem;                  // KC x 16 KB
  uint8_t* sB = smem + KC * 16384;     // KC x 28 KB
  uint64_t* bars = (uint64_t*)(sB + KC * 28672);
  uint32_t* tbase = (uint32_t*)(bars + 4);
  const int warp = threadIdx.x / 32, lane = threadIdx.x % 32;
  if (threadIdx.x == 0) {
    mbar_init(&bars[0], 1);
    mbar_init(&bars[1], 1);
    fence_barrier_init();
  }
  if (warp == 1) tmem_alloc(tbase, 256);
  tc_fence_before();
  __syncthreads();
  tc_fence_after();
  const uint32_t tm = *tbase;
  if (warp == 0 && lane == 0) {
    mbar_arrive_expect_tx(&bars[0], KC * (16384 + 28672));
    for (int c = 0; c < KC; ++c) {
      for (int q = 0; q < 4; ++q) tma_2d_g2s(sA + c * 16384 + q * 4096, &amap, c * 128, q * 32, &bars[0]);
      bulk_g2s(sB + c * 28672, Bpk + (size_t)c * 28672, 28672, &bars[0]);
    }
  }
  if (warp == 1 && lane == 0) {
    mbar_wait(&bars[0], 0);
    tc_fence_after();
    const uint32_t id = idesc_i8(M, N);
    for (int c = 0; c < KC; ++c)
      for (int kk = 0; kk < 4; ++kk) {
        uint64_t ad = sdesc_k128(smem_u32(sA + c * 16384)) + (uint64_t)(2 * kk);
        uint64_t bd = sdesc_k128(smem_u32(sB + c * 28672)) + (uint64_t)(2 * kk);
        mma_i8(tm, ad, bd, id, (c | kk) != 0);
      }
    mma_commit(&bars[1]);
  }
  if (warp >= 2) {
    mbar_wait(&bars[1], 0);
    tc_fence_after();
    const int q = warp % 4;
    const int row = q * 32 + lane;
    for (int s = 0; s < N / 32; ++s) {
      int32_t v[32];
      tmem_ld32(tm + ((uint32_t)(q * 32) << 16) + s * 32, v);
      tmem_wait_ld();
      for (int j = 0; j < 32; ++j) D[row * N + s * 32 + j] = v[j];
    }
  }
  tc_fence_before();
  __syncthreads();
  if (warp == 1) tmem_dealloc(tm, 256);
}

__global__ void pack_b(const int8_t* B, int8_t* Bpk) {  // B[N][K] row-major -> swizzled tiles
  for (int i = threadIdx.x + blockIdx.x * blockDim.x; i < N * K; i += gridDim.x * blockDim.x) {
    int n = i / K, k = i % K, c = k / 128;
    Bpk[(size_t)c * 28672 + swz128(n, k % 128)] = B[i];
  }
}

typedef CUresult (*PFN_encodeTiled)(CUtensorMap*, CUtensorMapDataType, cuuint32_t, void*,
                                    const cuuint64_t*, const cuuint64_t*, const cuuint32_t*,
                                    const cuuint32_t*, CUtensorMapInterleave, CUtensorMapSwizzle,
                                    CUtensorMapL2promotion, CUtensorMapFloatOOBfill);
int main() {
  std::vector<int8_t> A(M * K), B(N * K);
  srand(1);
  for (auto& a : A) a = (int8_t)(rand() % 256 - 128);
  for (auto& b : B) b = (int8_t)(rand() % 256 - 128);
  int8_t *dA, *dB, *dBpk;
  int32_t* dD;
  cudaMalloc(&dA, M * K); cudaMalloc(&dB, N * K); cudaMalloc(&dBpk, KC * 28672); cudaMalloc(&dD, M * N * 4);
  cudaMemcpy(dA, A.data(), M * K, cudaMemcpyHostToDevice);
  cudaMemcpy(dB, B.data(), N * K, cudaMemcpyHostToDevice);
  pack_b<<<64, 256>>>(dB, dBpk);
  void* p = nullptr; cudaDriverEntryPointQueryResult q;
  cudaGetDriverEntryPoint("cuTensorMapEncodeTiled", &p, cudaEnableDefault, &q);
  CUtensorMap map;
  cuuint64_t gdim[2] = {K, M}; cuuint64_t gstr[1] = {K}; cuuint32_t box[2] = {128, 32}, es[2] = {1, 1};
  CUresult r = ((PFN_encodeTiled)p)(&map, CU_TENSOR_MAP_DATA_TYPE_UINT8, 2, dA, gdim, gstr, box, es,
      CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_128B, CU_TENSOR_MAP_L2_PROMOTION_L2_256B,
      CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
  if (r) { printf("encode failed %d\n", (int)r); return 1; }
  int smem = KC * (16384 + 28672) + 2048;
  cudaFuncSetAttribute(probe_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, smem);
  probe_kernel<<<1, 192, smem>>>(map, dBpk, dD);
  cudaError_t e = cudaDeviceSynchronize();
  if (e) { printf("kernel error %s\n", cudaGetErrorString(e)); return 1; }
  std::vector<int32_t> D(M * N);
  cudaMemcpy(D.data(), dD, M * N * 4, cudaMemcpyDeviceToHost);
  long bad = 0;
  for (int i = 0; i < M; ++i)
    for (int j = 0; j < N; ++j) {
      int32_t ref = 0;
      for (int k = 0; k < K; ++k) ref += (int32_t)A[i * K + k] * B[j * K + k];
      if (ref != D[i * N + j]) { if (bad < 5) printf("mismatch D[%d][%d] = %d ref %d\n", i, j, D[i * N + j], ref); ++bad; }
    }
  printf("umma i8 probe: %ld mismatches of %d\n", bad, M * N);
  return bad != 0;
}
