// Check of the CTA-pair (cta_group::2) kind::i8 MMA used by the int8 hot kernel: a cluster of 2
// CTAs computes D[256 x 224] = A[256 x K] B[224 x K]^T (K = 256), CTA r holding A rows
// [128r, 128r+128) and B rows [112r, 112r+112), and each CTA reads its 128 rows of D from TMEM.
#include <cuda.h>
#include <cuda_runtime.h>
#include <cstdio>
#include <cstdlib>
#include <vector>
#include "../../paper_1210_7325_b200/csrc/umma.cuh"
using namespace gls::umma;

constexpr int M = 256, N = 224, K = 256, KC = K / 128, BH = N / 2;
constexpr int ATILE = 128 * 128, BTILE = BH * 128;

__global__ void __cluster_dims__(2, 1, 1) __launch_bounds__(192, 1)
    probe2_kernel(const __grid_constant__ CUtensorMap amap, const __grid_constant__ CUtensorMap bmap, int32_t* D) {
  extern __shared__ __align__(1024) uint8_t smem_raw[];
  uint8_t* smem = (uint8_t*)(((uintptr_t)smem_raw + 1023) & ~(uintptr_t)1023);
  uint8_t* sA = smem;
  uint8_t* sB = smem + KC * ATILE;
  uint64_t* bars = (uint64_t*)(sB + KC * BTILE);
  uint32_t* tbase = (uint32_t*)(bars + 4);
  const int warp = threadIdx.x / 32, lane = threadIdx.x % 32;
  const uint32_t rank = cluster_ctarank();
  if (threadIdx.x == 0) {
    mbar_init(&bars[0], 1);  // full (leader's is used)
    mbar_init(&bars[1], 1);  // tmem full (both)
    fence_barrier_init();
  }
  if (warp == 1) tmem_alloc_pair(tbase, 256);
  tc_fence_before();
  __syncthreads();
  cluster_sync_all();
  tc_fence_after();
  const uint32_t tm = *tbase;
  const uint32_t full_leader = mapa_shared(smem_u32(&bars[0]), 0);
  if (warp == 0 && lane == 0) {
    if (rank == 0) mbar_arrive_expect_tx(&bars[0], 2 * KC * (ATILE + BTILE));
    for (int c = 0; c < KC; ++c) {
      for (int q = 0; q < 4; ++q)
        tma_2d_g2s_pair(sA + c * ATILE + q * 4096, &amap, c * 128, rank * 128 + q * 32, full_leader);
      tma_2d_g2s_pair(sB + c * BTILE, &bmap, c * 128, rank * BH, full_leader);
    }
  }
  if (rank == 0 && warp == 1 && lane == 0) {
    mbar_wait(&bars[0], 0);
    tc_fence_after();
    const uint32_t id = idesc_i8(M, N);
    for (int c = 0; c < KC; ++c)
      for (int kk = 0; kk < 4; ++kk) {
        uint64_t ad = sdesc_k128(smem_u32(sA + c * ATILE)) + (uint64_t)(2 * kk);
        uint64_t bd = sdesc_k128(smem_u32(sB + c * BTILE)) + (uint64_t)(2 * kk);
        mma_i8_pair(tm, ad, bd, id, (c | kk) != 0);
      }
    mma_commit_pair_mc(&bars[1], 3);
  }
  if (warp >= 2) {
    mbar_wait(&bars[1], 0);
    tc_fence_after();
    const int q = warp % 4;
    const int row = rank * 128 + q * 32 + lane;
    for (int s = 0; s < N / 32; ++s) {
      int32_t v[32];
      tmem_ld32(tm + ((uint32_t)(q * 32) << 16) + s * 32, v);
      tmem_wait_ld();
      for (int j = 0; j < 32; ++j) D[row * N + s * 32 + j] = v[j];
    }
  }
  tc_fence_before();
  __syncthreads();
  cluster_sync_all();
  if (warp == 1) tmem_dealloc_pair(tm, 256);
}

typedef CUresult (*PFN_encodeTiled)(CUtensorMap*, CUtensorMapDataType, cuuint32_t, void*,
                                    const cuuint64_t*, const cuuint64_t*, const cuuint32_t*,
                                    const cuuint32_t*, CUtensorMapInterleave, CUtensorMapSwizzle,
                                    CUtensorMapL2promotion, CUtensorMapFloatOOBfill);
int main() {
  std::vector<int8_t> A(M * K), B(N * K);
  srand(2);
  for (auto& a : A) a = (int8_t)(rand() % 256 - 128);
  for (auto& b : B) b = (int8_t)(rand() % 256 - 128);
  int8_t *dA, *dB;
  int32_t* dD;
  cudaMalloc(&dA, M * K); cudaMalloc(&dB, N * K); cudaMalloc(&dD, M * N * 4);
  cudaMemset(dD, 0xff, M * N * 4);
  cudaMemcpy(dA, A.data(), M * K, cudaMemcpyHostToDevice);
  cudaMemcpy(dB, B.data(), N * K, cudaMemcpyHostToDevice);
  void* p = nullptr; cudaDriverEntryPointQueryResult q;
  cudaGetDriverEntryPoint("cuTensorMapEncodeTiled", &p, cudaEnableDefault, &q);
  auto enc = (PFN_encodeTiled)p;
  CUtensorMap amap, bmap;
  cuuint64_t gA[2] = {K, M}, gB[2] = {K, N}, st[1] = {K};
  cuuint32_t boxA[2] = {128, 32}, boxB[2] = {128, BH}, es[2] = {1, 1};
  CUresult r1 = enc(&amap, CU_TENSOR_MAP_DATA_TYPE_UINT8, 2, dA, gA, st, boxA, es, CU_TENSOR_MAP_INTERLEAVE_NONE,
      CU_TENSOR_MAP_SWIZZLE_128B, CU_TENSOR_MAP_L2_PROMOTION_L2_256B, CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
  CUresult r2 = enc(&bmap, CU_TENSOR_MAP_DATA_TYPE_UINT8, 2, dB, gB, st, boxB, es, CU_TENSOR_MAP_INTERLEAVE_NONE,
      CU_TENSOR_MAP_SWIZZLE_128B, CU_TENSOR_MAP_L2_PROMOTION_L2_256B, CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
  if (r1 || r2) { printf("encode failed %d %d\n", (int)r1, (int)r2); return 1; }
  int smem = KC * (ATILE + BTILE) + 2048;
  cudaFuncSetAttribute(probe2_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, smem);
  probe2_kernel<<<2, 192, smem>>>(amap, bmap, dD);
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
  printf("umma i8 pair probe: %ld mismatches of %d\n", bad, M * N);
  return bad != 0;
}
