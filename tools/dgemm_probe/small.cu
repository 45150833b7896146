// Diagnostics: the small-product path of dgemm() (dgemm_small_kernel, 32 x 32 tiles) against a naive
// GPU GEMM, and the latency of dgemm() at the shapes of the recursion's deep levels.  Run twice, with
// GLS_DGEMM_SMALL=0 (128 x 64 tiles + split-K) and =1.
#include <cstdio>
#include <cstdlib>
#include <cmath>
#include <vector>
#include <cuda_runtime.h>
#include "../../paper_1210_7325_b200/csrc/gls_internal.cuh"
using namespace gls;
__global__ void naive(int64_t M, int64_t N, int64_t K, double alpha, const double* A, int64_t lda, const double* B,
                      int64_t ldb, char tb, double beta, double* C, int64_t ldc) {
  int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
  if (i >= M * N) return;
  int64_t m = i % M, n = i / M;
  double s = 0;
  for (int64_t k = 0; k < K; ++k) s += A[m + k * lda] * (tb == 'T' ? B[n + k * ldb] : B[k + n * ldb]);
  C[m + n * ldc] = alpha * s + beta * C[m + n * ldc];
}
int main() {
  const int64_t L = 2000;
  std::vector<double> h(L * L);
  srand(3);
  for (auto& x : h) x = (double)rand() / RAND_MAX - 0.5;
  double *A, *B, *C0, *C1, *ws;
  cudaMalloc(&A, L * L * 8); cudaMalloc(&B, L * L * 8); cudaMalloc(&C0, L * L * 8); cudaMalloc(&C1, L * L * 8);
  cudaMalloc(&ws, kSplitKWsDoubles * 8);
  cudaMemcpy(A, h.data(), L * L * 8, cudaMemcpyHostToDevice);
  for (auto& x : h) x = (double)rand() / RAND_MAX - 0.5;
  cudaMemcpy(B, h.data(), L * L * 8, cudaMemcpyHostToDevice);
  struct Case { int64_t M, N, K; char tb; double beta; int flags; };
  Case cs[] = {{128, 128, 128, 'T', 0, 0}, {128, 128, 128, 'N', 1, 0}, {100, 77, 333, 'T', 1, 0}, {100, 77, 333, 'N', 0, 0},
               {256, 256, 256, 'T', 0, 0}, {384, 768, 768, 'T', 0, GEMM_KMAX_COL}, {384, 384, 768, 'T', 1, GEMM_LOWER_C},
               {384, 768, 768, 'N', 0, GEMM_KMIN_COL}, {610, 640, 640, 'T', 0, GEMM_KMAX_COL},
               {610, 610, 640, 'T', 1, GEMM_LOWER_C}, {610, 640, 610, 'N', 0, GEMM_KMAX_ROW}, {1000, 500, 1000, 'N', 0, 0}};
  cudaEvent_t e0, e1; cudaEventCreate(&e0); cudaEventCreate(&e1);
  for (auto& c : cs) {
    cudaMemcpy(C0, h.data(), L * L * 8, cudaMemcpyHostToDevice);
    cudaMemcpy(C1, h.data(), L * L * 8, cudaMemcpyHostToDevice);
    // correctness with dense operands and flags = 0 (the flags assume triangular operands)
    naive<<<(unsigned)((c.M * c.N + 255) / 256), 256>>>(c.M, c.N, c.K, 1.5, A, L, B, L, c.tb, c.beta, C0, L);
    dgemm(0, c.M, c.N, c.K, 1.5, A, L, 'N', B, L, c.tb, c.beta, C1, L, 0, nullptr, ws);
    cudaDeviceSynchronize();
    double mx = 0, ref = 0;
    std::vector<double> r0(c.M), r1(c.M);
    for (int64_t n = 0; n < c.N; ++n) {
      cudaMemcpy(r0.data(), C0 + n * L, c.M * 8, cudaMemcpyDeviceToHost);
      cudaMemcpy(r1.data(), C1 + n * L, c.M * 8, cudaMemcpyDeviceToHost);
      for (int64_t m = 0; m < c.M; ++m) { mx = fmax(mx, fabs(r0[m] - r1[m])); ref = fmax(ref, fabs(r0[m])); }
    }
    for (int r = 0; r < 3; ++r) dgemm(0, c.M, c.N, c.K, 1.0, A, L, 'N', B, L, c.tb, 0.0, C1, L, c.flags, nullptr, ws);
    const int reps = 20;
    cudaEventRecord(e0);
    for (int r = 0; r < reps; ++r) dgemm(0, c.M, c.N, c.K, 1.0, A, L, 'N', B, L, c.tb, 0.0, C1, L, c.flags, nullptr, ws);
    cudaEventRecord(e1);
    cudaEventSynchronize(e1);
    float ms; cudaEventElapsedTime(&ms, e0, e1);
    printf("M=%5lld N=%5lld K=%5lld N%c beta=%g flags=%d  max|err|/max|C| = %.2e  %7.2f us  %s\n", (long long)c.M,
           (long long)c.N, (long long)c.K, c.tb, c.beta, c.flags, mx / ref, 1e3 * ms / reps,
           cudaGetErrorString(cudaGetLastError()));
  }
  return 0;
}
