// Diagnostics: throughput of the setup GEMM (csrc/dgemm.cu) at the shapes of the top levels of the
// recursive Cholesky + inverse at n = 1e4.
#include <cstdio>
#include <cuda_runtime.h>
#include "../../paper_1210_7325_b200/csrc/gls_internal.cuh"
using namespace gls;
int main() {
  const int64_t n = 10000, h = 5024, h2 = n - h;
  double *A, *B, *C;
  cudaMalloc(&A, n * n * 8); cudaMalloc(&B, n * n * 8); cudaMalloc(&C, n * n * 8);
  cudaMemset(A, 0, n * n * 8); cudaMemset(B, 0, n * n * 8); cudaMemset(C, 0, n * n * 8);
  cudaEvent_t e0, e1; cudaEventCreate(&e0); cudaEventCreate(&e1);
  struct Case { const char* name; int64_t M, N, K; char ta, tb; int flags; double flops; };
  Case cs[] = {
    {"L21=A21 T11^T (KMAX_COL)", h2, h, h, 'N', 'T', GEMM_KMAX_COL, (double)h2 * h * h},
    {"A22-=L21 L21^T (LOWER_C)", h2, h2, h, 'N', 'T', GEMM_LOWER_C, (double)h2 * h2 * h},
    {"Y=L21 T11 (KMIN_COL)", h2, h, h, 'N', 'N', GEMM_KMIN_COL, (double)h2 * h * h},
    {"T21=-T22 Y (KMAX_ROW)", h2, h, h2, 'N', 'N', GEMM_KMAX_ROW, (double)h2 * h * h2},
    {"dense NN 4096^3", 4096, 4096, 4096, 'N', 'N', 0, 2.0 * 4096.0 * 4096 * 4096},
    {"dense NT 4096^3", 4096, 4096, 4096, 'N', 'T', 0, 2.0 * 4096.0 * 4096 * 4096},
    {"dense NN 1250^3", 1250, 1250, 1250, 'N', 'N', 0, 2.0 * 1250.0 * 1250 * 1250},
    {"dense NN 312^3", 312, 312, 312, 'N', 'N', 0, 2.0 * 312.0 * 312 * 312},
  };
  for (auto& c : cs) {
    for (int r = 0; r < 2; ++r) dgemm(0, c.M, c.N, c.K, 1.0, A, n, c.ta, B, n, c.tb, 0.0, C, n, c.flags, nullptr);
    cudaEventRecord(e0);
    const int reps = 5;
    for (int r = 0; r < reps; ++r) dgemm(0, c.M, c.N, c.K, 1.0, A, n, c.ta, B, n, c.tb, 0.0, C, n, c.flags, nullptr);
    cudaEventRecord(e1); cudaEventSynchronize(e1);
    float ms; cudaEventElapsedTime(&ms, e0, e1);
    printf("%-28s M=%5lld N=%5lld K=%5lld  %8.3f ms  %6.2f TF/s (useful flops)\n", c.name, (long long)c.M,
           (long long)c.N, (long long)c.K, ms / reps, c.flops / (ms / reps * 1e-3) / 1e12);
  }
  printf("err: %s\n", cudaGetErrorString(cudaDeviceSynchronize()));
}
