// Diagnostics: correctness of dgemm() (csrc/dgemm.cu, both its kernels) against a naive FP64 GPU GEMM on
// random operands, for the shapes / transposes / triangular flags gls_create uses, incl. ragged edges and
// more tiles than SMs; prints the max relative error per case and the time.
#include <cstdio>
#include <cstdlib>
#include <cmath>
#include <vector>
#include <cuda_runtime.h>
#include "../../paper_1210_7325_b200/csrc/gls_internal.cuh"
using namespace gls;

__global__ void naive(int64_t M, int64_t N, int64_t K, double alpha, const double* A, int64_t lda, char ta,
                      const double* B, int64_t ldb, char tb, double beta, double* C, int64_t ldc) {
  int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
  if (i >= M * N) return;
  int64_t m = i % M, n = i / M;
  double s = 0;
  for (int64_t k = 0; k < K; ++k) {
    double a = ta == 'T' ? A[k + m * lda] : A[m + k * lda];
    double b = tb == 'T' ? B[n + k * ldb] : B[k + n * ldb];
    s += a * b;
  }
  C[m + n * ldc] = alpha * s + beta * C[m + n * ldc];
}

int main() {
  const int64_t L = 6000;
  std::vector<double> h(L * L);
  srand(1);
  for (auto& x : h) x = (double)rand() / RAND_MAX - 0.5;
  double *A, *B, *C0, *C1;
  cudaMalloc(&A, L * L * 8); cudaMalloc(&B, L * L * 8); cudaMalloc(&C0, L * L * 8); cudaMalloc(&C1, L * L * 8);
  cudaMemcpy(A, h.data(), L * L * 8, cudaMemcpyHostToDevice);
  for (auto& x : h) x = (double)rand() / RAND_MAX - 0.5;
  cudaMemcpy(B, h.data(), L * L * 8, cudaMemcpyHostToDevice);
  struct Case { int64_t M, N, K; char ta, tb; double beta; int cap; };
  Case cs[] = {{128, 64, 300, 'N', 'T', 0, 0}, {128, 64, 300, 'N', 'N', 0, 0}, {1000, 700, 300, 'N', 'N', 0, 0},
               {1000, 700, 300, 'N', 'T', 1, 0}, {3000, 2900, 1500, 'N', 'N', 0, 0}, {3000, 2900, 1500, 'N', 'T', 0, 0},
               {2001, 1999, 777, 'N', 'N', 1, 264}, {2001, 1999, 777, 'N', 'T', 0, 264}, {5000, 5000, 5000, 'N', 'T', 0, 0},
               {5000, 5000, 5000, 'N', 'N', 0, 0}, {4976, 5024, 5024, 'N', 'T', 0, 0}, {4976, 5024, 4976, 'N', 'N', 1, 0}};
  cudaEvent_t e0, e1; cudaEventCreate(&e0); cudaEventCreate(&e1);
  for (auto& c : cs) {
    cudaMemcpy(C0, h.data(), L * L * 8, cudaMemcpyHostToDevice);
    cudaMemcpy(C1, h.data(), L * L * 8, cudaMemcpyHostToDevice);
    const int64_t lda = L, ldb = L, ldc = L;
    naive<<<(unsigned)((c.M * c.N + 255) / 256), 256>>>(c.M, c.N, c.K, 1.5, A, lda, c.ta, B, ldb, c.tb, c.beta, C0, ldc);
    cudaEventRecord(e0);
    dgemm(0, c.M, c.N, c.K, 1.5, A, lda, c.ta, B, ldb, c.tb, c.beta, C1, ldc, 0, nullptr, nullptr, c.cap);
    cudaEventRecord(e1);
    cudaDeviceSynchronize();
    float ms; cudaEventElapsedTime(&ms, e0, e1);
    std::vector<double> r0(c.M), r1(c.M);
    double mx = 0, ref = 0;
    for (int64_t n = 0; n < c.N; n += 1) {
      cudaMemcpy(r0.data(), C0 + n * ldc, c.M * 8, cudaMemcpyDeviceToHost);
      cudaMemcpy(r1.data(), C1 + n * ldc, c.M * 8, cudaMemcpyDeviceToHost);
      for (int64_t m = 0; m < c.M; ++m) { mx = fmax(mx, fabs(r0[m] - r1[m])); ref = fmax(ref, fabs(r0[m])); }
      if (c.N > 1000) n += 37;
    }
    printf("M=%5lld N=%5lld K=%5lld %c%c beta=%g cap=%d  max|err|/max|C| = %.3e  %.3f ms  %.2f TF/s  %s\n",
           (long long)c.M, (long long)c.N, (long long)c.K, c.ta, c.tb, c.beta, c.cap, mx / ref, ms,
           2.0 * c.M * c.N * c.K / (ms * 1e-3) / 1e12, cudaGetErrorString(cudaGetLastError()));
  }
}
