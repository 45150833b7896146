// Diagnostics: chol_inv_leaf128 (csrc/chol_inv.cu, the blocked 128-row leaf) and the round-1 128-row node
// (chol_inv_node128) on one random SPD block: max error of L and T = L^{-1} against a CPU Cholesky +
// inverse in double, time per launch, and (GLS_LEAF_PROF) clock64 cycles per phase of the new leaf.
// Build: nvcc -gencode arch=compute_100a,code=sm_100a -O3 -std=c++17 -I include \
//        tools/leaf_probe/leaf_probe.cu paper_1210_7325_b200/csrc/dgemm.cu -lcuda -o tools/leaf_probe/leaf_probe
#define GLS_LEAF_PROF 1
#include "../../paper_1210_7325_b200/csrc/chol_inv.cu"

#include <cmath>
#include <cstdio>
#include <mutex>
#include <set>
#include <utility>

namespace gls {
bool first_use_on_device(const void* key) {
  static std::mutex mu;
  static std::set<std::pair<const void*, int>> seen;
  int dev = 0;
  cudaGetDevice(&dev);
  std::lock_guard<std::mutex> g(mu);
  return seen.insert({key, dev}).second;
}
cudaError_t gls_pool_alloc(void** p, size_t bytes, int, cudaStream_t s) { return cudaMallocAsync(p, bytes, s); }
}  // namespace gls

using namespace gls;

static void cpu_chol_inv(int n, const std::vector<double>& A, std::vector<double>& L, std::vector<double>& T) {
  L.assign((size_t)n * n, 0.0);
  T.assign((size_t)n * n, 0.0);
  for (int j = 0; j < n; ++j) {
    double d = A[j + (size_t)j * n];
    for (int k = 0; k < j; ++k) d -= L[j + (size_t)k * n] * L[j + (size_t)k * n];
    const double ljj = std::sqrt(d);
    L[j + (size_t)j * n] = ljj;
    for (int i = j + 1; i < n; ++i) {
      double s = A[i + (size_t)j * n];
      for (int k = 0; k < j; ++k) s -= L[i + (size_t)k * n] * L[j + (size_t)k * n];
      L[i + (size_t)j * n] = s / ljj;
    }
  }
  for (int c = 0; c < n; ++c) {  // forward substitution L t = e_c
    for (int i = c; i < n; ++i) {
      double s = (i == c) ? 1.0 : 0.0;
      for (int k = c; k < i; ++k) s -= L[i + (size_t)k * n] * T[k + (size_t)c * n];
      T[i + (size_t)c * n] = s / L[i + (size_t)i * n];
    }
  }
}

int main() {
  const int ld = 160;
  for (int nb : {128, 100, 77, 16, 5}) {
    std::vector<double> A((size_t)ld * ld, 0.0), Z((size_t)nb * nb);
    srand(7 + nb);
    for (auto& z : Z) z = (double)rand() / RAND_MAX - 0.5;
    for (int i = 0; i < nb; ++i)
      for (int j = 0; j < nb; ++j) {
        double s = (i == j) ? 1.0 : 0.0;
        for (int k = 0; k < nb; ++k) s += Z[i + (size_t)k * nb] * Z[j + (size_t)k * nb] / nb;
        A[i + (size_t)j * ld] = s;
      }
    std::vector<double> Ac((size_t)nb * nb);
    for (int j = 0; j < nb; ++j)
      for (int i = 0; i < nb; ++i) Ac[i + (size_t)j * nb] = A[i + (size_t)j * ld];
    std::vector<double> Lr, Tr;
    cpu_chol_inv(nb, Ac, Lr, Tr);
    double *dA, *dA0, *dT;
    CholStatus* st;
    cudaMalloc(&dA, A.size() * 8);
    cudaMalloc(&dA0, A.size() * 8);
    cudaMalloc(&dT, A.size() * 8);
    cudaMalloc(&st, sizeof(CholStatus));
    cudaMemcpy(dA0, A.data(), A.size() * 8, cudaMemcpyHostToDevice);
    cudaFuncSetAttribute(chol_inv_leaf128, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)blk::SMEM);
    cudaFuncSetAttribute(chol_inv_node128, cudaFuncAttributeMaxDynamicSharedMemorySize,
                         (int)(6 * LEAF * LLD * sizeof(double)));
    for (int which = 0; which < 2; ++which) {
      if (which == 1 && (nb <= 64)) continue;
      cudaEvent_t e0, e1;
      cudaEventCreate(&e0);
      cudaEventCreate(&e1);
      unsigned long long zero[8] = {};
      float best = 1e9f;
      for (int it = 0; it < 21; ++it) {
        cudaMemcpy(dA, dA0, A.size() * 8, cudaMemcpyDeviceToDevice);
        maxdiag_kernel<<<1, 256>>>(nb, dA, ld, st);
        if (it == 1) cudaMemcpyToSymbol(g_leaf_prof, zero, sizeof(zero));
        cudaEventRecord(e0);
        if (which == 0) chol_inv_leaf128<<<1, blk::THREADS, blk::SMEM>>>(nb, dA, dT, ld, 0, st);
        else chol_inv_node128<<<1, LEAF_THREADS, 6 * LEAF * LLD * sizeof(double)>>>(nb, dA, dT, ld, 0, st);
        cudaEventRecord(e1);
        cudaEventSynchronize(e1);
        float ms = 0.f;
        cudaEventElapsedTime(&ms, e0, e1);
        if (it > 0 && ms < best) best = ms;
      }
      cudaError_t err = cudaDeviceSynchronize();
      std::vector<double> Lg(A.size()), Tg(A.size());
      cudaMemcpy(Lg.data(), dA, A.size() * 8, cudaMemcpyDeviceToHost);
      cudaMemcpy(Tg.data(), dT, A.size() * 8, cudaMemcpyDeviceToHost);
      CholStatus hs;
      cudaMemcpy(&hs, st, sizeof(hs), cudaMemcpyDeviceToHost);
      double eL = 0, eT = 0, mT = 0;
      for (int j = 0; j < nb; ++j)
        for (int i = j; i < nb; ++i) {
          eL = fmax(eL, fabs(Lg[i + (size_t)j * ld] - Lr[i + (size_t)j * nb]));
          eT = fmax(eT, fabs(Tg[i + (size_t)j * ld] - Tr[i + (size_t)j * nb]));
          mT = fmax(mT, fabs(Tr[i + (size_t)j * nb]));
        }
      if (eT > 1e-12) {  // where: the worst 16 x 16 block of T
        for (int bj = 0; bj * 16 < nb; ++bj)
          for (int bi = bj; bi * 16 < nb; ++bi) {
            double e = 0;
            for (int j = bj * 16; j < std::min(nb, bj * 16 + 16); ++j)
              for (int i = std::max(j, bi * 16); i < std::min(nb, bi * 16 + 16); ++i)
                e = fmax(e, fabs(Tg[i + (size_t)j * ld] - Tr[i + (size_t)j * nb]));
            if (e > 1e-12) printf("   T block (%d,%d) err %.2e\n", bi, bj, e);
          }
      }
      double upper = 0;
      for (int j = 0; j < nb; ++j)
        for (int i = 0; i < j; ++i) upper = fmax(upper, fabs(Tg[i + (size_t)j * ld]));
      printf("%s nb=%3d: %7.2f us  max|dL| %.2e  max|dT| %.2e (max|T| %.2f)  T upper %.1e  fail=%llx  %s\n",
             which == 0 ? "leaf128" : "node128", nb, best * 1e3, eL, eT, mT, upper, (unsigned long long)hs.fail,
             cudaGetErrorString(err));
      if (which == 0) {
        unsigned long long pr[8];
        cudaMemcpyFromSymbol(pr, g_leaf_prof, sizeof(pr));
        printf("   cycles per launch: load %llu  diag16 %llu  panel %llu  trailing+T %llu  writeback %llu"
               "  | per diag16: chol %llu  inverse %llu\n",
               pr[0] / 20, pr[1] / 20, pr[2] / 20, pr[3] / 20, pr[4] / 20, pr[5] / 20 / ((nb + 15) / 16),
               pr[6] / 20 / ((nb + 15) / 16));
      }
    }
  }
  return 0;
}
