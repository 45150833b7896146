// gen_device.cu -- device-side genotype generator for synthetic X_R (bench / test input only;
// built into its own library libglsgen_dev.so, not part of libgls.so's solve path).
//
// Implements, independently of gen/glsgen.c, the same counter-based Philox4x32-10 draw:
//   key = seed, counter = (c lo, c hi, r, stream)
//   q_c      = 0.05 + 0.45 * (u + 0.5) 2^-32           (stream 5, word 0; product and sum rounded
//                                                        separately -- no FMA contraction)
//   g(c, r)  = [(u_a + 0.5) 2^-32 < q_c] + [(u_b + 0.5) 2^-32 < q_c]   (stream 6, words 0 and 1)
// Genotypes are small integers, so the GPU and CPU generators agree bit for bit
// (tests/test_gpu_parity.py::test_device_generator_matches_cpu).
#include <cuda_runtime.h>
#include <stdint.h>

namespace {

__device__ __forceinline__ void philox(uint32_t c0, uint32_t c1, uint32_t c2, uint32_t c3,
                                       uint64_t seed, uint32_t& o0, uint32_t& o1) {
  uint32_t k0 = (uint32_t)seed, k1 = (uint32_t)(seed >> 32);
#pragma unroll
  for (int r = 0; r < 10; ++r) {
    const uint32_t hi0 = __umulhi(0xD2511F53u, c0), lo0 = 0xD2511F53u * c0;
    const uint32_t hi1 = __umulhi(0xCD9E8D57u, c2), lo1 = 0xCD9E8D57u * c2;
    const uint32_t n0 = hi1 ^ c1 ^ k0, n2 = hi0 ^ c3 ^ k1;
    c0 = n0;
    c1 = lo1;
    c2 = n2;
    c3 = lo0;
    k0 += 0x9E3779B9u;
    k1 += 0xBB67AE85u;
  }
  o0 = c0;
  o1 = c1;
}

__device__ __forceinline__ double unit_open(uint32_t u) {
  return __dmul_rn(__dadd_rn((double)u, 0.5), 2.3283064365386963e-10);
}

__global__ void gen_xr_kernel(uint64_t seed, int64_t n, uint64_t col0, int64_t ncols, double* X,
                              int64_t ld) {
  for (int64_t j = blockIdx.y; j < ncols; j += gridDim.y) {
    const uint64_t c = col0 + (uint64_t)j;
    uint32_t u, dummy;
    philox((uint32_t)c, (uint32_t)(c >> 32), 0u, 5u, seed, u, dummy);
    const double q = __dadd_rn(0.05, __dmul_rn(0.45, unit_open(u)));
    double* col = X + j * ld;
    for (int64_t r = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; r < n;
         r += (int64_t)gridDim.x * blockDim.x) {
      uint32_t a, b;
      philox((uint32_t)c, (uint32_t)(c >> 32), (uint32_t)r, 6u, seed, a, b);
      col[r] = (double)((unit_open(a) < q) + (unit_open(b) < q));
    }
  }
}

}  // namespace

extern "C" {

// Fill X (device, column-major, leading dimension ld >= n) with genotype columns [col0, col0+ncols).
// Returns a cudaError_t value (0 = success).  Asynchronous on `stream`.
int glsgen_dev_xr(uint64_t seed, int64_t n, uint64_t col0, int64_t ncols, double* X, int64_t ld,
                  void* stream) {
  if (ncols <= 0 || n <= 0) return 0;
  const int threads = 256;
  int64_t bx = (n + threads - 1) / threads;
  if (bx > 64) bx = 64;
  int64_t by = ncols < 65535 ? ncols : 65535;
  gen_xr_kernel<<<dim3((unsigned)bx, (unsigned)by), threads, 0, (cudaStream_t)stream>>>(seed, n, col0,
                                                                                       ncols, X, ld);
  return (int)cudaGetLastError();
}

}  // extern "C"
