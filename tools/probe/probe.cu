// Step-0 box probe: FP64 DMMA (mma.sync m8n8k4 f64) and DFMA peak microbenchmarks,
// pinned H2D / D2H bandwidth, device properties. Not part of the product path.
#include <cstdio>
#include <cstdlib>
#include <cuda_runtime.h>
#include <vector>
#include <algorithm>

#define CK(x) do { cudaError_t e = (x); if (e != cudaSuccess) { printf("CUDA %s at %d: %s\n", #x, __LINE__, cudaGetErrorString(e)); exit(1);} } while (0)

template <int NACC>
__global__ void dmma_loop(double* out, int iters, double seed) {
  double a = seed + threadIdx.x * 1e-9, b = seed * 0.5;
  double c[NACC][2];
#pragma unroll
  for (int i = 0; i < NACC; ++i) { c[i][0] = 0; c[i][1] = 0; }
  for (int it = 0; it < iters; ++it) {
#pragma unroll
    for (int i = 0; i < NACC; ++i) {
      asm volatile("mma.sync.aligned.m8n8k4.row.col.f64.f64.f64.f64 {%0,%1}, {%2}, {%3}, {%0,%1};\n"
                   : "+d"(c[i][0]), "+d"(c[i][1]) : "d"(a), "d"(b));
    }
  }
  double s = 0;
#pragma unroll
  for (int i = 0; i < NACC; ++i) s += c[i][0] + c[i][1];
  if (s == 12345.678) out[0] = s;
}

template <int NACC>
__global__ void dfma_loop(double* out, int iters, double seed) {
  double a = seed + threadIdx.x * 1e-9, b = 0.999999;
  double c[NACC];
#pragma unroll
  for (int i = 0; i < NACC; ++i) c[i] = i;
  for (int it = 0; it < iters; ++it) {
#pragma unroll
    for (int i = 0; i < NACC; ++i) c[i] = fma(c[i], b, a);
  }
  double s = 0;
#pragma unroll
  for (int i = 0; i < NACC; ++i) s += c[i];
  if (s == 12345.678) out[0] = s;
}

int main(int argc, char** argv) {
  cudaDeviceProp p; CK(cudaGetDeviceProperties(&p, 0));
  printf("device %s sms=%d l2=%d smem_optin=%zu regs/sm=%d clock_khz=%d memclk_khz=%d busw=%d\n",
         p.name, p.multiProcessorCount, p.l2CacheSize, p.sharedMemPerBlockOptin, p.regsPerMultiprocessor,
         p.clockRate, p.memoryClockRate, p.memoryBusWidth);
  size_t fr, tot; CK(cudaMemGetInfo(&fr, &tot)); printf("mem free=%.1f GB total=%.1f GB\n", fr/1e9, tot/1e9);
  double* d; CK(cudaMalloc(&d, 8));
  cudaEvent_t e0, e1; cudaEventCreate(&e0); cudaEventCreate(&e1);
  int sms = p.multiProcessorCount;
  // DMMA: warps per SM sweep
  for (int wps : {4, 8, 16}) {
    int iters = 20000;
    dim3 grid(sms * 1), block(32 * wps);
    dmma_loop<8><<<grid, block>>>(d, 100, 1.0);
    CK(cudaDeviceSynchronize());
    cudaEventRecord(e0);
    dmma_loop<8><<<grid, block>>>(d, iters, 1.0);
    cudaEventRecord(e1); CK(cudaEventSynchronize(e1));
    float ms; cudaEventElapsedTime(&ms, e0, e1);
    double flops = 2.0 * 256 * 8 * (double)iters * grid.x * wps;
    printf("DMMA m8n8k4 burst: warps/SM=%d  %.2f TFLOP/s  (%.3f ms)\n", wps, flops / ms / 1e9, ms);
  }
  // sustained ~4 s
  {
    int wps = 8, iters = 20000; dim3 grid(sms), block(32 * wps);
    double flops1 = 2.0 * 256 * 8 * (double)iters * grid.x * wps;
    cudaEventRecord(e0); int reps = 0; float ms = 0;
    while (ms < 4000) { dmma_loop<8><<<grid, block>>>(d, iters, 1.0); reps++; cudaEventRecord(e1); CK(cudaEventSynchronize(e1)); cudaEventElapsedTime(&ms, e0, e1); }
    printf("DMMA m8n8k4 sustained(4s): %.2f TFLOP/s\n", flops1 * reps / ms / 1e9);
  }
  for (int wps : {8, 16, 32}) {
    int iters = 20000; dim3 grid(sms), block(32 * wps);
    dfma_loop<8><<<grid, block>>>(d, 100, 1.0); CK(cudaDeviceSynchronize());
    cudaEventRecord(e0);
    dfma_loop<8><<<grid, block>>>(d, iters, 1.0);
    cudaEventRecord(e1); CK(cudaEventSynchronize(e1));
    float ms; cudaEventElapsedTime(&ms, e0, e1);
    double flops = 2.0 * 32 * 8 * (double)iters * grid.x * wps;
    printf("DFMA burst: warps/SM=%d  %.2f TFLOP/s\n", wps, flops / ms / 1e9);
  }
  // H2D / D2H pinned
  size_t bytes = (size_t)2 << 30;
  void *h, *dd; CK(cudaMallocHost(&h, bytes)); CK(cudaMalloc(&dd, bytes));
  memset(h, 1, bytes);
  for (int dir = 0; dir < 2; ++dir) {
    float best = 1e9;
    for (int r = 0; r < 5; ++r) {
      cudaEventRecord(e0);
      if (dir == 0) cudaMemcpyAsync(dd, h, bytes, cudaMemcpyHostToDevice); else cudaMemcpyAsync(h, dd, bytes, cudaMemcpyDeviceToHost);
      cudaEventRecord(e1); CK(cudaEventSynchronize(e1)); float ms; cudaEventElapsedTime(&ms, e0, e1); best = std::min(best, ms);
    }
    printf("%s pinned 2GiB: %.1f GB/s\n", dir == 0 ? "H2D" : "D2H", bytes / best / 1e6);
  }
  // bidirectional concurrent
  {
    cudaStream_t s1, s2; cudaStreamCreate(&s1); cudaStreamCreate(&s2);
    size_t half = bytes / 2;
    cudaEventRecord(e0);
    cudaMemcpyAsync(dd, h, half, cudaMemcpyHostToDevice, s1);
    cudaMemcpyAsync((char*)h + half, (char*)dd + half, half, cudaMemcpyDeviceToHost, s2);
    cudaDeviceSynchronize(); cudaEventRecord(e1); cudaEventSynchronize(e1);
    float ms; cudaEventElapsedTime(&ms, e0, e1);
    printf("H2D+D2H concurrent 1GiB each: %.1f GB/s aggregate\n", 2 * half / ms / 1e6);
  }
  return 0;
}
