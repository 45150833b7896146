// Diagnostics: dependent-chain latency (cycles per op, one warp) of the FP64 scalar ops, 64-bit shuffles,
// rsqrt(double) and a shared-memory store -> __syncwarp -> load round trip on this GPU.
#include <cstdio>
#include <cuda_runtime.h>
__global__ void lat(double x0, long long* out, double* sink) {
  __shared__ double sm[64];
  const int lane = threadIdx.x;
  double x = x0 + lane * 1e-9, y = 1.0000001;
  long long t0, t1;
  const int N = 1024;
  t0 = clock64();
  for (int i = 0; i < N; ++i) x = fma(x, y, 1e-12);
  t1 = clock64(); out[0] = (t1 - t0) / N;
  t0 = clock64();
  for (int i = 0; i < N; ++i) x = x * y;
  t1 = clock64(); out[1] = (t1 - t0) / N;
  t0 = clock64();
  for (int i = 0; i < N; ++i) x = __shfl_sync(0xffffffffu, x, (lane + 1) & 31);
  t1 = clock64(); out[2] = (t1 - t0) / N;
  double r = x;
  t0 = clock64();
  for (int i = 0; i < N; ++i) r = rsqrt(r + 1.5);
  t1 = clock64(); out[3] = (t1 - t0) / N;
  t0 = clock64();
  for (int i = 0; i < N; ++i) {
    sm[lane] = r;
    __syncwarp();
    r = sm[(lane + 1) & 31] + 1e-300;
    __syncwarp();
  }
  t1 = clock64(); out[4] = (t1 - t0) / N;
  float f = (float)x;
  t0 = clock64();
  for (int i = 0; i < N; ++i) f = fmaf(f, 1.0000001f, 1e-7f);
  t1 = clock64(); out[5] = (t1 - t0) / N;
  double a[2] = {x, r}, b = y;
  double c[2] = {0, 0};
  t0 = clock64();
  for (int i = 0; i < N; ++i)
    asm volatile("mma.sync.aligned.m8n8k4.row.col.f64.f64.f64.f64 {%0,%1}, {%2}, {%3}, {%0,%1};\n"
                 : "+d"(c[0]), "+d"(c[1]) : "d"(a[0]), "d"(b));
  t1 = clock64(); out[6] = (t1 - t0) / N;
  t0 = clock64();
  for (int i = 0; i < N; ++i) x = sqrt(x);
  t1 = clock64(); out[7] = (t1 - t0) / N;
  sink[lane] = x + r + f + c[0] + c[1];
}
int main() {
  long long* o; double* s;
  cudaMallocManaged(&o, 64 * 8); cudaMallocManaged(&s, 64 * 8);
  for (int k = 0; k < 2; ++k) { lat<<<1, 32>>>(1.1, o, s); cudaDeviceSynchronize(); }
  const char* nm[] = {"DFMA", "DMUL", "SHFL(f64)", "rsqrt(f64)", "STS+syncwarp+LDS", "FFMA", "DMMA m8n8k4 (acc chain)", "sqrt(f64)"};
  for (int i = 0; i < 8; ++i) printf("%-28s %lld cycles\n", nm[i], o[i]);
  return 0;
}
