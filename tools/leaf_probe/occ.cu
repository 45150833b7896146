// Diagnostics: how many clusters of 2 / 4 / 8 CTAs of the int8 hot kernel's shape (384 threads, ~215 KB
// dynamic shared memory, one CTA per SM) can be resident at once on this GPU.
#include <cstdio>
#include <cuda_runtime.h>
__global__ void k384(int* p) { if (p) p[threadIdx.x] = 0; }
int main() {
  cudaFuncSetAttribute(k384, cudaFuncAttributeMaxDynamicSharedMemorySize, 219648);
  cudaFuncSetAttribute(k384, cudaFuncAttributeNonPortableClusterSizeAllowed, 1);
  int sms = 0;
  cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, 0);
  for (int cs : {1, 2, 4, 8, 16}) {
    cudaLaunchConfig_t cfg = {};
    cudaLaunchAttribute at[1];
    at[0].id = cudaLaunchAttributeClusterDimension;
    at[0].val.clusterDim.x = cs; at[0].val.clusterDim.y = 1; at[0].val.clusterDim.z = 1;
    cfg.gridDim = dim3(cs * 64); cfg.blockDim = dim3(384); cfg.dynamicSmemBytes = 219648;
    cfg.attrs = at; cfg.numAttrs = 1;
    int n = -1;
    cudaError_t e = cudaOccupancyMaxActiveClusters(&n, k384, &cfg);
    printf("cluster %2d: %3d clusters resident = %3d SMs of %d (%s)\n", cs, n, n * cs, sms, cudaGetErrorString(e));
  }
  return 0;
}
