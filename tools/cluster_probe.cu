// How many clusters of C CTAs (384 threads, ~227 KB dynamic smem: the megakernel's
// footprint) can be co-resident on this GPU: the persistent grid must fit in one wave.
#include <cstdio>
#include <cuda_runtime.h>
__global__ void k(int* out) {
  extern __shared__ int s[];
  if (threadIdx.x == 0) { s[0] = blockIdx.x; out[blockIdx.x] = s[0]; }
}
int main() {
  int dev = 0, sms = 0;
  cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev);
  const int smem = 227 * 1024;
  cudaFuncSetAttribute(k, cudaFuncAttributeMaxDynamicSharedMemorySize, smem);
  cudaFuncSetAttribute(k, cudaFuncAttributeNonPortableClusterSizeAllowed, 1);
  printf("SMs %d\n", sms);
  for (int c : {1, 2, 4, 8, 16}) {
    cudaLaunchConfig_t cfg = {};
    cfg.gridDim = dim3(c * 64);
    cfg.blockDim = dim3(384);
    cfg.dynamicSmemBytes = smem;
    cudaLaunchAttribute a[1];
    a[0].id = cudaLaunchAttributeClusterDimension;
    a[0].val.clusterDim.x = c; a[0].val.clusterDim.y = 1; a[0].val.clusterDim.z = 1;
    cfg.attrs = a; cfg.numAttrs = 1;
    int n = -1;
    cudaError_t e = cudaOccupancyMaxActiveClusters(&n, k, &cfg);
    printf("cluster %2d: max active clusters %d -> %d CTAs (%s)\n", c, n, n * c, cudaGetErrorString(e));
  }
  return 0;
}
