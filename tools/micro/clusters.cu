// How many clusters of size 2/4/8/16 can be co-resident with ~200 KB shared
// memory per CTA (one CTA per SM) on this GPU.
#include <cstdio>
#include <cuda_runtime.h>
__global__ void k(int* p) { extern __shared__ int s[]; if (p) p[0] = s[0]; }
int main() {
  int sms; cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, 0);
  cudaFuncSetAttribute(k, cudaFuncAttributeNonPortableClusterSizeAllowed, 1);
  for (int smem : {100 * 1024, 200 * 1024}) {
    cudaFuncSetAttribute(k, cudaFuncAttributeMaxDynamicSharedMemorySize, smem);
    for (int c : {1, 2, 4, 8, 16}) {
      cudaLaunchConfig_t cfg = {};
      cudaLaunchAttribute a; a.id = cudaLaunchAttributeClusterDimension;
      a.val.clusterDim.x = c; a.val.clusterDim.y = 1; a.val.clusterDim.z = 1;
      cfg.gridDim = dim3(sms / c * c); cfg.blockDim = dim3(192); cfg.dynamicSmemBytes = smem;
      cfg.attrs = &a; cfg.numAttrs = 1;
      int n = -1; cudaError_t e = cudaOccupancyMaxActiveClusters(&n, k, &cfg);
      printf("smem %3d KB cluster %2d: max active clusters %3d (%3d CTAs) %s\n", smem / 1024, c, n, n * c,
             cudaGetErrorString(e));
    }
  }
  return 0;
}
