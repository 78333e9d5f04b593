// How many clusters of 1/2/4 CTAs (192 threads, S KiB dynamic smem) can be
// co-resident on this GPU (cudaOccupancyMaxActiveClusters)? A persistent grid
// larger than this runs its surplus clusters in a second wave.
#include <cuda_runtime.h>
#include <cstdio>
__global__ void k(int* p) { if (p) p[0] = 1; }
int main() {
  int sms = 0;
  cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, 0);
  cudaFuncSetAttribute(k, cudaFuncAttributeMaxDynamicSharedMemorySize, 232448);
  cudaFuncSetAttribute(k, cudaFuncAttributeNonPortableClusterSizeAllowed, 1);
  for (int cs : {1, 2, 4, 8}) {
    for (int smem : {100 * 1024, 200 * 1024, 232448}) {
      cudaLaunchConfig_t lc = {};
      lc.gridDim = dim3(sms / cs * cs);
      lc.blockDim = dim3(192);
      lc.dynamicSmemBytes = smem;
      cudaLaunchAttribute at[1];
      at[0].id = cudaLaunchAttributeClusterDimension;
      at[0].val.clusterDim.x = cs; at[0].val.clusterDim.y = 1; at[0].val.clusterDim.z = 1;
      lc.attrs = at; lc.numAttrs = 1;
      int n = -1;
      cudaError_t e = cudaOccupancyMaxActiveClusters(&n, k, &lc);
      printf("cluster %d smem %6d: max active clusters %d (%d CTAs of %d SMs) err=%d\n", cs, smem, n, n * cs, sms, (int)e);
    }
  }
  return 0;
}
