// Probe: how many clusters of CS CTAs (288 threads, ~220 KB shared memory,
// one CTA per SM) can be co-resident on this GPU (GPC packing).
#include <cstdio>
#include <cuda_runtime.h>
__global__ void k(int* p) {
  extern __shared__ int s[];
  if (threadIdx.x == 0 && p) p[blockIdx.x] = s[0];
}
int main() {
  cudaFuncSetAttribute(k, cudaFuncAttributeMaxDynamicSharedMemorySize, 227 * 1024);
  cudaFuncSetAttribute(k, cudaFuncAttributeNonPortableClusterSizeAllowed, 1);
  for (size_t smem : {size_t(220 * 1024), size_t(110 * 1024)}) {
    for (int cs : {1, 2, 3, 4, 5, 6, 8, 16}) {
      cudaLaunchConfig_t cfg = {};
      cfg.gridDim = dim3(cs * 64);
      cfg.blockDim = dim3(288);
      cfg.dynamicSmemBytes = smem;
      cudaLaunchAttribute at[1];
      at[0].id = cudaLaunchAttributeClusterDimension;
      at[0].val.clusterDim.x = cs;
      at[0].val.clusterDim.y = 1;
      at[0].val.clusterDim.z = 1;
      cfg.attrs = at;
      cfg.numAttrs = 1;
      int n = -1;
      cudaError_t e = cudaOccupancyMaxActiveClusters(&n, k, &cfg);
      printf("smem %zu KB cs %2d: max active clusters %d (%d CTAs) %s\n", smem / 1024, cs, n, n * cs,
             e == cudaSuccess ? "" : cudaGetErrorString(e));
    }
  }
  return 0;
}
