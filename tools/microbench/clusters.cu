// Resident-cluster capacity of a 768-thread, ~218 KB shared-memory kernel for cluster sizes 1..8
// (cudaOccupancyMaxActiveClusters): the slot count kernel 2b's grid planner divides by.
#include <cstdio>
#include <cuda_runtime.h>
__global__ void k768(int* p) { extern __shared__ int s[]; if (p) p[threadIdx.x] = s[threadIdx.x]; }
int main() {
  int smems[] = {105536, 150000, 198720, 218176, 225000};
  for (int smem : smems) {
    cudaFuncSetAttribute(k768, cudaFuncAttributeMaxDynamicSharedMemorySize, smem);
    cudaFuncSetAttribute(k768, cudaFuncAttributeNonPortableClusterSizeAllowed, 1);
    printf("smem %d:", smem);
    for (int G = 1; G <= 16; ++G) {
      cudaLaunchConfig_t cfg = {};
      cfg.gridDim = dim3(G, 1, 1);
      cfg.blockDim = dim3(768);
      cfg.dynamicSmemBytes = smem;
      cudaLaunchAttribute a[1];
      a[0].id = cudaLaunchAttributeClusterDimension;
      a[0].val.clusterDim.x = G; a[0].val.clusterDim.y = 1; a[0].val.clusterDim.z = 1;
      cfg.attrs = a; cfg.numAttrs = 1;
      int n = -1;
      cudaError_t e = cudaOccupancyMaxActiveClusters(&n, k768, &cfg);
      if (e != cudaSuccess) { cudaGetLastError(); printf(" G%d:err", G); }
      else printf(" G%d:%d(%d SMs)", G, n, n * G);
    }
    printf("\n");
  }
  return 0;
}
