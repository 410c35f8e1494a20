// How many thread-block clusters of a given size can be co-resident (one CTA per SM:
// 512 threads, ~155 KB dynamic shared memory, like the C-A cluster tier).
#include <cstdio>
__global__ void kdummy(int *p) { if (p) p[threadIdx.x] = 0; }
int main() {
  cudaFuncSetAttribute(kdummy, cudaFuncAttributeMaxDynamicSharedMemorySize, 160 * 1024);
  cudaFuncSetAttribute(kdummy, cudaFuncAttributeNonPortableClusterSizeAllowed, 1);
  for (int cs = 1; cs <= 16; cs *= 2) {
    cudaLaunchConfig_t cfg = {};
    cfg.gridDim = dim3(cs * 64);
    cfg.blockDim = dim3(512);
    cfg.dynamicSmemBytes = 155 * 1024;
    cudaLaunchAttribute at[1];
    at[0].id = cudaLaunchAttributeClusterDimension;
    at[0].val.clusterDim.x = cs; at[0].val.clusterDim.y = 1; at[0].val.clusterDim.z = 1;
    cfg.attrs = at; cfg.numAttrs = 1;
    int n = -1;
    cudaError_t e = cudaOccupancyMaxActiveClusters(&n, kdummy, &cfg);
    printf("cluster size %2d: max active clusters %3d (%3d SMs)  %s\n", cs, n, n * cs, cudaGetErrorString(e));
  }
  return 0;
}
