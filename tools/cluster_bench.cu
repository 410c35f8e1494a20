// Microbenchmark: cycles per cluster.sync() and per (sync + DSMEM read of a remote slot)
// for cluster sizes 1..16, 256 threads per CTA.  nvcc -gencode arch=compute_100a,code=sm_100a
#include <cooperative_groups.h>
#include <cstdio>
namespace cg = cooperative_groups;
__global__ void kbench(unsigned long long *out, int iters, int mode) {
  __shared__ double slot[2];
  cg::cluster_group cl = cg::this_cluster();
  int r = cl.block_rank(), cs = cl.num_blocks();
  slot[0] = r; slot[1] = r;
  cl.sync();
  double acc = 0;
  long long t0 = clock64();
  for (int it = 0; it < iters; ++it) {
    if (mode == 0) {
      cl.sync();
    } else if (mode == 1) {
      if (threadIdx.x == 0) slot[it & 1] = it + r;
      cl.sync();
      if (threadIdx.x < 32) {
        double x = (threadIdx.x < cs) ? *cl.map_shared_rank(&slot[it & 1], threadIdx.x) : 0;
        for (int o = 16; o; o >>= 1) x += __shfl_xor_sync(~0u, x, o);
        acc += x;
      }
      __syncthreads();
    } else {
      __syncthreads();
    }
  }
  long long t1 = clock64();
  if (threadIdx.x == 0 && r == 0) out[blockIdx.x / cs] = (t1 - t0) / iters;
  if (acc == -1) out[0] = 0;
}
int main() {
  unsigned long long *d, h[64];
  cudaMalloc(&d, 64 * 8);
  for (int mode = 0; mode < 3; ++mode)
    for (int cs = 1; cs <= 16; cs *= 2) {
      cudaFuncSetAttribute(kbench, cudaFuncAttributeNonPortableClusterSizeAllowed, 1);
      cudaLaunchConfig_t cfg = {};
      cfg.gridDim = dim3(cs);
      cfg.blockDim = dim3(256);
      cudaLaunchAttribute at[1];
      at[0].id = cudaLaunchAttributeClusterDimension;
      at[0].val.clusterDim.x = cs; at[0].val.clusterDim.y = 1; at[0].val.clusterDim.z = 1;
      cfg.attrs = at; cfg.numAttrs = 1;
      cudaLaunchKernelEx(&cfg, kbench, d, 1000, mode);
      cudaError_t e = cudaDeviceSynchronize();
      cudaMemcpy(h, d, 8, cudaMemcpyDeviceToHost);
      printf("mode %d (%s) cs %2d: %llu cycles/iter  %s\n", mode, mode == 0 ? "cluster.sync" : mode == 1 ? "sync+dsmem" : "syncthreads",
             cs, h[0], cudaGetErrorString(e));
    }
  return 0;
}
