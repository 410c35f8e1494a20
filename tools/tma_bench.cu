// tma_bench.cu — TMA read throughput of a column-major fp32 4096 x 4096 matrix (64 MB) by
// boxes of BR rows x BC columns, 128 CTAs (tile = 128-row block, Q = 4 K parts), a ring of NST
// stages per CTA, one thread issuing and waiting (no compute).  Prints GB/s per box shape.
//   nvcc -gencode arch=compute_100a,code=sm_100a -O3 -std=c++17 -o tools/tma_bench tools/tma_bench.cu
#include <cuda.h>
#include <cudaTypedefs.h>
#include <cuda_runtime.h>

#include <cstdio>
#include <cstring>

__device__ __forceinline__ uint32_t su(const void *p) { return (uint32_t)__cvta_generic_to_shared(p); }

__global__ void __launch_bounds__(32) k_tma(const __grid_constant__ CUtensorMap tm, int m, int n, int BR, int BC, int NST,
                                            int T, int Q) {
  extern __shared__ __align__(1024) unsigned char sm[];
  __shared__ __align__(8) unsigned long long bar[16];
  if (threadIdx.x != 0) return;
  for (int i = 0; i < NST; ++i) asm volatile("mbarrier.init.shared::cta.b64 [%0], 1;" ::"r"(su(&bar[i])));
  asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
  const int tile = blockIdx.x % T, q = blockIdx.x / T;
  const int rows_per_tile = m / T;
  const int c0 = q * n / Q, c1 = (q + 1) * n / Q;
  const int stage_bytes = BR * BC * 4;
  int k = 0;
  for (int r = tile * rows_per_tile; r < (tile + 1) * rows_per_tile; r += BR)
    for (int c = c0; c < c1; c += BC, ++k) {
      const int s = k % NST;
      if (k >= NST) {
        uint32_t done = 0, ph = ((k / NST) - 1) & 1;
        do {
          asm volatile("{.reg .pred p; mbarrier.try_wait.parity.shared::cta.b64 p, [%1], %2; selp.u32 %0,1,0,p;}"
                       : "=r"(done) : "r"(su(&bar[s])), "r"(ph) : "memory");
        } while (!done);
      }
      asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(su(&bar[s])), "r"(stage_bytes) : "memory");
      asm volatile(
          "cp.async.bulk.tensor.2d.shared::cluster.global.tile.mbarrier::complete_tx::bytes [%0], [%1, {%2, %3}], [%4];" ::"r"(
              su(sm + (size_t)s * stage_bytes)),
          "l"(reinterpret_cast<uint64_t>(&tm)), "r"(r), "r"(c), "r"(su(&bar[s]))
          : "memory");
    }
  for (int j = k - NST; j < k; ++j) {
    if (j < 0) continue;
    const int s = j % NST;
    uint32_t done = 0, ph = (j / NST) & 1;
    do {
      asm volatile("{.reg .pred p; mbarrier.try_wait.parity.shared::cta.b64 p, [%1], %2; selp.u32 %0,1,0,p;}"
                   : "=r"(done) : "r"(su(&bar[s])), "r"(ph) : "memory");
    } while (!done);
  }
}

int main() {
  const int m = 4096, n = 4096;
  float *W;
  cudaMalloc(&W, (size_t)m * n * 4);
  cudaMemset(W, 0, (size_t)m * n * 4);
  void *fp = nullptr;
  cudaDriverEntryPointQueryResult qr;
  cudaGetDriverEntryPoint("cuTensorMapEncodeTiled", &fp, cudaEnableDefault, &qr);
  auto enc = reinterpret_cast<PFN_cuTensorMapEncodeTiled_v12000>(fp);
  struct Cfg { int BR, BC, NST, T, Q; } cfgs[] = {{128, 32, 8, 32, 4}, {128, 32, 12, 32, 4}, {256, 16, 8, 16, 8},
                                                  {256, 32, 6, 16, 8}, {128, 64, 4, 32, 4}, {256, 8, 12, 16, 8},
                                                  {128, 32, 8, 128, 1}};
  for (auto c : cfgs) {
    CUtensorMap tm;
    memset(&tm, 0, sizeof(tm));
    cuuint64_t dims[2] = {(cuuint64_t)m, (cuuint64_t)n};
    cuuint64_t str[1] = {(cuuint64_t)m * 4};
    cuuint32_t box[2] = {(cuuint32_t)c.BR, (cuuint32_t)c.BC}, es[2] = {1, 1};
    enc(&tm, CU_TENSOR_MAP_DATA_TYPE_FLOAT32, 2, W, dims, str, box, es, CU_TENSOR_MAP_INTERLEAVE_NONE,
        CU_TENSOR_MAP_SWIZZLE_NONE, CU_TENSOR_MAP_L2_PROMOTION_L2_256B, CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
    const int smem = c.BR * c.BC * 4 * c.NST;
    cudaFuncSetAttribute(k_tma, cudaFuncAttributeMaxDynamicSharedMemorySize, smem);
    cudaEvent_t e0, e1;
    cudaEventCreate(&e0);
    cudaEventCreate(&e1);
    float best = 1e9;
    for (int rep = 0; rep < 5; ++rep) {
      cudaEventRecord(e0);
      k_tma<<<c.T * c.Q, 32, smem>>>(tm, m, n, c.BR, c.BC, c.NST, c.T, c.Q);
      cudaEventRecord(e1);
      cudaEventSynchronize(e1);
      float ms;
      cudaEventElapsedTime(&ms, e0, e1);
      best = ms < best ? ms : best;
    }
    printf("box %3dx%-3d stages %2d grid %3d (T %d Q %d): %7.1f us  %6.0f GB/s  %s\n", c.BR, c.BC, c.NST, c.T * c.Q, c.T,
           c.Q, best * 1e3, (double)m * n * 4 / (best * 1e-3) / 1e9, cudaGetErrorString(cudaGetLastError()));
  }
  return 0;
}
