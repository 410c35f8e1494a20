// mma_issue_bench.cu — issue cost of tcgen05.mma kind::i8 (M = 128, K = 32, TS mode: A in TMEM,
// B in shared memory) per instruction, for N = 16 .. 256, from one issuing thread, and from two
// issuing warps into disjoint accumulators.  148 CTAs (one per SM); prints cycles per MMA.
//   nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o tools/mma_issue_bench tools/mma_issue_bench.cu
#include <cstdio>
#include <cstdint>
#include <cuda_runtime.h>

__device__ __forceinline__ uint32_t smem_u32(const void *p) { return (uint32_t)__cvta_generic_to_shared(p); }
__device__ __forceinline__ uint64_t smem_desc(uint32_t addr) {
  return (uint64_t)((addr & 0x3FFFF) >> 4) | ((uint64_t)(128 >> 4) << 16) | ((uint64_t)(256 >> 4) << 32) | (1ull << 46);
}
__device__ __forceinline__ void mma_ts(uint32_t d, uint32_t a, uint64_t bdesc, uint32_t idesc, uint32_t acc) {
  asm volatile("{\n\t.reg .pred p;\n\tsetp.ne.b32 p, %4, 0;\n\t"
               "tcgen05.mma.cta_group::1.kind::i8 [%0], [%1], %2, %3, p;\n\t}\n" ::"r"(d), "r"(a), "l"(bdesc),
               "r"(idesc), "r"(acc));
}
__device__ __forceinline__ void mma_ss(uint32_t d, uint64_t adesc, uint64_t bdesc, uint32_t idesc, uint32_t acc) {
  asm volatile("{\n\t.reg .pred p;\n\tsetp.ne.b32 p, %4, 0;\n\t"
               "tcgen05.mma.cta_group::1.kind::i8 [%0], %1, %2, %3, p;\n\t}\n" ::"r"(d), "l"(adesc), "l"(bdesc),
               "r"(idesc), "r"(acc));
}
__device__ __forceinline__ void commit(uint32_t mbar) {
  asm volatile("tcgen05.commit.cta_group::1.mbarrier::arrive::one.shared::cluster.b64 [%0];\n" ::"r"(mbar) : "memory");
}
__device__ __forceinline__ void mbar_wait(uint32_t addr, uint32_t phase) {
  uint32_t done = 0;
  do {
    asm volatile("{\n\t.reg .pred p;\n\tmbarrier.try_wait.parity.shared::cta.b64 p, [%1], %2;\n\tselp.u32 %0, 1, 0, p;\n\t}\n"
                 : "=r"(done) : "r"(addr), "r"(phase) : "memory");
  } while (!done);
}

// MODE 0: TS one issuer; 1: SS one issuer; 2: TS two issuing warps; 3: TS four issuing warps
template <int MODE>
__global__ void __launch_bounds__(128, 1) k_mma(int N, int iters, unsigned long long *cyc) {
  extern __shared__ __align__(1024) unsigned char sm[];
  __shared__ uint32_t tb;
  __shared__ __align__(8) unsigned long long bar[4];
  const int warp = threadIdx.x >> 5;
  for (int i = threadIdx.x; i < 65536 / 4; i += blockDim.x) reinterpret_cast<uint32_t *>(sm)[i] = 0x01010101u * (i & 3);
  if (warp == 0) {
    asm volatile("tcgen05.alloc.cta_group::1.sync.aligned.shared::cta.b32 [%0], 512;\n" ::"r"(smem_u32(&tb)));
    asm volatile("tcgen05.relinquish_alloc_permit.cta_group::1.sync.aligned;\n");
  }
  if (threadIdx.x == 0) {
    for (int i = 0; i < 4; ++i) asm volatile("mbarrier.init.shared::cta.b64 [%0], 1;\n" ::"r"(smem_u32(&bar[i])));
    asm volatile("fence.mbarrier_init.release.cluster;\n" ::: "memory");
  }
  asm volatile("fence.proxy.async.shared::cta;\n" ::: "memory");
  asm volatile("tcgen05.fence::before_thread_sync;\n" ::: "memory");
  __syncthreads();
  asm volatile("tcgen05.fence::after_thread_sync;\n" ::: "memory");
  const uint32_t idesc = (2u << 4) | (1u << 7) | (1u << 10) | ((uint32_t)(N >> 3) << 17) | ((uint32_t)(128 >> 4) << 24);
  const uint64_t bdesc = smem_desc(smem_u32(sm));
  const uint64_t adesc = smem_desc(smem_u32(sm + 32768));
  const uint32_t a_t = tb + 448;              // A in TMEM columns 448.. (64 columns)
  (void)N;
  long long t0 = clock64();
  // NWARP issuing warps (one elected lane each), 16 straight-line MMAs per iteration into 4
  // accumulators of the warp's own TMEM quarter (columns [warp*112, warp*112+112))
  constexpr int NWARP = MODE == 2 ? 2 : (MODE == 3 ? 4 : 1);
  if (warp < NWARP && (threadIdx.x & 31) == 0) {
    const uint32_t dq = tb + (uint32_t)(warp * (NWARP == 4 ? 96 : 192));
    const uint32_t span = (uint32_t)(NWARP == 4 ? 96 : 192) / 4u;      // 4 accumulators per warp
    for (int it = 0; it < iters / 16; ++it) {
#pragma unroll
      for (int u = 0; u < 16; ++u) {
        const uint32_t d = dq + (uint32_t)(u & 3) * (span < (uint32_t)N ? 0u : span);
        if (MODE == 1) mma_ss(d, adesc, bdesc, idesc, 1u);
        else mma_ts(d, a_t + 8 * (u & 7), bdesc, idesc, 1u);
      }
    }
    commit(smem_u32(&bar[warp]));
    mbar_wait(smem_u32(&bar[warp]), 0);
  }
  __syncthreads();
  long long t1 = clock64();
  if (threadIdx.x == 0) atomicAdd(cyc, (unsigned long long)(t1 - t0));
  asm volatile("tcgen05.fence::before_thread_sync;\n" ::: "memory");
  __syncthreads();
  if (warp == 0) {
    asm volatile("tcgen05.fence::after_thread_sync;\n" ::: "memory");
    asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, 512;\n" ::"r"(tb));
  }
}

template <int MODE>
static void run(const char *name, int N) {
  unsigned long long *cyc;
  cudaMalloc(&cyc, 8);
  const int iters = 4096;
  cudaFuncSetAttribute(k_mma<MODE>, cudaFuncAttributeMaxDynamicSharedMemorySize, 65536);
  for (int rep = 0; rep < 2; ++rep) {
    cudaMemset(cyc, 0, 8);
    k_mma<MODE><<<148, 128, 65536>>>(N, iters, cyc);
  }
  cudaError_t e = cudaDeviceSynchronize();
  unsigned long long c = 0;
  cudaMemcpy(&c, cyc, 8, cudaMemcpyDeviceToHost);
  const double per = (double)c / 148.0 / (MODE == 2 ? 2 * iters : MODE == 3 ? 4 * iters : iters);
  printf("%-10s N=%3d  %6.1f cycles/MMA  (math floor %5.1f)  %s\n", name, N, per, 128.0 * N / 256.0,
         e == cudaSuccess ? "" : cudaGetErrorString(e));
  cudaFree(cyc);
}

int main() {
  for (int N : {16, 32, 64}) {
    run<0>("TS", N);
    run<1>("SS", N);
    run<2>("TS 2 warps", N);
    run<3>("TS 4 warps", N);
  }
  return 0;
}
