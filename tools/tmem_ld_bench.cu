// tmem_ld_bench.cu — TMEM read throughput per SM for the tcgen05.ld shapes the residual's
// epilogue could use (the PRECISE residual is bounded by TMEM reads).
// One CTA per SM (148), NW warps; each warp reads its lane quarter (warp % 4) of a 512-column
// TMEM allocation repeatedly; bytes read / cycles per SM is printed per shape and warp count.
//   nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o tools/tmem_ld_bench tools/tmem_ld_bench.cu
#include <cstdio>
#include <cstdint>
#include <cuda_runtime.h>

__device__ __forceinline__ uint32_t smem_u32(const void *p) { return (uint32_t)__cvta_generic_to_shared(p); }

#define LD8(shape, base)                                                                                   \
  asm volatile("tcgen05.ld.sync.aligned." shape ".b32 {%0,%1,%2,%3,%4,%5,%6,%7}, [%8];\n"              \
               : "=r"(v[0]), "=r"(v[1]), "=r"(v[2]), "=r"(v[3]), "=r"(v[4]), "=r"(v[5]), "=r"(v[6]), "=r"(v[7]) \
               : "r"(base))
#define LD16(shape, base)                                                                                  \
  asm volatile("tcgen05.ld.sync.aligned." shape ".b32 {%0,%1,%2,%3,%4,%5,%6,%7,%8,%9,%10,%11,%12,%13,%14,%15}, [%16];\n" \
               : "=r"(v[0]), "=r"(v[1]), "=r"(v[2]), "=r"(v[3]), "=r"(v[4]), "=r"(v[5]), "=r"(v[6]), "=r"(v[7]), \
                 "=r"(v[8]), "=r"(v[9]), "=r"(v[10]), "=r"(v[11]), "=r"(v[12]), "=r"(v[13]), "=r"(v[14]), "=r"(v[15]) \
               : "r"(base))
#define LD32(shape, base)                                                                                  \
  asm volatile("tcgen05.ld.sync.aligned." shape ".b32 {%0,%1,%2,%3,%4,%5,%6,%7,%8,%9,%10,%11,%12,%13,%14,%15,"   \
               "%16,%17,%18,%19,%20,%21,%22,%23,%24,%25,%26,%27,%28,%29,%30,%31}, [%32];\n"                   \
               : "=r"(v[0]), "=r"(v[1]), "=r"(v[2]), "=r"(v[3]), "=r"(v[4]), "=r"(v[5]), "=r"(v[6]), "=r"(v[7]), \
                 "=r"(v[8]), "=r"(v[9]), "=r"(v[10]), "=r"(v[11]), "=r"(v[12]), "=r"(v[13]), "=r"(v[14]), "=r"(v[15]), \
                 "=r"(v[16]), "=r"(v[17]), "=r"(v[18]), "=r"(v[19]), "=r"(v[20]), "=r"(v[21]), "=r"(v[22]), "=r"(v[23]), \
                 "=r"(v[24]), "=r"(v[25]), "=r"(v[26]), "=r"(v[27]), "=r"(v[28]), "=r"(v[29]), "=r"(v[30]), "=r"(v[31]) \
               : "r"(base))

// SHAPE: 0 = 32x32b.x8, 1 = 32x32b.x16, 2 = 32x32b.x32, 3 = 16x256b.x2 (8 regs), 4 = 16x128b.x4 (8 regs),
//        5 = 32x32b.x8 pair in flight (two loads, one wait)
template <int SHAPE>
__global__ void __launch_bounds__(512, 1) k_ld(int iters, unsigned long long *cyc, unsigned *sink) {
  __shared__ uint32_t tb;
  const int warp = threadIdx.x >> 5;
  if (warp == 0) {
    asm volatile("tcgen05.alloc.cta_group::1.sync.aligned.shared::cta.b32 [%0], 512;\n" ::"r"(smem_u32(&tb)));
    asm volatile("tcgen05.relinquish_alloc_permit.cta_group::1.sync.aligned;\n");
  }
  asm volatile("tcgen05.fence::before_thread_sync;\n" ::: "memory");
  __syncthreads();
  asm volatile("tcgen05.fence::after_thread_sync;\n" ::: "memory");
  const uint32_t base = tb + ((uint32_t)(32 * (warp & 3)) << 16);
  const int colw = 32 * ((warp >> 2) & 3);   // warps of the same quarter read different columns
  unsigned acc = 0;
  uint32_t v[32];
  __syncthreads();
  long long t0 = clock64();
  for (int it = 0; it < iters; ++it) {
    const uint32_t a = base + (uint32_t)((colw + 8 * (it & 3)) & 511);
    if (SHAPE == 0) { LD8("32x32b.x8", a); }
    else if (SHAPE == 1) { LD16("32x32b.x16", a); }
    else if (SHAPE == 2) { LD32("32x32b.x32", a); }
    else if (SHAPE == 3) { LD8("16x256b.x2", a); }
    else if (SHAPE == 4) { LD8("16x128b.x4", a); }
    else {
      LD8("32x32b.x8", a);
      asm volatile("tcgen05.ld.sync.aligned.32x32b.x8.b32 {%0,%1,%2,%3,%4,%5,%6,%7}, [%8];\n"
                   : "=r"(v[8]), "=r"(v[9]), "=r"(v[10]), "=r"(v[11]), "=r"(v[12]), "=r"(v[13]), "=r"(v[14]), "=r"(v[15])
                   : "r"(a + 128));
    }
    asm volatile("tcgen05.wait::ld.sync.aligned;\n" ::: "memory");
    const int nr = SHAPE == 1 ? 16 : SHAPE == 2 ? 32 : SHAPE == 5 ? 16 : 8;
#pragma unroll
    for (int i = 0; i < 32; ++i)
      if (i < nr) acc ^= v[i];
  }
  __syncthreads();
  long long t1 = clock64();
  if (threadIdx.x == 0) atomicAdd(cyc, (unsigned long long)(t1 - t0));
  if (acc == 0x12345678u) sink[0] = acc;
  asm volatile("tcgen05.fence::before_thread_sync;\n" ::: "memory");
  __syncthreads();
  if (warp == 0) {
    asm volatile("tcgen05.fence::after_thread_sync;\n" ::: "memory");
    asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, 512;\n" ::"r"(tb));
  }
}

template <int SHAPE>
static void run(const char *name, int bytes_per_thread, int nw) {
  unsigned long long *cyc;
  unsigned *sink;
  cudaMalloc(&cyc, 8);
  cudaMalloc(&sink, 4);
  cudaMemset(cyc, 0, 8);
  const int iters = 4096;
  k_ld<SHAPE><<<148, 32 * nw>>>(iters, cyc, sink);
  cudaDeviceSynchronize();
  cudaMemset(cyc, 0, 8);
  k_ld<SHAPE><<<148, 32 * nw>>>(iters, cyc, sink);
  cudaError_t e = cudaDeviceSynchronize();
  unsigned long long c = 0;
  cudaMemcpy(&c, cyc, 8, cudaMemcpyDeviceToHost);
  const double per_sm_cyc = (double)c / 148.0;
  const double bytes = (double)iters * nw * 32 * bytes_per_thread;
  printf("%-22s warps=%2d  %7.1f B/clk/SM  %s\n", name, nw, bytes / per_sm_cyc, e == cudaSuccess ? "" : cudaGetErrorString(e));
  cudaFree(cyc);
  cudaFree(sink);
}

int main() {
  for (int nw : {4, 8, 16}) {
    run<0>("32x32b.x8", 32, nw);
    run<1>("32x32b.x16", 64, nw);
    run<2>("32x32b.x32", 128, nw);
    run<3>("16x256b.x2", 32, nw);
    run<4>("16x128b.x4", 32, nw);
    run<5>("32x32b.x8 x2 in flight", 64, nw);
  }
  return 0;
}
