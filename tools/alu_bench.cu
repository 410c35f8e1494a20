// alu_bench.cu — per-SM throughput (thread-ops per clock) of the arithmetic the residual
// epilogue can use: DFMA, DADD, FFMA, I2F.F64.S32, I2F.F32.S32, F2F.F64.F32, F2F.F32.F64,
// IMAD, IMAD.WIDE.  148 CTAs x 512 threads, 8 independent chains per thread.
//   nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o tools/alu_bench tools/alu_bench.cu
#include <cstdio>
#include <cstdint>
#include <cuda_runtime.h>

template <int OP>
__global__ void __launch_bounds__(512, 1) k_alu(int iters, unsigned long long *cyc, double *sink, int seed) {
  double d[8];
  float f[8];
  int x[8];
  long long y[8];
#pragma unroll
  for (int i = 0; i < 8; ++i) {
    d[i] = 1.0 + 1e-9 * (threadIdx.x + i + seed);
    f[i] = 1.0f + 1e-6f * (threadIdx.x + i);
    x[i] = (int)threadIdx.x * 7 + i + seed;
    y[i] = x[i];
  }
  __syncthreads();
  long long t0 = clock64();
  for (int it = 0; it < iters; ++it) {
#pragma unroll
    for (int i = 0; i < 8; ++i) {
      if (OP == 0) d[i] = fma(d[i], 0.999999, 1e-7);                       // DFMA
      if (OP == 1) d[i] = d[i] + 1e-7;                                      // DADD
      if (OP == 2) f[i] = fmaf(f[i], 0.999999f, 1e-7f);                     // FFMA
      if (OP == 3) { d[i] = (double)x[i]; x[i] = x[i] + 1 + (int)(d[i] == 0.0); }   // I2F.F64 (+IADD)
      if (OP == 4) { f[i] = (float)x[i]; x[i] = x[i] + 1 + (int)(f[i] == 0.0f); }   // I2F.F32 (+IADD)
      if (OP == 5) { d[i] = (double)f[i]; f[i] = f[i] + (float)(d[i] == 0.0); }     // F2F.F64.F32 (+FADD)
      if (OP == 6) { f[i] = (float)d[i]; d[i] = d[i] + (double)(f[i] == 0.0f); }    // F2F.F32.F64 (+DADD)
      if (OP == 7) x[i] = x[i] * 257 + 3;                                   // IMAD
      if (OP == 8) y[i] = (long long)x[i] * 65536 + y[i];                    // IMAD.WIDE
      if (OP == 9) d[i] = __longlong_as_double(y[i] + 0x4338000000000000LL) - 6755399441055744.0 + d[i];   // magic i64->f64
    }
  }
  __syncthreads();
  long long t1 = clock64();
  if (threadIdx.x == 0) atomicAdd(cyc, (unsigned long long)(t1 - t0));
  double s = 0;
#pragma unroll
  for (int i = 0; i < 8; ++i) s += d[i] + f[i] + x[i] + (double)y[i];
  if (s == 12345.678) sink[0] = s;
}

template <int OP>
static void run(const char *name) {
  unsigned long long *cyc;
  double *sink;
  cudaMalloc(&cyc, 8);
  cudaMalloc(&sink, 8);
  const int iters = 2048;
  for (int rep = 0; rep < 2; ++rep) {
    cudaMemset(cyc, 0, 8);
    k_alu<OP><<<148, 512>>>(iters, cyc, sink, rep);
    cudaDeviceSynchronize();
  }
  unsigned long long c = 0;
  cudaMemcpy(&c, cyc, 8, cudaMemcpyDeviceToHost);
  const double per_sm = (double)c / 148.0;
  printf("%-14s %6.1f ops/clk/SM\n", name, (double)iters * 8 * 512 / per_sm);
  cudaFree(cyc);
  cudaFree(sink);
}

int main() {
  run<0>("DFMA");
  run<1>("DADD");
  run<2>("FFMA");
  run<3>("I2F.F64+IADD");
  run<4>("I2F.F32+IADD");
  run<5>("F2F.F64.F32+");
  run<6>("F2F.F32.F64+");
  run<7>("IMAD");
  run<8>("IMAD.WIDE");
  run<9>("magic i64->f64");
  return 0;
}
