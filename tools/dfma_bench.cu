// DFMA throughput (many independent chains) and dependent latency on one GPU (diagnostics).
#include <cstdio>
#include <cuda_runtime.h>
template <int CH>
__global__ void k_thr(double *out, int iters, double a, double b) {
  double x[CH];
  for (int c = 0; c < CH; ++c) x[c] = threadIdx.x + c;
  for (int i = 0; i < iters; ++i)
#pragma unroll
    for (int c = 0; c < CH; ++c) x[c] = fma(x[c], a, b);
  double s = 0;
  for (int c = 0; c < CH; ++c) s += x[c];
  if (s == 12345.678) out[0] = s;
}
__global__ void k_lat(double *out, int iters, double a, double b, long long *cyc) {
  double x = threadIdx.x;
  long long t0 = clock64();
  for (int i = 0; i < iters; ++i) x = fma(x, a, b);
  long long t1 = clock64();
  if (threadIdx.x == 0) cyc[0] = t1 - t0;
  if (x == 12345.678) out[0] = x;
}
int main() {
  double *out; long long *cyc; cudaMalloc(&out, 8); cudaMalloc(&cyc, 8);
  int sms; cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, 0);
  cudaEvent_t e0, e1; cudaEventCreate(&e0); cudaEventCreate(&e1);
  const int iters = 20000;
  for (int blocks_per_sm : {1, 2, 4, 8}) {
    k_thr<8><<<sms * blocks_per_sm, 256>>>(out, 10, 1.0000001, 1e-9);
    cudaEventRecord(e0);
    k_thr<8><<<sms * blocks_per_sm, 256>>>(out, iters, 1.0000001, 1e-9);
    cudaEventRecord(e1); cudaEventSynchronize(e1);
    float ms; cudaEventElapsedTime(&ms, e0, e1);
    double flops = 2.0 * 8 * iters * 256.0 * sms * blocks_per_sm;
    printf("{\"dfma_tflops\": %.2f, \"warps_per_sm\": %d}\n", flops / ms / 1e9, 8 * blocks_per_sm);
  }
  k_lat<<<1, 32>>>(out, iters, 1.0000001, 1e-9, cyc);
  long long c; cudaMemcpy(&c, cyc, 8, cudaMemcpyDeviceToHost);
  printf("{\"dfma_dependent_latency_clk\": %.2f}\n", (double)c / iters);
  return 0;
}
