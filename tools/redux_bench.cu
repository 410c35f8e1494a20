#include <cstdio>
__global__ void k(unsigned *out, long long *cyc, int mode) {
  unsigned v = threadIdx.x * 2654435761u;
  double d = threadIdx.x * 0.37;
  long long t0 = clock64();
  for (int i = 0; i < 1000; ++i) {
    if (mode == 0) v = __reduce_max_sync(0xffffffffu, v) + i;
    else if (mode == 1) { for (int o = 16; o; o >>= 1) v = max(v, __shfl_xor_sync(0xffffffffu, v, o)); v += i; }
    else if (mode == 2) { for (int o = 16; o; o >>= 1) d = fmax(d, __shfl_xor_sync(0xffffffffu, d, o)); d += 1.0; }
    else if (mode == 3) { v = __shfl_sync(0xffffffffu, v, (v + i) & 31) + 1; }
    else if (mode == 4) { d = 1.0 / (d + 1.0); }
    else if (mode == 5) { d = fma(d, 1.0000001, 0.5); }
  }
  long long t1 = clock64();
  if (threadIdx.x == 0) *cyc = (t1 - t0) / 1000;
  out[threadIdx.x] = v + (unsigned)d;
}
int main() {
  unsigned *o; long long *c, h;
  cudaMalloc(&o, 4096); cudaMalloc(&c, 8);
  const char *nm[] = {"redux.max.u32", "5x shfl+max u32", "5x shfl+fmax f64", "shfl idx", "f64 1/x", "dfma chain"};
  for (int m = 0; m < 6; ++m) {
    k<<<1, 32>>>(o, c, m); cudaDeviceSynchronize();
    cudaMemcpy(&h, c, 8, cudaMemcpyDeviceToHost);
    printf("%-20s %lld cycles\n", nm[m], h);
  }
}
