#include <cstdio>
template <int M>
__global__ void k(double *out, long long *cyc, double a, double b) {
  double d = threadIdx.x * 0.37; float f = threadIdx.x * 0.1f; int iv = threadIdx.x; unsigned u = threadIdx.x;
  long long t0 = clock64();
#pragma unroll 1
  for (int i = 0; i < 4096; ++i) {
    if (M == 0) d = fma(d, a, b);
    if (M == 1) f = fmaf(f, (float)a, (float)b);
    if (M == 2) iv = iv * 3 + 1;
    if (M == 3) d = d + a;
    if (M == 4) u = __shfl_xor_sync(0xffffffffu, u, 1) + 1;
    if (M == 5) d = __shfl_xor_sync(0xffffffffu, d, 1) + 1.0;
    if (M == 6) u = __reduce_add_sync(0xffffffffu, u) & 31;
    if (M == 7) d = fmax(d, a) * b;
  }
  long long t1 = clock64();
  if (threadIdx.x == 0) *cyc = (t1 - t0) / 4096;
  out[threadIdx.x] = d + f + iv + u;
}
template <int M> void run(const char *nm, double *o, long long *c) {
  k<M><<<1, 32>>>(o, c, 1.0000001, 0.5); cudaDeviceSynchronize();
  long long h; cudaMemcpy(&h, c, 8, cudaMemcpyDeviceToHost);
  printf("%-22s %lld cycles\n", nm, h);
}
int main() {
  double *o; long long *c;
  cudaMalloc(&o, 4096); cudaMalloc(&c, 8);
  run<1>("ffma chain", o, c); run<0>("dfma chain", o, c); run<3>("dadd chain", o, c); run<2>("imad chain", o, c);
  run<4>("shfl u32 chain", o, c); run<5>("shfl f64 chain", o, c); run<6>("redux.add chain", o, c); run<7>("dmnmx+dmul chain", o, c);
}
