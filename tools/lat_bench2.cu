#include <cstdio>
template <int M>
__global__ void k(double *out, long long *cyc, double a, double b) {
  double d = threadIdx.x * 0.37 + 1.0; unsigned u = threadIdx.x;
  __shared__ double sm[64];
  sm[threadIdx.x] = d;
  __syncthreads();
  long long t0 = clock64();
#pragma unroll 1
  for (int i = 0; i < 256; ++i) {
#pragma unroll
    for (int j = 0; j < 16; ++j) {
      if (M == 0) d = fma(d, a, b);
      if (M == 1) d = __shfl_xor_sync(0xffffffffu, d, 1);
      if (M == 2) u = __reduce_add_sync(0xffffffffu, u);
      if (M == 3) d = rsqrt(d);
      if (M == 4) d = __drcp_rn(d);
      if (M == 5) d = 1.0 / d;
      if (M == 6) d = sqrt(d);
      if (M == 7) d = sm[(int)d & 31];
      if (M == 8) __syncthreads();
      if (M == 9) d = d + a;
    }
  }
  long long t1 = clock64();
  if (threadIdx.x == 0) *cyc = (t1 - t0) * 100 / (256 * 16);
  out[threadIdx.x] = d + u;
}
template <int M> void run(const char *nm, double *o, long long *c, int nt) {
  k<M><<<1, nt>>>(o, c, 1.0000001, 0.5); cudaDeviceSynchronize();
  long long h; cudaMemcpy(&h, c, 8, cudaMemcpyDeviceToHost);
  printf("%-16s (%4d thr) %6.2f cycles/op\n", nm, nt, h / 100.0);
}
int main() {
  double *o; long long *c;
  cudaMalloc(&o, 8192); cudaMalloc(&c, 8);
  run<0>("dfma", o, c, 32); run<9>("dadd", o, c, 32); run<1>("shfl f64", o, c, 32); run<2>("redux.add", o, c, 32);
  run<3>("rsqrt f64", o, c, 32); run<4>("drcp_rn", o, c, 32); run<5>("1/x f64", o, c, 32); run<6>("sqrt f64", o, c, 32);
  run<7>("lds dep", o, c, 32); run<8>("syncthreads", o, c, 32); run<8>("syncthreads", o, c, 512); run<8>("syncthreads", o, c, 1024);
}
