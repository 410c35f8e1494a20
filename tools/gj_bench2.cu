// Timing dissection of the Gauss-Jordan step structure (q=48, 512 threads).
#include <cstdio>
#include "../paper_1710_07946_b200/csrc/ca.cu"
using namespace lra;
template <int MODE>
__global__ void kgj(double *out, long long *cyc) {
  __shared__ CAShared sh;
  extern __shared__ double A[];
  const int q = 48, Q = 48, AS = 96, nt = 512;
  for (int e = threadIdx.x; e < q * AS; e += nt) A[e] = (e % 97) * 0.01 + 1.0;
  __syncthreads();
  const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5, nw = nt >> 5;
  long long t0 = clock64();
  unsigned long long used = 0;
  double acc = 0;
  for (int t = 0; t < q; ++t) {
    int p = t;
    if (MODE & 1) {   // pivot search
      unsigned long long key = 0ull; int arow = 0x7fffffff;
      for (int a = lane; a < q; a += 32) {
        if ((used >> a) & 1ull) continue;
        const double v = fabs(A[a * AS + t]);
        const unsigned long long k = dkey(v);
        if (arow == 0x7fffffff || k > key) { key = k; arow = a; }
      }
      const unsigned long long mk = warp_max_key(key);
      p = (int)__reduce_min_sync(0xffffffffu, (key == mk && arow != 0x7fffffff) ? (unsigned)arow : 0xffffffffu);
      used |= 1ull << p;
    }
    const double d = A[p * AS + t];
    const double rd = (MODE & 2) ? 1.0 / d : d;
    double fa[4], pv[6];
#pragma unroll
    for (int k = 0; k < 4; ++k) { const int a = warp + k * nw; fa[k] = (a < q) ? A[a * AS + t] : 0.0; }
#pragma unroll
    for (int m = 0; m < 6; ++m) { const int b = lane + 32 * m; pv[m] = (b < AS) ? A[p * AS + b] * rd : 0.0; }
    if (MODE & 4) __syncthreads();
    if (MODE & 8) {
#pragma unroll
      for (int k = 0; k < 4; ++k) {
        const int a = warp + k * nw;
        if (a >= q) continue;
#pragma unroll
        for (int m = 0; m < 6; ++m) {
          const int b = lane + 32 * m;
          if (b >= AS) continue;
          double x;
          if (a == p) x = (b == t) ? 1.0 : pv[m];
          else x = (b == t) ? 0.0 : fma(-fa[k], pv[m], A[a * AS + b]);
          A[a * AS + b] = x;
        }
      }
    } else {
      for (int k = 0; k < 4; ++k) for (int m = 0; m < 6; ++m) acc += fa[k] * pv[m];
    }
    if (MODE & 16) __syncthreads();
  }
  long long t1 = clock64();
  if (tid == 0) *cyc = (t1 - t0) / q;
  if (acc == 12345.0) out[0] = acc;
}
template <int M> void run(double *dO, long long *dc) {
  kgj<M><<<1, 512, 48 * 96 * 8>>>(dO, dc);
  cudaDeviceSynchronize();
  long long c; cudaMemcpy(&c, dc, 8, cudaMemcpyDeviceToHost);
  printf("mode %2d: %lld cycles/step\n", M, c);
}
int main() {
  double *dO; long long *dc;
  cudaMalloc(&dO, 8); cudaMalloc(&dc, 8);
  run<0>(dO, dc); run<1>(dO, dc); run<2>(dO, dc); run<4>(dO, dc); run<16>(dO, dc); run<20>(dO, dc);
  run<8>(dO, dc); run<24>(dO, dc); run<28>(dO, dc); run<29>(dO, dc); run<31>(dO, dc);
  return 0;
}
