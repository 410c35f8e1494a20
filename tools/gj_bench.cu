// Microbenchmark of lra::gj_inverse (48x48, 512 threads): cycles per call, and an
// accuracy check of the result.  Build: nvcc -gencode arch=compute_100a,code=sm_100a -O3
#include <cstdio>
#include <cstdlib>
#include "../paper_1710_07946_b200/csrc/ca.cu"
using namespace lra;
__global__ void kgj(const double *G, double *out, long long *cyc, int q, int reps) {
  __shared__ CAShared sh;
  extern __shared__ double A[];
  const int Q = 48, AS = 2 * Q;
  long long tot = 0;
  for (int r = 0; r < reps; ++r) {
    for (int e = threadIdx.x; e < q * AS; e += blockDim.x) {
      int a = e / AS, b = e % AS;
      A[e] = b < Q ? (b < q ? G[a * q + b] : 0.0) : ((b - Q) == a ? 1.0 : 0.0);
    }
    __syncthreads();
    long long t0 = clock64();
    bool ok = gj_inverse(&sh, A, q, Q, AS, blockDim.x);
    __syncthreads();
    tot += clock64() - t0;
    if (!ok && threadIdx.x == 0) printf("singular\n");
  }
  for (int e = threadIdx.x; e < q * q; e += blockDim.x) {
    int t = e / q, j = e % q;
    out[t * q + j] = A[sh.piv[t] * AS + Q + j];
  }
  if (threadIdx.x == 0) *cyc = tot / reps;
}
int main() {
  const int q = 48;
  double *h = (double *)malloc(q * q * 8), *hi = (double *)malloc(q * q * 8);
  srand(1);
  for (int i = 0; i < q * q; ++i) h[i] = rand() / (double)RAND_MAX - 0.5;
  double *dG, *dO; long long *dc, c;
  cudaMalloc(&dG, q * q * 8); cudaMalloc(&dO, q * q * 8); cudaMalloc(&dc, 8);
  cudaMemcpy(dG, h, q * q * 8, cudaMemcpyHostToDevice);
  kgj<<<1, 512, q * 96 * 8>>>(dG, dO, dc, q, 20);
  printf("err %s\n", cudaGetErrorString(cudaDeviceSynchronize()));
  cudaMemcpy(&c, dc, 8, cudaMemcpyDeviceToHost);
  cudaMemcpy(hi, dO, q * q * 8, cudaMemcpyDeviceToHost);
  double mx = 0;
  for (int i = 0; i < q; ++i) for (int j = 0; j < q; ++j) {
    double s = 0; for (int k = 0; k < q; ++k) s += h[i * q + k] * hi[k * q + j];
    s -= (i == j); mx = fabs(s) > mx ? fabs(s) : mx;
  }
  printf("gj_inverse q=%d: %lld cycles/call (%.1f us @1.965GHz), max|G X - I| = %.3e\n", q, c, c / 1965.0, mx);
  return 0;
}
