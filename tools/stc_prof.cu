// stc_prof.cu — per-role phase counters of k_sketch_tc (config-2 shape, fp32 W 4096 x 4096,
// lbar 48): builds the kernel file with STC_PROF=1 and prints average cycles per K-step.
//   nvcc -gencode arch=compute_100a,code=sm_100a -O3 -std=c++17 --expt-relaxed-constexpr -Iinclude \
//        -DSTC_PROF=1 -o tools/stc_prof tools/stc_prof.cu
#include "../paper_1710_07946_b200/csrc/sketch_tc.cu"

#include <cstdio>
#include <random>
#include <vector>

int main(int argc, char **argv) {
  const int64_t m = 4096, n = 4096, lb = argc > 1 ? atoi(argv[1]) : 48;
  std::vector<float> W(m * n);
  std::vector<double> Om(n * lb);
  std::mt19937 g(1);
  std::normal_distribution<float> N(0.f, 1.f);
  for (auto &x : W) x = N(g);
  for (auto &x : Om) x = (double)N(g);
  float *dW;
  double *dO, *dY;
  cudaMalloc(&dW, m * n * 4);
  cudaMalloc(&dO, n * lb * 8);
  cudaMalloc(&dY, m * lb * 8);
  cudaMemcpy(dW, W.data(), m * n * 4, cudaMemcpyHostToDevice);
  cudaMemcpy(dO, Om.data(), n * lb * 8, cudaMemcpyHostToDevice);
  lra::SketchArgs a{};
  a.kind = LRA_MUL_GAUSSIAN;
  a.dtype = LRA_F32;
  a.m = m;
  a.n = n;
  a.lbar = lb;
  a.ldw = m;
  a.w = dW;
  a.y = dY;
  a.ldy = m;
  const size_t bytes = lra::sketch_tc_scratch_bytes(m, n, lb, 1);
  void *scr;
  cudaMalloc(&scr, bytes);
  cudaMemset(scr, 0, bytes);
  lra::Prof pf;
  for (int rep = 0; rep < 3; ++rep) {
    unsigned long long z[16] = {};
    cudaMemcpyToSymbol(lra::g_stc_cyc, z, sizeof(z));
    static unsigned long long zt[1024][4];
    cudaMemcpyToSymbol(lra::g_stc_t, zt, sizeof(zt));
    cudaEvent_t e0, e1;
    cudaEventCreate(&e0);
    cudaEventCreate(&e1);
    cudaEventRecord(e0);
    cudaError_t e = lra::launch_sketch_tc(a, 1, dO, n, scr, bytes, 0, &pf);
    cudaEventRecord(e1);
    cudaError_t e2 = cudaDeviceSynchronize();
    float ms = 0;
    cudaEventElapsedTime(&ms, e0, e1);
    unsigned long long c[16];
    cudaMemcpyFromSymbol(c, lra::g_stc_cyc, sizeof(c));
    const double ks = (double)c[10];
    printf("launch %s / %s  %.1f us  K-steps %llu\n", cudaGetErrorString(e), cudaGetErrorString(e2), ms * 1e3, c[10]);
    const char *nm[10] = {"dig wait W", "dig wait A-empty", "dig compute+store", "mma wait A", "mma wait B",
                          "mma issue", "prod wait W-empty", "prod wait B-empty", "epi wait acc", "epi work"};
    for (int k = 0; k < 10; ++k) printf("  %-20s %10.1f cycles per K-step\n", nm[k], (double)c[k] / (ks > 0 ? ks : 1));
    int P = 0;
    cudaDeviceGetAttribute(&P, cudaDevAttrMultiProcessorCount, 0);
    unsigned long long T[1024][4];
    cudaMemcpyFromSymbol(T, lra::g_stc_t, sizeof(T));
    unsigned long long t0 = ~0ull, tmaxs = 0, tmaxe = 0, tmine = ~0ull;
    int ncta = 0;
    while (ncta < 1024 && T[ncta][0] != 0) ++ncta;
    P = ncta;
    for (int c = 0; c < P; ++c) {
      t0 = T[c][0] < t0 ? T[c][0] : t0;
      tmaxs = T[c][0] > tmaxs ? T[c][0] : tmaxs;
      tmaxe = T[c][2] > tmaxe ? T[c][2] : tmaxe;
      tmine = T[c][2] < tmine ? T[c][2] : tmine;
    }
    printf("  CTA start spread %.1f us, first end %.1f us, last end %.1f us (from first start)\n", (tmaxs - t0) * 1e-3,
           (tmine - t0) * 1e-3, (tmaxe - t0) * 1e-3);
    if (rep == 2) {
      for (int c = 0; c < P; ++c) printf("%d:%.0f/%.0f%s", c, (T[c][1] - T[c][0]) * 1e-3, (T[c][2] - T[c][0]) * 1e-3, c % 12 == 11 ? "\n" : " ");
      printf("\n");
    }
    printf("  CTAs %d\n", P);
    printf("  per CTA: role loops %.0f cycles, last-arriver %.0f, alloc+init %.0f\n", (double)c[11] / P,
           (double)c[12] / P, (double)c[13] / P);
  }
  return 0;
}
