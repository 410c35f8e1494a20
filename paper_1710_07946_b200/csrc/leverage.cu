// leverage.cu — NEXT-4: SVD-based leverage scores (eq. eqlevsc with beta = 1) of
// the columns of a k x N block B (B = W[I,:], or B = W[:,J]^T for row scores) and the
// Exactly(l) sampling of Alg C.1 (algsmplex) — the subalgorithm of DMM08 that
// the paper runs inside C-A iterations (section ststc-alvrg).
//
// Scores: G = B B^T (k x k, fp64), its eigenpairs by the one-sided Jacobi nucleus kernel (for
// a symmetric PSD G the SVD is the eigendecomposition: Sr = U_r, TS = U_r Lambda_r^{-1}), then
// p_j = (1/r) sum_t (u_t . b_j)(u_t . b_j / lambda_t) = ||(V_r)_{j,:}||^2 / r, one thread per j.
// Sampling: one CTA, the sequential prefix sum P (the oracle's order), then per draw the
// smallest i with u P_{N-1} < P_i by binary search (reading C31); p == NULL means the uniform
// scores p_j = 1/N of section slrasmpav.  Expected(l) (Alg C.2):
// independent keep decisions u_j < min{1, l p_j} and an ordered compaction (reading C33).
#include "kernels.cuh"

namespace lra {

// B[s][j] (k x N row-major): side 0 -> W[I[s], j] (N = n), side 1 -> W[j, I[s]] (N = m)
__global__ void k_lev_gather(OpView op, const int64_t *I, int k, int side, double *B) {
  const int s = blockIdx.y;
  const int64_t N = side ? op.m : op.n;
  for (int64_t j = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; j < N; j += (int64_t)gridDim.x * blockDim.x)
    B[(int64_t)s * N + j] = side ? op.at(j, I[s]) : op.at(I[s], j);
}

// G[a + b k] = G[b + a k] = sum_j B[a][j] B[b][j]; one CTA per (a, b >= a)... per pair index
__global__ void __launch_bounds__(256) k_lev_gram(const double *B, int64_t N, int k, double *G) {
  const int a = blockIdx.x, b = blockIdx.y;
  if (b > a) return;
  __shared__ double red[8];
  double acc = 0.0;
  for (int64_t j = threadIdx.x; j < N; j += blockDim.x) acc = fma(B[(int64_t)a * N + j], B[(int64_t)b * N + j], acc);
  acc = warp_sum(acc);
  if ((threadIdx.x & 31) == 0) red[threadIdx.x >> 5] = acc;
  __syncthreads();
  if (threadIdx.x == 0) {
    double t = 0.0;
    for (int w = 0; w < 8; ++w) t += red[w];
    G[a + (int64_t)b * k] = t;
    G[b + (int64_t)a * k] = t;
  }
}

// p_j = (1/r) sum_t (Sr_t . b_j)(TS_t . b_j); Sr, TS: k x r column-major in shared memory
__global__ void __launch_bounds__(128) k_lev_scores(const double *B, int64_t N, int k, int r, const double *Sr,
                                                    const double *TS, const int32_t *status, double *p) {
  extern __shared__ double sm[];
  if (status && *status != LRA_OK) return;
  double *S = sm, *T = sm + (size_t)k * r;
  for (int e = threadIdx.x; e < k * r; e += blockDim.x) {
    S[e] = Sr[e];
    T[e] = TS[e];
  }
  __syncthreads();
  const int64_t j = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (j >= N) return;
  double acc = 0.0;
  for (int t = 0; t < r; ++t) {
    double z = 0.0, y = 0.0;
    for (int i = 0; i < k; ++i) {
      const double bij = B[(int64_t)i * N + j];
      z = fma(S[(size_t)t * k + i], bij, z);
      y = fma(T[(size_t)t * k + i], bij, y);
    }
    acc = fma(z, y, acc);
  }
  p[j] = acc / (double)r;
}

// Alg C.1 with the caller's uniforms: P = sequential prefix sums of p (thread 0), then each
// draw by binary search; d_t = 1 / sqrt(l p_{i_t})
__global__ void __launch_bounds__(256) k_lev_sample(const double *p, int64_t N, int l, const double *u, double *P,
                                                    int64_t *idx, double *dsc, const int32_t *status) {
  if (status && *status != LRA_OK) return;
  const double pu = 1.0 / (double)N;                  // p == NULL: uniform scores (section slrasmpav)
  if (threadIdx.x == 0) {
    double acc = 0.0;
    for (int64_t i = 0; i < N; ++i) {
      acc = __dadd_rn(acc, p ? p[i] : pu);
      P[i] = acc;
    }
  }
  __syncthreads();
  const double tot = P[N - 1];
  for (int t = threadIdx.x; t < l; t += blockDim.x) {
    const double x = __dmul_rn(u[t], tot);
    int64_t lo = 0, hi = N;                           // smallest i with P[i] > x
    while (lo < hi) {
      const int64_t mid = (lo + hi) >> 1;
      if (P[mid] > x) hi = mid; else lo = mid + 1;
    }
    if (lo > N - 1) lo = N - 1;
    idx[t] = lo;
    if (dsc) dsc[t] = 1.0 / sqrt((double)l * (p ? p[lo] : pu));
  }
}

// Alg C.2 (Expected(l), reading C33): j is kept iff u_j < min{1, l p_j} (fp64, the oracle's
// operations), the kept j compacted in ascending order by one CTA: per 1024-wide chunk a ballot
// per warp, an exclusive scan of the 32 warp counts, then the running offset.  count gets the
// number kept; idx / dsc receive the first min(count, cap) of them.
__global__ void __launch_bounds__(1024) k_sample_expected(const double *p, int64_t N, int l, const double *u,
                                                          int64_t cap, int64_t *idx, double *dsc, int64_t *count,
                                                          const int32_t *status) {
  if (status && *status != LRA_OK) return;
  __shared__ int wc[32];
  __shared__ int64_t base;
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  const double pu = 1.0 / (double)N;
  if (threadIdx.x == 0) base = 0;
  __syncthreads();
  for (int64_t c0 = 0; c0 < N; c0 += 1024) {
    const int64_t j = c0 + threadIdx.x;
    double pj = 0.0;
    bool keep = false;
    if (j < N) {
      pj = p ? p[j] : pu;
      keep = u[j] < fmin(1.0, __dmul_rn((double)l, pj));
    }
    const unsigned bal = __ballot_sync(0xffffffffu, keep);
    if (lane == 0) wc[warp] = __popc(bal);
    __syncthreads();
    if (warp == 0) {
      int v = wc[lane];
      for (int o = 1; o < 32; o <<= 1) {
        const int y = __shfl_up_sync(0xffffffffu, v, o);
        if (lane >= o) v += y;
      }
      wc[lane] = v;                                     // inclusive
    }
    __syncthreads();
    const int64_t b0 = base;
    if (keep) {
      const int64_t t = b0 + (warp ? wc[warp - 1] : 0) + __popc(bal & ((1u << lane) - 1u));
      if (t < cap) {
        idx[t] = j;
        if (dsc) dsc[t] = 1.0 / fmin(1.0, sqrt(__dmul_rn((double)l, pj)));
      }
    }
    __syncthreads();
    if (threadIdx.x == 0) base = b0 + wc[31];
    __syncthreads();
  }
  if (threadIdx.x == 0) *count = base;
}

size_t leverage_scratch_bytes(int k, int r, int64_t N) {
  return ((size_t)k * N + (size_t)k * k + 2 * (size_t)k * r) * 8 + 512;
}

cudaError_t launch_leverage_scores(const OpView &op, const int64_t *I, int k, int side, int r, double *p,
                                   int32_t *status, void *scratch, cudaStream_t st, int *nlaunch, Prof *pf) {
  const int64_t N = side ? op.m : op.n;
  double *B = reinterpret_cast<double *>(scratch);
  double *G = B + (size_t)k * N;
  double *Sr = G + (size_t)k * k;
  double *TS = Sr + (size_t)k * r;
  pf->begin("k_leverage", st);
  k_lev_gather<<<dim3(32, (unsigned)k), 256, 0, st>>>(op, I, k, side, B);
  k_lev_gram<<<dim3((unsigned)k, (unsigned)k), 256, 0, st>>>(B, N, k, G);
  cudaError_t e = cudaGetLastError();
  pf->end(st);
  if (e != cudaSuccess) return e;
  NucArgs na{};
  na.op = op;
  na.I = I;            // unused with Gd
  na.J = I;
  na.k = k;
  na.l = k;
  na.r = r;
  na.TS = TS;
  na.Sr = Sr;
  na.status = status;
  na.Gd = G;
  FacArgs fa{};        // no factors
  fa.k = k;
  fa.l = k;
  fa.r = r;
  int nl = 0;
  if ((e = launch_nucleus(na, fa, 1, st, &nl, pf)) != cudaSuccess) return e;
  const size_t sm = (size_t)2 * k * r * 8;
  e = cudaFuncSetAttribute(k_lev_scores, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)sm);
  if (e != cudaSuccess) return e;
  pf->begin("k_leverage", st);
  k_lev_scores<<<(unsigned)((N + 127) / 128), 128, sm, st>>>(B, N, k, r, Sr, TS, status, p);
  pf->end(st);
  *nlaunch += 3 + nl;
  return cudaGetLastError();
}

cudaError_t launch_sample_exactly(const double *p, int64_t N, int l, const double *u, double *P, int64_t *idx,
                                  double *dsc, const int32_t *status, cudaStream_t st, int *nlaunch, Prof *pf) {
  pf->begin("k_lev_sample", st);
  k_lev_sample<<<1, 256, 0, st>>>(p, N, l, u, P, idx, dsc, status);
  pf->end(st);
  *nlaunch += 1;
  return cudaGetLastError();
}

cudaError_t launch_sample_expected(const double *p, int64_t N, int l, const double *u, int64_t cap, int64_t *idx,
                                   double *dsc, int64_t *count, const int32_t *status, cudaStream_t st, int *nlaunch,
                                   Prof *pf) {
  pf->begin("k_lev_sample", st);
  k_sample_expected<<<1, 1024, 0, st>>>(p, N, l, u, cap, idx, dsc, count, status);
  pf->end(st);
  *nlaunch += 1;
  return cudaGetLastError();
}

}  // namespace lra
