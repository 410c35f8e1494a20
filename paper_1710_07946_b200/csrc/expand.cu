// expand.cu — rectangular generators (NEXT-3): greedy expansion of the column set of a k x g
// submatrix C_g = R[:, J] of R = W[I, :] to k x l (Alg D.4 "algrup").  The column
// b appended at each step maximizes v2(C_g | b)^2 = v2(C_g)^2 (1 + b^T (C_g C_g^T)^{-1} b)
// (eq. eqbun): score_j = ||L^{-1} b_j||^2 with L L^T = C_g C_g^T.  Per step: k_exp_chol (one
// CTA: Gram matrix + Cholesky in fp64), k_exp_scores (one thread per column: forward
// substitution with L in shared memory), k_exp_pick (one CTA: max, then the smallest column
// with score >= (1 - tau) max, reading C11).  R is gathered once (k x n fp64, row-major).
#include "kernels.cuh"

namespace lra {

// R[s][j] = W[I[s], j]  (k x n row-major)
__global__ void k_exp_gather(OpView op, const int64_t *I, int k, double *R) {
  const int s = blockIdx.y;
  for (int64_t j = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; j < op.n; j += (int64_t)gridDim.x * blockDim.x)
    R[(int64_t)s * op.n + j] = op.at(I[s], j);
}

// L (k x k, row-major, lower) with L L^T = C C^T, C = R[:, J[0..g)]; ok[0] = 0 if not SPD
__global__ void __launch_bounds__(256) k_exp_chol(const double *R, int64_t n, int k, const int64_t *J, int g,
                                                  double *L, int *ok, const int *stop) {
  extern __shared__ double Ms[];          // k x k
  if (stop && *stop) return;
  for (int e = threadIdx.x; e < k * k; e += blockDim.x) {
    const int a = e / k, b = e % k;
    double acc = 0.0;
    if (b <= a)
      for (int c = 0; c < g; ++c) acc = fma(R[(int64_t)a * n + J[c]], R[(int64_t)b * n + J[c]], acc);
    Ms[e] = acc;
  }
  __syncthreads();
  if (threadIdx.x == 0) {                  // left-looking Cholesky (k <= 128: serial is fine)
    int good = 1;
    for (int j = 0; j < k && good; ++j) {
      double d = Ms[j * k + j];
      for (int t = 0; t < j; ++t) d = fma(-Ms[j * k + t], Ms[j * k + t], d);
      if (!(d > 0.0)) { good = 0; break; }
      const double ljj = sqrt(d);
      Ms[j * k + j] = ljj;
      for (int i = j + 1; i < k; ++i) {
        double v = Ms[i * k + j];
        for (int t = 0; t < j; ++t) v = fma(-Ms[i * k + t], Ms[j * k + t], v);
        Ms[i * k + j] = v / ljj;
      }
    }
    ok[0] = good;
  }
  __syncthreads();
  for (int e = threadIdx.x; e < k * k; e += blockDim.x) L[e] = (e % k <= e / k) ? Ms[e] : 0.0;
}

// score[j] = ||L^{-1} R[:, j]||^2 (-1 for the columns already chosen)
__global__ void __launch_bounds__(128) k_exp_scores(const double *R, int64_t n, int k, const double *L,
                                                    const int64_t *J, int g, double *score, const int *stop) {
  extern __shared__ double Ls[];
  if (stop && *stop) return;
  for (int e = threadIdx.x; e < k * k; e += blockDim.x) Ls[e] = L[e];
  __syncthreads();
  const int64_t j = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (j >= n) return;
  double z[128];
  double sc = 0.0;
  for (int i = 0; i < k; ++i) {
    double v = R[(int64_t)i * n + j];
    for (int t = 0; t < i; ++t) v = fma(-Ls[i * k + t], z[t], v);
    z[i] = v / Ls[i * k + i];
    sc = fma(z[i], z[i], sc);
  }
  for (int c = 0; c < g; ++c)
    if (J[c] == j) sc = -1.0;
  score[j] = sc;
}

// J[g] <- smallest j with score[j] >= (1 - tau) max
__global__ void __launch_bounds__(1024) k_exp_pick(const double *score, int64_t n, double tau, int64_t *J, int g,
                                                   const int *stop) {
  __shared__ double red[32];
  if (stop && *stop) return;
  __shared__ unsigned long long ri[32];
  double mx = -INFINITY;
  for (int64_t j = threadIdx.x; j < n; j += 1024) mx = fmax(mx, score[j]);
  mx = warp_max(mx);
  if ((threadIdx.x & 31) == 0) red[threadIdx.x >> 5] = mx;
  __syncthreads();
  mx = -INFINITY;
  for (int w = 0; w < 32; ++w) mx = fmax(mx, red[w]);
  const double thr = (1.0 - tau) * mx;
  unsigned long long best = ~0ull;
  for (int64_t j = threadIdx.x; j < n; j += 1024)
    if (score[j] >= thr && (unsigned long long)j < best) best = (unsigned long long)j;
  for (int o = 16; o > 0; o >>= 1) {
    const unsigned long long b2 = __shfl_xor_sync(0xffffffffu, best, o);
    best = b2 < best ? b2 : best;
  }
  __syncthreads();
  if ((threadIdx.x & 31) == 0) ri[threadIdx.x >> 5] = best;
  __syncthreads();
  if (threadIdx.x == 0) {
    unsigned long long b = ~0ull;
    for (int w = 0; w < 32; ++w) b = ri[w] < b ? ri[w] : b;
    J[g] = (int64_t)b;
  }
}

cudaError_t launch_expand_columns(const OpView &op, const int64_t *I, int k, int64_t *J, int g0, int l, double tau,
                                  void *scratch, int *ok, cudaStream_t st, int *nlaunch, Prof *pf) {
  double *R = reinterpret_cast<double *>(scratch);
  double *L = R + (size_t)k * op.n;
  double *score = L + (size_t)k * k;
  pf->begin("k_expand", st);
  k_exp_gather<<<dim3(32, (unsigned)k), 256, 0, st>>>(op, I, k, R);
  cudaError_t e = cudaGetLastError();
  int nl = 1;
  const size_t sm = (size_t)k * k * 8;
  cudaFuncSetAttribute(k_exp_chol, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)sm);
  cudaFuncSetAttribute(k_exp_scores, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)sm);
  for (int g = g0; g < l && e == cudaSuccess; ++g) {
    k_exp_chol<<<1, 256, sm, st>>>(R, op.n, k, J, g, L, ok, nullptr);
    k_exp_scores<<<(unsigned)((op.n + 127) / 128), 128, sm, st>>>(R, op.n, k, L, J, g, score, nullptr);
    k_exp_pick<<<1, 1024, 0, st>>>(score, op.n, tau, J, g, nullptr);
    nl += 3;
    e = cudaGetLastError();
  }
  pf->end(st);
  *nlaunch += nl;
  return e;
}

// ---------------------------------------------------------------- greedy contraction
// Def defgrdc: remove from C_g = R[:, J[0..g)] the column of minimal leverage
// ||L^{-1} c_j||^2 (L L^T = C_g C_g^T), ties: the smallest slot within (1 + tau) min; the other
// slots keep their order.  lev[t] for the g slots (thread per slot, the k_exp_scores arithmetic).
__global__ void __launch_bounds__(128) k_con_scores(const double *R, int64_t n, int k, const double *L,
                                                    const int64_t *J, int g, double *lev, const int *stop) {
  extern __shared__ double Ls[];
  if (stop && *stop) return;
  for (int e = threadIdx.x; e < k * k; e += blockDim.x) Ls[e] = L[e];
  __syncthreads();
  const int t = blockIdx.x * blockDim.x + threadIdx.x;
  if (t >= g) return;
  const int64_t j = J[t];
  double z[128];
  double sc = 0.0;
  for (int i = 0; i < k; ++i) {
    double v = R[(int64_t)i * n + j];
    for (int c = 0; c < i; ++c) v = fma(-Ls[i * k + c], z[c], v);
    z[i] = v / Ls[i * k + i];
    sc = fma(z[i], z[i], sc);
  }
  lev[t] = sc;
}

// one thread: remove the slot; in refinement mode (stop != null) removing the last slot (the
// column just appended) is the fixed point: set *stop.
__global__ void k_con_pick(const double *lev, int g, double tau, int64_t *J, int *stop) {
  if (stop && *stop) return;
  double mn = INFINITY;
  for (int t = 0; t < g; ++t) mn = fmin(mn, lev[t]);
  const double thr = (1.0 + tau) * mn;
  int ts = g - 1;
  for (int t = 0; t < g; ++t)
    if (lev[t] <= thr) { ts = t; break; }
  if (stop && ts == g - 1) { *stop = 1; return; }
  for (int t = ts; t + 1 < g; ++t) J[t] = J[t + 1];
}

// count of cycles that changed J (refinement diagnostics)
__global__ void k_con_count(const int *stop, int *changed) {
  if (!*stop) ++*changed;
}

cudaError_t launch_contract_columns(const OpView &op, const int64_t *I, int k, int64_t *J, int g0, int l, double tau,
                                    void *scratch, int *ok, cudaStream_t st, int *nlaunch, Prof *pf) {
  double *R = reinterpret_cast<double *>(scratch);
  double *L = R + (size_t)k * op.n;
  double *lev = L + (size_t)k * k;
  pf->begin("k_contract", st);
  k_exp_gather<<<dim3(32, (unsigned)k), 256, 0, st>>>(op, I, k, R);
  cudaError_t e = cudaGetLastError();
  int nl = 1;
  const size_t sm = (size_t)k * k * 8;
  cudaFuncSetAttribute(k_exp_chol, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)sm);
  cudaFuncSetAttribute(k_con_scores, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)sm);
  for (int g = g0; g > l && e == cudaSuccess; --g) {
    k_exp_chol<<<1, 256, sm, st>>>(R, op.n, k, J, g, L, ok, nullptr);
    k_con_scores<<<(unsigned)((g + 127) / 128), 128, sm, st>>>(R, op.n, k, L, J, g, lev, nullptr);
    k_con_pick<<<1, 1, 0, st>>>(lev, g, tau, J, nullptr);
    nl += 3;
    e = cudaGetLastError();
  }
  pf->end(st);
  *nlaunch += nl;
  return e;
}

// p = 1 expand-contract cycles on J (l slots; the buffer holds l + 1): stop / changed are
// device ints (zeroed by the caller); every launch after the fixed point is a no-op.
cudaError_t launch_refine_columns(const OpView &op, const int64_t *I, int k, int64_t *J, int l, int cycles,
                                  double tau, void *scratch, int *ok, int *stop, int *changed, cudaStream_t st,
                                  int *nlaunch, Prof *pf) {
  double *R = reinterpret_cast<double *>(scratch);
  double *L = R + (size_t)k * op.n;
  double *score = L + (size_t)k * k;
  pf->begin("k_refine", st);
  k_exp_gather<<<dim3(32, (unsigned)k), 256, 0, st>>>(op, I, k, R);
  cudaError_t e = cudaGetLastError();
  int nl = 1;
  const size_t sm = (size_t)k * k * 8;
  cudaFuncSetAttribute(k_exp_chol, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)sm);
  cudaFuncSetAttribute(k_exp_scores, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)sm);
  cudaFuncSetAttribute(k_con_scores, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)sm);
  for (int c = 0; c < cycles && e == cudaSuccess; ++c) {
    k_exp_chol<<<1, 256, sm, st>>>(R, op.n, k, J, l, L, ok, stop);
    k_exp_scores<<<(unsigned)((op.n + 127) / 128), 128, sm, st>>>(R, op.n, k, L, J, l, score, stop);
    k_exp_pick<<<1, 1024, 0, st>>>(score, op.n, tau, J, l, stop);
    k_exp_chol<<<1, 256, sm, st>>>(R, op.n, k, J, l + 1, L, ok, stop);
    k_con_scores<<<(unsigned)((l + 1 + 127) / 128), 128, sm, st>>>(R, op.n, k, L, J, l + 1, score, stop);
    k_con_pick<<<1, 1, 0, st>>>(score, l + 1, tau, J, stop);
    k_con_count<<<1, 1, 0, st>>>(stop, changed);
    nl += 7;
    e = cudaGetLastError();
  }
  pf->end(st);
  *nlaunch += nl;
  return e;
}

}  // namespace lra
