// qrp.cu — NEXT-3: Householder QR with column pivoting as greedy column expansion (Alg D.3
// "alg1tor"), the first stage of the r-projective column selection of Alg 7.1
// ("algprjvlm").
//
// X = W[I, :] is gathered once as a k x n fp64 row-major matrix (row stride n: a thread owns
// columns, so every row access of a warp is coalesced).  One cooperative launch runs the q
// steps with one grid barrier per step:
//   (a) every CTA picks the pivot from the trailing squared norms of step g (the same fixed
//       reduction in every CTA, so all CTAs agree without another barrier): M = max, then the
//       smallest column with norm >= (1 - tau) M (reading C11);
//   (b) every CTA rebuilds the Householder vector v = x + sign(x0)||x|| e1 of the pivot's
//       trailing part and beta = 2 / v^T v in shared memory;
//   (c) each thread applies I - beta v v^T to its columns (v^T y and the updates in ascending
//       row order, separately rounded products and sums — the oracle's order, so pivots and
//       the reflected values are bit-identical), sets the pivot column to -sign(x0)||x|| e1,
//       and computes its columns' trailing norms of step g + 1 into the other norm buffer.
#include <cooperative_groups.h>

#include "kernels.cuh"

namespace lra {
namespace cg = cooperative_groups;

constexpr int QRP_NT = 256;

__global__ void k_qrp_gather(OpView op, const int64_t *I, int k, double *X) {
  const int s = blockIdx.y;
  for (int64_t j = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; j < op.n; j += (int64_t)gridDim.x * blockDim.x)
    X[(int64_t)s * op.n + j] = op.at(I[s], j);
}

struct QrpArgs {
  double *X;             // k x n row-major
  int64_t n;
  int k, q;
  double tau;
  double *nrm;           // 2 x n trailing squared norms (double-buffered by step parity)
  int64_t *piv;          // q pivots
  double *R;             // optional q x n column-major output (ld ldr)
  int64_t ldr;
  double *Rt;            // optional n x q column-major output
  int32_t *status;
};

__global__ void __launch_bounds__(QRP_NT) k_qrp(QrpArgs a) {
  cg::grid_group grid = cg::this_grid();
  extern __shared__ double v[];                  // k (Householder vector)
  __shared__ double s_red[QRP_NT / 32];
  __shared__ long long s_idx[QRP_NT / 32];
  __shared__ double s_beta, s_alpha;
  __shared__ long long s_p;
  __shared__ int s_bad;
  const int64_t n = a.n;
  const int k = a.k;
  const int64_t t0 = (int64_t)blockIdx.x * blockDim.x + threadIdx.x, stride = (int64_t)gridDim.x * blockDim.x;
  const int lane = threadIdx.x & 31, wid = threadIdx.x >> 5;
  // step-0 norms
  for (int64_t j = t0; j < n; j += stride) {
    double acc = 0.0;
    for (int i = 0; i < k; ++i) {
      const double x = a.X[(int64_t)i * n + j];
      acc = __dadd_rn(acc, __dmul_rn(x, x));
    }
    a.nrm[j] = acc;
  }
  grid.sync();
  // The pivot column of step g is overwritten only after the step's grid barrier: every CTA
  // reads it in (b) of the same step.
  int64_t pend = -1;
  int pend_g = 0;
  double pend_alpha = 0.0;
  auto flush = [&]() {
    if (pend >= 0) {
      a.X[(int64_t)pend_g * n + pend] = pend_alpha;
      for (int i = pend_g + 1; i < k; ++i) a.X[(int64_t)i * n + pend] = 0.0;
      pend = -1;
    }
  };
  for (int g = 0; g < a.q; ++g) {
    flush();
    const double *nr = a.nrm + (int64_t)(g & 1) * n;
    double *nw = a.nrm + (int64_t)((g + 1) & 1) * n;
    // ---- (a) pivot: max, then the smallest column inside the slack window
    double mx = -1.0;
    for (int64_t j = threadIdx.x; j < n; j += blockDim.x) mx = fmax(mx, nr[j]);
    for (int o = 16; o > 0; o >>= 1) mx = fmax(mx, __shfl_xor_sync(0xffffffffu, mx, o));
    if (lane == 0) s_red[wid] = mx;
    __syncthreads();
    if (threadIdx.x == 0) {
      double M = s_red[0];
      for (int w = 1; w < QRP_NT / 32; ++w) M = fmax(M, s_red[w]);
      s_red[0] = M;
      s_bad = !(M > 0.0) || !isfinite(M);
    }
    __syncthreads();
    const double M = s_red[0];
    if (s_bad) {
      if (blockIdx.x == 0 && threadIdx.x == 0) a.status[0] = LRA_ESINGULAR;
      return;                                     // every CTA sees the same M
    }
    const double thr = (1.0 - a.tau) * M;
    long long best = 0x7fffffffffffffffll;
    for (int64_t j = threadIdx.x; j < n; j += blockDim.x)
      if (nr[j] >= thr) { best = j; break; }     // ascending j per thread: the first is its smallest
    for (int o = 16; o > 0; o >>= 1) {
      const long long other = __shfl_xor_sync(0xffffffffu, best, o);
      best = other < best ? other : best;
    }
    __syncthreads();
    if (lane == 0) s_idx[wid] = best;
    __syncthreads();
    if (threadIdx.x == 0) {
      long long b = s_idx[0];
      for (int w = 1; w < QRP_NT / 32; ++w) b = s_idx[w] < b ? s_idx[w] : b;
      s_p = b;
    }
    __syncthreads();
    const int64_t p = s_p;
    // ---- (b) Householder vector of the pivot's trailing part
    for (int i = threadIdx.x; i < k - g; i += blockDim.x) v[i] = a.X[(int64_t)(g + i) * n + p];
    __syncthreads();
    if (threadIdx.x == 0) {
      const double alpha = sqrt(nr[p]);
      const double sgn = v[0] >= 0.0 ? 1.0 : -1.0;
      v[0] = __dadd_rn(v[0], __dmul_rn(sgn, alpha));
      double vtv = 0.0;
      for (int i = 0; i < k - g; ++i) vtv = __dadd_rn(vtv, __dmul_rn(v[i], v[i]));
      s_beta = __ddiv_rn(2.0, vtv);
      s_alpha = -sgn * alpha;
      if (blockIdx.x == 0) a.piv[g] = p;
    }
    __syncthreads();
    const double beta = s_beta;
    // ---- (c) apply the reflection to the owned columns; trailing norms of step g + 1
    for (int64_t j = t0; j < n; j += stride) {
      if (nr[j] < 0.0) {                          // chosen earlier: trailing part is zero
        nw[j] = -1.0;
        continue;
      }
      if (j == p) {
        pend = j;
        pend_g = g;
        pend_alpha = s_alpha;
        nw[j] = -1.0;
        continue;
      }
      double w = 0.0;
      for (int i = 0; i < k - g; ++i) w = __dadd_rn(w, __dmul_rn(v[i], a.X[(int64_t)(g + i) * n + j]));
      const double t = __dmul_rn(beta, w);
      double acc = 0.0;
      for (int i = 0; i < k - g; ++i) {
        double *x = a.X + (int64_t)(g + i) * n + j;
        const double y = __dsub_rn(*x, __dmul_rn(t, v[i]));
        *x = y;
        if (i > 0) acc = __dadd_rn(acc, __dmul_rn(y, y));
      }
      nw[j] = acc;
    }
    grid.sync();
  }
  flush();
  // ---- outputs: the first q rows (R: q x n column-major, Rt: n x q column-major)
  for (int64_t j = t0; j < n; j += stride)
    for (int t = 0; t < a.q; ++t) {
      const double x = a.X[(int64_t)t * n + j];
      if (a.R) a.R[j * a.ldr + t] = x;
      if (a.Rt) a.Rt[(int64_t)t * n + j] = x;
    }
}

size_t qrp_scratch_bytes(int k, int64_t n) { return ((size_t)k * n + 2 * (size_t)n) * 8 + 256; }

cudaError_t launch_qrp(const OpView &op, const int64_t *I, int k, int q, double tau, int64_t *piv, double *R,
                       int64_t ldr, double *Rt, int32_t *status, void *scratch, cudaStream_t st, int *nlaunch,
                       Prof *pf) {
  QrpArgs a{};
  a.X = reinterpret_cast<double *>(scratch);
  a.nrm = a.X + (size_t)k * op.n;
  a.n = op.n;
  a.k = k;
  a.q = q;
  a.tau = tau;
  a.piv = piv;
  a.R = R;
  a.ldr = ldr;
  a.Rt = Rt;
  a.status = status;
  pf->begin("k_qrp", st);
  k_qrp_gather<<<dim3(32, (unsigned)k), 256, 0, st>>>(op, I, k, a.X);
  cudaError_t e = cudaGetLastError();
  if (e != cudaSuccess) return e;
  int dev = 0, sms = 0, per_sm = 0;
  cudaGetDevice(&dev);
  cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev);
  const size_t smem = (size_t)k * 8;
  e = cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, k_qrp, QRP_NT, smem);
  if (e != cudaSuccess) return e;
  int64_t grid = (op.n + QRP_NT - 1) / QRP_NT;
  if (grid > (int64_t)sms * per_sm) grid = (int64_t)sms * per_sm;
  if (grid > sms) grid = sms;
  cudaLaunchConfig_t cfg = {};
  cfg.gridDim = dim3((unsigned)grid);
  cfg.blockDim = dim3(QRP_NT);
  cfg.dynamicSmemBytes = smem;
  cfg.stream = st;
  cudaLaunchAttribute attr[1];
  attr[0].id = cudaLaunchAttributeCooperative;
  attr[0].val.cooperative = 1;
  cfg.attrs = attr;
  cfg.numAttrs = 1;
  e = cudaLaunchKernelEx(&cfg, k_qrp, a);
  pf->end(st);
  *nlaunch += 2;
  return e;
}

}  // namespace lra
