// residual.cu — the a-posteriori check rho = ||W - CUR||_F / ||W||_F (eq. eqcur0,
// P:1153-1155) with CUR = A*B, A m x r, B r x n (fp64).
//
// k_residual: one CTA per 128 x 128 tile of W (column-major).  The rank-r product is
// accumulated in fp64 registers (8 x 8 per thread, DFMA) from A/B panels staged in shared
// memory 16 k-columns at a time (A and B stay L2-resident across tiles); the epilogue
// streams the W tile once with 16-byte loads, forms d = W - AB and accumulates sum d^2
// and sum W^2 in fp64.  Per-tile partials are summed in a fixed order by k_reduce, so the
// result is deterministic.  (PRECISE mode; the tensor-core FAST mode is not in this build.)
#include "kernels.cuh"

namespace lra {

constexpr int RS_T = 128;    // tile edge
constexpr int RS_KC = 16;    // k-chunk
constexpr int RS_NT = 256;


__device__ __forceinline__ void cp_async16(void *smem, const void *gmem) {
  const unsigned sa = (unsigned)__cvta_generic_to_shared(smem);
  asm volatile("cp.async.cg.shared.global [%0], [%1], 16;\n" ::"r"(sa), "l"(gmem));
}
__device__ __forceinline__ void cp_async_wait_all() { asm volatile("cp.async.wait_all;\n" ::: "memory"); }

// grid: (tiles_m * tiles_n, nb).  Thread (tx, ty) owns rows tx + 16 i and columns ty*8 + j
// (i, j < 8): the A-panel reads of a warp are 16 consecutive doubles (conflict-free) and the
// W reads are 64-byte column segments.  For fp32 W the whole 128 x 128 tile is prefetched
// into shared memory with cp.async at the start, overlapping the fp64 FMA loop.
template <typename TW>
__global__ void __launch_bounds__(RS_NT) k_residual(ResArgs a) {
  __shared__ __align__(16) double As[RS_KC][RS_T];
  __shared__ __align__(16) double Bs[RS_KC][RS_T];
  __shared__ double red[2][RS_NT / 32];
  extern __shared__ __align__(16) float Wsm[];          // [RS_T cols][RS_T rows] (fp32 only)
  const int64_t b = blockIdx.y;
  const int64_t tile = blockIdx.x;
  if (a.status && a.status[b] != LRA_OK) return;
  const int64_t tm = tile % a.tiles_m, tn = tile / a.tiles_m;
  const int64_t row0 = tm * RS_T, col0 = tn * RS_T;
  const int tid = threadIdx.x, tx = tid & 15, ty = tid >> 4;
  const double *A = a.A + b * a.a_stride;
  const double *B = a.B + b * a.b_stride;
  const TW *W = reinterpret_cast<const TW *>(a.w) + b * a.w_stride;
  constexpr bool PRE = sizeof(TW) == 4;
  const bool full = row0 + RS_T <= a.m && col0 + RS_T <= a.n && (a.ldw & 3) == 0 &&
                    ((reinterpret_cast<uintptr_t>(W) & 15) == 0);
  if (PRE && full) {
    // 128 columns x 512 B, 16-byte chunks: chunk e -> column e / 32, rows 4 (e % 32) ..
    for (int e = tid; e < RS_T * (RS_T / 4); e += RS_NT) {
      const int col = e >> 5, r4 = (e & 31) * 4;
      cp_async16(&Wsm[col * RS_T + r4], W + (col0 + col) * a.ldw + row0 + r4);
    }
    asm volatile("cp.async.commit_group;\n" ::: "memory");
  }
  double acc[8][8];
#pragma unroll
  for (int x = 0; x < 8; ++x)
#pragma unroll
    for (int y = 0; y < 8; ++y) acc[x][y] = 0.0;
  for (int k0 = 0; k0 < a.r; k0 += RS_KC) {
    for (int e = tid; e < RS_KC * RS_T; e += RS_NT) {
      int kk = e / RS_T, i = e % RS_T;
      int64_t gi = row0 + i;
      As[kk][i] = (k0 + kk < a.r && gi < a.m) ? A[(int64_t)(k0 + kk) * a.m + gi] : 0.0;
    }
    for (int e = tid; e < RS_KC * RS_T; e += RS_NT) {
      int j = e / RS_KC, kk = e % RS_KC;
      int64_t gj = col0 + j;
      Bs[kk][j] = (k0 + kk < a.r && gj < a.n) ? B[gj * a.r + k0 + kk] : 0.0;
    }
    __syncthreads();
#pragma unroll 4
    for (int kk = 0; kk < RS_KC; ++kk) {
      double av[8], bv[8];
#pragma unroll
      for (int x = 0; x < 8; ++x) av[x] = As[kk][tx + 16 * x];
#pragma unroll
      for (int x = 0; x < 4; ++x) {
        double2 u = reinterpret_cast<const double2 *>(&Bs[kk][ty * 8])[x];
        bv[2 * x] = u.x; bv[2 * x + 1] = u.y;
      }
#pragma unroll
      for (int x = 0; x < 8; ++x)
#pragma unroll
        for (int y = 0; y < 8; ++y) acc[x][y] = fma(av[x], bv[y], acc[x][y]);
    }
    __syncthreads();
  }
  double num = 0.0, den = 0.0;
  if (PRE && full) {
    cp_async_wait_all();
    __syncthreads();
#pragma unroll
    for (int y = 0; y < 8; ++y) {
      const float *wc = &Wsm[(ty * 8 + y) * RS_T + tx];
#pragma unroll
      for (int x = 0; x < 8; ++x) {
        const double w = (double)wc[16 * x];
        const double d = w - acc[x][y];
        num = fma(d, d, num);
        den = fma(w, w, den);
      }
    }
  } else {
#pragma unroll
    for (int y = 0; y < 8; ++y) {
      const int64_t gj = col0 + ty * 8 + y;
      if (gj >= a.n) continue;
#pragma unroll
      for (int x = 0; x < 8; ++x) {
        const int64_t gi = row0 + tx + 16 * x;
        if (gi < a.m) {
          const double w = (double)W[gj * a.ldw + gi];
          const double d = w - acc[x][y];
          num = fma(d, d, num);
          den = fma(w, w, den);
        }
      }
    }
  }
  num = warp_sum(num);
  den = warp_sum(den);
  if ((tid & 31) == 0) {
    red[0][tid >> 5] = num;
    red[1][tid >> 5] = den;
  }
  __syncthreads();
  if (tid == 0) {
    double s0 = 0.0, s1 = 0.0;
    for (int w = 0; w < RS_NT / 32; ++w) { s0 += red[0][w]; s1 += red[1][w]; }
    a.partial[b * a.tiles_m * a.tiles_n + tile] = make_double2(s0, s1);
  }
}

// per problem: fixed-order sum of its tile partials -> num2[b], den2[b]
__global__ void __launch_bounds__(256) k_reduce(const double2 *partial, int64_t ntiles, double *num2,
                                                double *den2, double scale_num, const int32_t *status) {
  __shared__ double r0[8], r1[8];
  const int64_t b = blockIdx.x;
  if (status && status[b] != LRA_OK) {
    if (threadIdx.x == 0) { num2[b] = NAN; den2[b] = NAN; }
    return;
  }
  double s0 = 0.0, s1 = 0.0;
  for (int64_t t = threadIdx.x; t < ntiles; t += 256) {
    double2 p = partial[b * ntiles + t];
    s0 += p.x;
    s1 += p.y;
  }
  s0 = warp_sum(s0);
  s1 = warp_sum(s1);
  if ((threadIdx.x & 31) == 0) { r0[threadIdx.x >> 5] = s0; r1[threadIdx.x >> 5] = s1; }
  __syncthreads();
  if (threadIdx.x == 0) {
    double x = 0.0, y = 0.0;
    for (int w = 0; w < 8; ++w) { x += r0[w]; y += r1[w]; }
    num2[b] = x * scale_num;
    den2[b] = y;
  }
}

cudaError_t launch_reduce(const double2 *partial, int64_t ntiles, int64_t nb, double *num2, double *den2,
                          const int32_t *status, cudaStream_t st, int *nlaunch, Prof *pf) {
  pf->begin("k_reduce", st);
  k_reduce<<<(unsigned)nb, 256, 0, st>>>(partial, ntiles, num2, den2, 1.0, status);
  pf->end(st);
  *nlaunch += 1;
  return cudaGetLastError();
}

cudaError_t launch_residual(ResArgs a, int64_t nb, double *num2, double *den2, cudaStream_t st, int *nlaunch, Prof *pf) {
  a.tiles_m = (a.m + RS_T - 1) / RS_T;
  a.tiles_n = (a.n + RS_T - 1) / RS_T;
  dim3 grid((unsigned)(a.tiles_m * a.tiles_n), (unsigned)nb);
  pf->begin("k_residual", st);
  if (a.dtype == LRA_F32) {
    const int sm = RS_T * RS_T * 4;
    cudaError_t e0 = cudaFuncSetAttribute(k_residual<float>, cudaFuncAttributeMaxDynamicSharedMemorySize, sm);
    if (e0 != cudaSuccess) return e0;
    k_residual<float><<<grid, RS_NT, sm, st>>>(a);
  } else {
    k_residual<double><<<grid, RS_NT, 0, st>>>(a);
  }
  pf->end(st);
  cudaError_t e = cudaGetLastError();
  if (e != cudaSuccess) return e;
  pf->begin("k_reduce", st);
  k_reduce<<<(unsigned)nb, 256, 0, st>>>(a.partial, a.tiles_m * a.tiles_n, num2, den2, 1.0, a.status);
  pf->end(st);
  *nlaunch += 2;
  return cudaGetLastError();
}

// ------------------------------------------------------------- sampled residual
// d_q = W(i_q, j_q) - A[i_q,:] B[:,j_q]; per-CTA partials of sum d^2.
__global__ void __launch_bounds__(256) k_sampled(OpView op, const double *A, const double *B, int r,
                                                 const int64_t *si, const int64_t *sj, int64_t Q,
                                                 double2 *partial) {
  __shared__ double red[8];
  double s = 0.0;
  for (int64_t q = (int64_t)blockIdx.x * 256 + threadIdx.x; q < Q; q += (int64_t)gridDim.x * 256) {
    const int64_t i = si[q], j = sj[q];
    double ab = 0.0;
    for (int t = 0; t < r; ++t) ab = fma(A[(int64_t)t * op.m + i], B[j * r + t], ab);
    const double d = op.at(i, j) - ab;
    s = fma(d, d, s);
  }
  s = warp_sum(s);
  if ((threadIdx.x & 31) == 0) red[threadIdx.x >> 5] = s;
  __syncthreads();
  if (threadIdx.x == 0) {
    double x = 0.0;
    for (int w = 0; w < 8; ++w) x += red[w];
    partial[blockIdx.x] = make_double2(x, 0.0);
  }
}

// dense ||W||_F^2 (per-CTA partials over column ranges)
template <typename TW>
__global__ void __launch_bounds__(256) k_sumsq(const TW *W, int64_t m, int64_t n, int64_t ldw, double2 *partial) {
  __shared__ double red[8];
  double s = 0.0;
  for (int64_t j = blockIdx.x; j < n; j += gridDim.x)
    for (int64_t i = threadIdx.x; i < m; i += 256) {
      double w = (double)W[j * ldw + i];
      s = fma(w, w, s);
    }
  s = warp_sum(s);
  if ((threadIdx.x & 31) == 0) red[threadIdx.x >> 5] = s;
  __syncthreads();
  if (threadIdx.x == 0) {
    double x = 0.0;
    for (int w = 0; w < 8; ++w) x += red[w];
    partial[blockIdx.x] = make_double2(0.0, x);
  }
}

// factored ||W||_F^2 = tr((A^T A)(B B^T)) + 2 sum_E E.(AB) + sum E^2 (one CTA per row
// block for the E terms; the Gram trace is computed by CTA 0 from the p x p Grams).
__global__ void __launch_bounds__(256) k_fact_den(FactOp f, int64_t n, double2 *partial) {
  __shared__ double red[8];
  double s = 0.0;
  // E terms over rows
  for (int64_t i = (int64_t)blockIdx.x * 256 + threadIdx.x; i < f.m; i += (int64_t)gridDim.x * 256) {
    for (int64_t e = f.rowptr[i]; e < f.rowptr[i + 1]; ++e) {
      const int64_t j = f.col[e];
      double ab = 0.0;
      for (int64_t t = 0; t < f.p; ++t) ab = fma(f.fa[t * f.m + i], f.fb[j * f.p + t], ab);
      const double v = f.val[e];
      s += 2.0 * v * ab + v * v;
    }
  }
  // Gram trace: CTA-strided over (t, u) pairs, each sum over rows / columns
  for (int64_t tu = blockIdx.x; tu < f.p * f.p; tu += gridDim.x) {
    const int64_t t = tu / f.p, u = tu % f.p;
    double ga = 0.0, gb = 0.0;
    for (int64_t i = threadIdx.x; i < f.m; i += 256) ga = fma(f.fa[t * f.m + i], f.fa[u * f.m + i], ga);
    for (int64_t j = threadIdx.x; j < n; j += 256) gb = fma(f.fb[j * f.p + t], f.fb[j * f.p + u], gb);
    ga = warp_sum(ga);
    gb = warp_sum(gb);
    __shared__ double ra[8], rb[8];
    if ((threadIdx.x & 31) == 0) { ra[threadIdx.x >> 5] = ga; rb[threadIdx.x >> 5] = gb; }
    __syncthreads();
    if (threadIdx.x == 0) {
      double x = 0.0, y = 0.0;
      for (int w = 0; w < 8; ++w) { x += ra[w]; y += rb[w]; }
      s += x * y;
    }
    __syncthreads();
  }
  s = warp_sum(s);
  if ((threadIdx.x & 31) == 0) red[threadIdx.x >> 5] = s;
  __syncthreads();
  if (threadIdx.x == 0) {
    double x = 0.0;
    for (int w = 0; w < 8; ++w) x += red[w];
    partial[blockIdx.x] = make_double2(0.0, x);
  }
}

// ------------------------------------------------ NEXT-2: q x s error submatrix statistics
// g[a * s + b] = W(rows[a], cols[b]) - A[rows[a], :] B[:, cols[b]]  (Section spstr)
__global__ void __launch_bounds__(256) k_error_sample(OpView op, const double *A, const double *B, int r,
                                                      const int64_t *rows, int64_t q, const int64_t *cols,
                                                      int64_t s, double *g) {
  const int64_t K = q * s;
  for (int64_t e = (int64_t)blockIdx.x * 256 + threadIdx.x; e < K; e += (int64_t)gridDim.x * 256) {
    const int64_t i = rows[e / s], j = cols[e % s];
    double ab = 0.0;
    for (int t = 0; t < r; ++t) ab = fma(A[(int64_t)t * op.m + i], B[j * r + t], ab);
    const double w = op.at(i, j);
    g[e] = w - ab;
    g[K + e] = w;        // the sampled entries of W (superfast estimate of ||W||_F^2)
  }
}
// one CTA: mu = sum g / K, var = sum (g - mu)^2 / K, sum g^2, sum W^2 (fixed order: deterministic)
__global__ void __launch_bounds__(1024) k_error_stats(const double *g, int64_t K, double *out3) {
  __shared__ double red[3][32];
  __shared__ double s_mu;
  double s1 = 0.0, s2 = 0.0, s3 = 0.0;
  for (int64_t e = threadIdx.x; e < K; e += 1024) {
    const double x = g[e], w = g[K + e];
    s1 += x;
    s2 = fma(x, x, s2);
    s3 = fma(w, w, s3);
  }
  s1 = warp_sum(s1);
  s2 = warp_sum(s2);
  s3 = warp_sum(s3);
  if ((threadIdx.x & 31) == 0) {
    red[0][threadIdx.x >> 5] = s1;
    red[1][threadIdx.x >> 5] = s2;
    red[2][threadIdx.x >> 5] = s3;
  }
  __syncthreads();
  if (threadIdx.x == 0) {
    double a = 0.0, b = 0.0, c = 0.0;
    for (int w = 0; w < 32; ++w) {
      a += red[0][w];
      b += red[1][w];
      c += red[2][w];
    }
    s_mu = a / (double)K;
    out3[0] = s_mu;
    out3[2] = b;
    out3[3] = c;
  }
  __syncthreads();
  const double mu = s_mu;
  double v = 0.0;
  for (int64_t e = threadIdx.x; e < K; e += 1024) {
    const double x = g[e] - mu;
    v = fma(x, x, v);
  }
  v = warp_sum(v);
  __syncthreads();
  if ((threadIdx.x & 31) == 0) red[0][threadIdx.x >> 5] = v;
  __syncthreads();
  if (threadIdx.x == 0) {
    double a = 0.0;
    for (int w = 0; w < 32; ++w) a += red[0][w];
    out3[1] = a / (double)K;
  }
}

// ||W[:,J]||_F^2, ||W[I,:]||_F^2, ||U||_F^2 -> out3 (one CTA each, fixed order)
__global__ void __launch_bounds__(1024) k_cert_norms(OpView op, const int64_t *I, const int64_t *J, int k, int l,
                                                     const double *U, double *out3) {
  __shared__ double red[32];
  const int which = blockIdx.x;
  double acc = 0.0;
  if (which == 0) {
    const int64_t tot = op.m * l;
    for (int64_t e = threadIdx.x; e < tot; e += 1024) {
      const double w = op.at(e % op.m, J[e / op.m]);
      acc = fma(w, w, acc);
    }
  } else if (which == 1) {
    const int64_t tot = (int64_t)k * op.n;
    for (int64_t e = threadIdx.x; e < tot; e += 1024) {
      const double w = op.at(I[e % k], e / k);
      acc = fma(w, w, acc);
    }
  } else {
    for (int64_t e = threadIdx.x; e < (int64_t)k * l; e += 1024) acc = fma(U[e], U[e], acc);
  }
  acc = warp_sum(acc);
  if ((threadIdx.x & 31) == 0) red[threadIdx.x >> 5] = acc;
  __syncthreads();
  if (threadIdx.x == 0) {
    double a = 0.0;
    for (int w = 0; w < 32; ++w) a += red[w];
    out3[which] = a;
  }
}

cudaError_t launch_cert_norms(const OpView &op, const int64_t *I, const int64_t *J, int k, int l, const double *U,
                              double *out3, cudaStream_t st) {
  k_cert_norms<<<3, 1024, 0, st>>>(op, I, J, k, l, U, out3);
  return cudaGetLastError();
}

cudaError_t launch_error_sample(const OpView &op, const double *A, const double *B, int r, const int64_t *rows,
                                int64_t q, const int64_t *cols, int64_t s, double *g, double *out3, cudaStream_t st,
                                int *nlaunch, Prof *pf) {
  const int64_t K = q * s;
  const unsigned grid = (unsigned)((K + 255) / 256 < 1184 ? (K + 255) / 256 : 1184);
  pf->begin("k_error_sample", st);
  k_error_sample<<<grid, 256, 0, st>>>(op, A, B, r, rows, q, cols, s, g);
  pf->end(st);
  cudaError_t e = cudaGetLastError();
  if (e != cudaSuccess) return e;
  k_error_stats<<<1, 1024, 0, st>>>(g, K, out3);
  *nlaunch += 2;
  return cudaGetLastError();
}

cudaError_t launch_sampled(const OpView &op, const double *A, const double *B, int r, const int64_t *si,
                           const int64_t *sj, int64_t Q, double2 *partial, int nblk, double *num2,
                           double *den2, cudaStream_t st, int *nlaunch, Prof *pf) {
  // partial layout: [0, nblk) sample partials, [nblk, 2 nblk) den partials
  pf->begin("k_sampled", st);
  k_sampled<<<nblk, 256, 0, st>>>(op, A, B, r, si, sj, Q, partial);
  pf->end(st);
  cudaError_t e = cudaGetLastError();
  if (e != cudaSuccess) return e;
  pf->begin("k_sumsq", st);
  if (op.kind == LRA_OP_DENSE) {
    if (op.dtype == LRA_F32)
      k_sumsq<float><<<nblk, 256, 0, st>>>((const float *)op.w, op.m, op.n, op.ldw, partial + nblk);
    else
      k_sumsq<double><<<nblk, 256, 0, st>>>((const double *)op.w, op.m, op.n, op.ldw, partial + nblk);
  } else {
    k_fact_den<<<nblk, 256, 0, st>>>(op.f, op.n, partial + nblk);
  }
  pf->end(st);
  if ((e = cudaGetLastError()) != cudaSuccess) return e;
  // both halves reduce in one fixed-order pass: num from .x of the first half, den from .y
  pf->begin("k_reduce", st);
  k_reduce<<<1, 256, 0, st>>>(partial, 2 * (int64_t)nblk, num2, den2,
                              (double)op.m * (double)op.n / (double)Q, nullptr);
  pf->end(st);
  *nlaunch += 3;
  return cudaGetLastError();
}

}  // namespace lra
