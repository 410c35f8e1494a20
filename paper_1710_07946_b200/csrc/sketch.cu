// sketch.cu — stage 1 of Alg 10.2: Y = W * M for the abridged randomized
// Hadamard / Fourier multipliers, the sparse +-1 multiplier
// and the dense Gaussian reference.
//
// W is column-major, so column c of Y is a signed (twiddled) sum of whole columns of W:
//   ARHT: k_t = (sigma mod s) + t*s,      coef = D[k_t] * (-1)^popcount(t & floor(sigma/s))
//   ARFT: k_t = 2^d (sigma mod s) + t,    coef = D[k_t] * omega_n^{t*sigma mod n}
//   SPARSE_PM1: k_t = sp_row[c*nnz+t],    coef = sp_sign[c*nnz+t]
// summed in ascending t with fp64 accumulation (one multiply, one add: bit-identical to
// the oracle, reading C23).  Each CTA streams 2^d (or nnz) columns over a 1024-row tile
// with 16-byte vector loads; the kernel is HBM-bound.
#include "kernels.cuh"

#include <cstdlib>

namespace lra {

constexpr int SK_NT = 256;
constexpr int SK_ROWS = SK_NT * 4;  // rows per CTA
constexpr int SK_MAXT = 64;         // max terms per output column (2^d <= 64, nnz <= 64)


template <typename TW>
__device__ __forceinline__ void load4(const TW *p, bool vec, int64_t rows_left, double v[4]);

template <>
__device__ __forceinline__ void load4<float>(const float *p, bool vec, int64_t rows_left, double v[4]) {
  if (vec && rows_left >= 4) {
    float4 f = __ldg(reinterpret_cast<const float4 *>(p));
    v[0] = f.x; v[1] = f.y; v[2] = f.z; v[3] = f.w;
  } else {
#pragma unroll
    for (int a = 0; a < 4; ++a) v[a] = a < rows_left ? (double)__ldg(p + a) : 0.0;
  }
}
template <>
__device__ __forceinline__ void load4<double>(const double *p, bool vec, int64_t rows_left, double v[4]) {
  if (vec && rows_left >= 4) {
    double2 a = __ldg(reinterpret_cast<const double2 *>(p));
    double2 b = __ldg(reinterpret_cast<const double2 *>(p) + 1);
    v[0] = a.x; v[1] = a.y; v[2] = b.x; v[3] = b.y;
  } else {
#pragma unroll
    for (int a = 0; a < 4; ++a) v[a] = a < rows_left ? __ldg(p + a) : 0.0;
  }
}

// grid: (row tiles, lbar, nb)
template <typename TW, bool CPLX>
__global__ void __launch_bounds__(SK_NT) k_sketch_structured(SketchArgs a) {
  __shared__ int64_t s_k[SK_MAXT];
  __shared__ double s_cr[SK_MAXT], s_ci[SK_MAXT];
  const int c = blockIdx.y;
  const int64_t b = blockIdx.z;
  const TW *W = reinterpret_cast<const TW *>(a.w) + b * a.w_stride;
  const int8_t *dsign = a.dsign;   // ARHT/ARFT blocks share one multiplier
  // the T signed taps of sampled column c, one thread per tap (independent loads in flight)
  const int T = a.kind == LRA_MUL_SPARSE_PM1 ? a.nnz : (1 << a.depth);
  for (int t = threadIdx.x; t < T; t += blockDim.x) {
    if (a.kind == LRA_MUL_SPARSE_PM1) {
      s_k[t] = a.sp_row[b * a.m_stride + (int64_t)c * a.nnz + t];
      s_cr[t] = (double)a.sp_sign[b * a.m_stride + (int64_t)c * a.nnz + t];
      s_ci[t] = 0.0;
    } else {
      const int64_t sigma = a.col[c];
      const int64_t q = (int64_t)1 << a.depth, s = a.n >> a.depth;
      if (a.kind == LRA_MUL_ARHT) {
        int64_t k = (sigma % s) + t * s;                         // H_{2^d} (x) I_s
        int par = __popcll((unsigned long long)(t & (sigma / s))) & 1;
        s_k[t] = k;
        s_cr[t] = (double)dsign[k] * (par ? -1.0 : 1.0);
        s_ci[t] = 0.0;
      } else {                                                   // ARFT closed form (reading C4)
        int64_t k = q * (sigma % s) + t;
        int64_t e = (t * sigma) % a.n;
        double ang = (2.0 * M_PI * (double)e) / (double)a.n;
        double sn, cs;
        sincos(ang, &sn, &cs);
        double dk = (double)dsign[k];
        s_k[t] = k;
        s_cr[t] = dk * cs;
        s_ci[t] = dk * sn;
      }
    }
  }
  __syncthreads();
  const int64_t i0 = (int64_t)blockIdx.x * SK_ROWS + (int64_t)threadIdx.x * 4;
  if (i0 >= a.m) return;
  const int64_t left = a.m - i0;
  const bool vec = ((a.ldw & 3) == 0) && ((reinterpret_cast<uintptr_t>(W) & 15) == 0);
  double accr[4] = {0.0, 0.0, 0.0, 0.0}, acci[4] = {0.0, 0.0, 0.0, 0.0};
  // all loads of a 16-term chunk in flight (raw TW values), then the ordered accumulation
  constexpr int CH = sizeof(TW) == 4 ? 16 : 8;
  for (int t0 = 0; t0 < T; t0 += CH) {
    TW v[CH][4];
#pragma unroll
    for (int u = 0; u < CH; ++u) {
      if (t0 + u < T) {
        const TW *src = W + s_k[t0 + u] * a.ldw + i0;
        if (vec && left >= 4) {
          if (sizeof(TW) == 4) {
            float4 f = __ldcs(reinterpret_cast<const float4 *>(src));
            v[u][0] = f.x; v[u][1] = f.y; v[u][2] = f.z; v[u][3] = f.w;
          } else {
            double2 d0 = __ldcs(reinterpret_cast<const double2 *>(src));
            double2 d1 = __ldcs(reinterpret_cast<const double2 *>(src) + 1);
            v[u][0] = d0.x; v[u][1] = d0.y; v[u][2] = d1.x; v[u][3] = d1.y;
          }
        } else {
#pragma unroll
          for (int r = 0; r < 4; ++r) v[u][r] = r < left ? src[r] : (TW)0;
        }
      }
    }
#pragma unroll
    for (int u = 0; u < CH; ++u) {
      if (t0 + u < T) {
        const double cr = s_cr[t0 + u];
#pragma unroll
        for (int r = 0; r < 4; ++r) accr[r] = __dadd_rn(accr[r], __dmul_rn(cr, (double)v[u][r]));
        if (CPLX) {
          const double ci = s_ci[t0 + u];
#pragma unroll
          for (int r = 0; r < 4; ++r) acci[r] = __dadd_rn(acci[r], __dmul_rn((double)v[u][r], ci));
        }
      }
    }
  }
  if (CPLX) {
    double2 *Y = reinterpret_cast<double2 *>(a.y) + b * a.y_stride + (int64_t)c * a.ldy;
#pragma unroll
    for (int r = 0; r < 4; ++r)
      if (r < left) Y[i0 + r] = make_double2(accr[r], acci[r]);
  } else {
    double *Y = reinterpret_cast<double *>(a.y) + b * a.y_stride + (int64_t)c * a.ldy;
    if (left >= 4 && ((reinterpret_cast<uintptr_t>(Y + i0) & 15) == 0)) {
      reinterpret_cast<double2 *>(Y + i0)[0] = make_double2(accr[0], accr[1]);
      reinterpret_cast<double2 *>(Y + i0)[1] = make_double2(accr[2], accr[3]);
    } else {
#pragma unroll
      for (int r = 0; r < 4; ++r)
        if (r < left) Y[i0 + r] = accr[r];
    }
  }
}

// Dense Gaussian reference Y = W * Omega, accumulated sequentially in k (ascending) per
// output in fp64.  When a K-chunk of Omega holds only fp32-representable values and W is
// fp32, every product is exact and FMA equals multiply-then-add; otherwise the product is
// rounded first (oracle order).  grid: (ceil(m/32), ceil(lbar/16), nb)
// Gaussian (and quasi-Gaussian) sketch Y = W * Omega, every output accumulated over k in
// ascending order (the oracle's order).  One warp per CTA computes a 32-row x 16-column tile,
// 4 x 4 outputs per lane (16 independent accumulators); W and Omega are staged through shared
// memory 32 k at a time while the next chunk's loads are already in flight (register
// prefetch).  When a product is exact in fp64 (fp32 W times an fp32-representable Omega — the
// fp32-rounded Gaussian and the integer quasi-Gaussian multipliers) one DFMA equals the
// oracle's rounded product + rounded sum; otherwise the two roundings are kept.
// Gaussian (and quasi-Gaussian) sketch Y = W * Omega, every output accumulated over k in
// ascending order (the oracle's order, so no split over k: the m x lbar outputs are the only
// parallelism, ~196k chains of 4096 DFMAs for config 2).  One CTA (4 warps) owns a 16-row
// tile and all lbar columns; thread (rg, cg) accumulates rows 2 rg, 2 rg + 1 x columns
// cg + 16 t (t < CT), i.e. 2 CT independent chains, so the grid has ~7 warps per SM and every
// SM sub-partition stays busy.  Per k a thread reads one 8-byte W pair and CT Omega values
// (broadcast within its column group) from shared memory.  32-k chunks: W by a 3-stage
// cp.async ring, Omega (column-major in global, k-major in shared memory) by register
// prefetch one chunk ahead.  When a product is exact in fp64 (fp32 W times an
// fp32-representable Omega — the fp32-rounded Gaussian and the integer quasi-Gaussian
// multipliers) one DFMA equals the oracle's rounded product + rounded sum; otherwise the two
// roundings are kept.
constexpr int GS_K = 32, GS_R = 16, GS_ST = 3, GS_NT = 128;

__device__ __forceinline__ void cpa16(void *dst, const void *src, int src_bytes) {
  asm volatile("cp.async.cg.shared.global [%0], [%1], 16, %2;\n" ::"r"((uint32_t)__cvta_generic_to_shared(dst)),
               "l"(src), "r"(src_bytes)
               : "memory");
}

template <typename TW, int CT>
__global__ void __launch_bounds__(GS_NT) k_sketch_gauss(SketchArgs a, const double *omega, int64_t ldo) {
  constexpr int LBP = 16 * CT;                                   // padded columns
  constexpr int NO = GS_K * LBP / GS_NT;                         // Omega values per thread per chunk
  constexpr int ST = GS_ST;
  __shared__ __align__(16) TW Wst[ST][GS_K][GS_R];
  __shared__ __align__(16) double Os[GS_K][LBP + 1];
  const int64_t b = blockIdx.y;
  const TW *W = reinterpret_cast<const TW *>(a.w) + b * a.w_stride;
  const int64_t r0 = (int64_t)blockIdx.x * GS_R;
  const int tid = threadIdx.x, rg = tid & 7, cg = tid >> 3;
  const int64_t nchunk = (a.n + GS_K - 1) / GS_K;
  const bool wvec = ((a.ldw * (int64_t)sizeof(TW)) % 16 == 0) && ((reinterpret_cast<uintptr_t>(W) & 15) == 0) &&
                    r0 + GS_R <= a.m;
  auto load_w = [&](int64_t ch, int stg) {
    const int64_t k0 = ch * GS_K;
    constexpr int WPER = 16 / (int)sizeof(TW);
    if (wvec) {
      for (int e = tid; e < GS_K * GS_R / WPER; e += GS_NT) {
        const int kk = e / (GS_R / WPER), rr = (e % (GS_R / WPER)) * WPER;
        const int64_t k = k0 + kk;
        cpa16(&Wst[stg][kk][rr], W + (k < a.n ? k : 0) * a.ldw + r0 + rr, k < a.n ? 16 : 0);
      }
    } else {
      for (int e = tid; e < GS_K * GS_R; e += GS_NT) {
        const int kk = e / GS_R, rr = e % GS_R;
        const int64_t k = k0 + kk, i = r0 + rr;
        Wst[stg][kk][rr] = (k < a.n && i < a.m) ? W[k * a.ldw + i] : (TW)0;
      }
    }
  };
  double opre[NO];
  auto load_o = [&](int64_t ch) {
    const int64_t k0 = ch * GS_K;
#pragma unroll
    for (int t = 0; t < NO; ++t) {
      const int e = tid + GS_NT * t, kk = e % GS_K, c = e / GS_K;
      const int64_t k = k0 + kk;
      opre[t] = (c < a.lbar && k < a.n) ? __ldg(omega + (int64_t)c * ldo + k) : 0.0;
    }
  };
  double acc[2][CT];
#pragma unroll
  for (int x = 0; x < 2; ++x)
#pragma unroll
    for (int y = 0; y < CT; ++y) acc[x][y] = 0.0;
  for (int p = 0; p < ST - 1; ++p) {
    if (p < nchunk) load_w(p, p);
    asm volatile("cp.async.commit_group;\n" ::: "memory");
  }
  load_o(0);
  for (int64_t ch = 0; ch < nchunk; ++ch) {
    if (ch + ST - 1 < nchunk) load_w(ch + ST - 1, (int)((ch + ST - 1) % ST));
    asm volatile("cp.async.commit_group;\n" ::: "memory");
    int ex = sizeof(TW) == 4;
#pragma unroll
    for (int t = 0; t < NO; ++t) {
      const int e = tid + GS_NT * t;
      Os[e % GS_K][e / GS_K] = opre[t];
      ex &= ((double)(float)opre[t] == opre[t]);
    }
    asm volatile("cp.async.wait_group %0;\n" ::"n"(ST - 1) : "memory");
    const bool exact = __syncthreads_and(ex);          // also publishes Os and this stage of W
    if (ch + 1 < nchunk) load_o(ch + 1);               // in flight during the chunk
    const int stg = (int)(ch % ST);
    const int kmax = (int)min((int64_t)GS_K, a.n - ch * GS_K);
#define GS_BODY(OPR)                                                                             \
  {                                                                                             \
    const double w0 = (double)Wst[stg][kk][2 * rg], w1 = (double)Wst[stg][kk][2 * rg + 1];      \
    _Pragma("unroll") for (int y = 0; y < CT; ++y) {                                            \
      const double o = Os[kk][cg + 16 * y];                                                     \
      acc[0][y] = OPR(w0, o, acc[0][y]);                                                        \
      acc[1][y] = OPR(w1, o, acc[1][y]);                                                        \
    }                                                                                           \
  }
#define GS_FMA(w, o, c) fma(w, o, c)
#define GS_RND(w, o, c) __dadd_rn(c, __dmul_rn(w, o))
    if (exact) {
      if (kmax == GS_K) {
#pragma unroll 8
        for (int kk = 0; kk < GS_K; ++kk) GS_BODY(GS_FMA)
      } else {
        for (int kk = 0; kk < kmax; ++kk) GS_BODY(GS_FMA)
      }
    } else {
      if (kmax == GS_K) {
#pragma unroll 8
        for (int kk = 0; kk < GS_K; ++kk) GS_BODY(GS_RND)
      } else {
        for (int kk = 0; kk < kmax; ++kk) GS_BODY(GS_RND)
      }
    }
#undef GS_BODY
#undef GS_FMA
#undef GS_RND
    __syncthreads();
  }
  asm volatile("cp.async.wait_group 0;\n" ::: "memory");
  double *Y = reinterpret_cast<double *>(a.y) + b * a.y_stride;
#pragma unroll
  for (int x = 0; x < 2; ++x)
#pragma unroll
    for (int y = 0; y < CT; ++y) {
      const int64_t i = r0 + 2 * rg + x, c = cg + 16 * y;
      if (i < a.m && c < a.lbar) Y[c * a.ldy + i] = acc[x][y];
    }
}

template <typename TW, int CT>
static cudaError_t launch_gauss_t(const SketchArgs &a, int64_t nb, const double *omega, int64_t ldo, cudaStream_t st) {
  dim3 grid((unsigned)((a.m + GS_R - 1) / GS_R), (unsigned)nb);
  k_sketch_gauss<TW, CT><<<grid, GS_NT, 0, st>>>(a, omega, ldo);
  return cudaGetLastError();
}

template <typename TW>
static cudaError_t launch_gauss(const SketchArgs &a, int64_t nb, const double *omega, int64_t ldo, cudaStream_t st) {
  switch ((a.lbar + 15) / 16) {
    case 1: return launch_gauss_t<TW, 1>(a, nb, omega, ldo, st);
    case 2: return launch_gauss_t<TW, 2>(a, nb, omega, ldo, st);
    case 3: return launch_gauss_t<TW, 3>(a, nb, omega, ldo, st);
    case 4: return launch_gauss_t<TW, 4>(a, nb, omega, ldo, st);
    case 5: return launch_gauss_t<TW, 5>(a, nb, omega, ldo, st);
    case 6: return launch_gauss_t<TW, 6>(a, nb, omega, ldo, st);
    case 7: return launch_gauss_t<TW, 7>(a, nb, omega, ldo, st);
    default: return cudaErrorInvalidValue;
  }
}

// ---------------------------------------------------------------- NEXT-1: all n columns
// W' = W D H_{n,d} P (Alg 10.1 stage 1 with u = n, the Table tb_fh protocol): for fiber f the
// 2^d columns k_t = f + t s of W feed the 2^d outputs sigma_u = f + u s, stored at column
// c_u = P^{-1}(sigma_u):  W'[:, c_u] = sum_t (D[k_t] (-1)^popcount(t & u)) W[:, k_t]  in the
// oracle's order (ascending t, fp64, one rounding to W's precision at the end, reading C25).
// Each fiber's columns are read once and its outputs written once: 2 m n s_e bytes (HBM).
// grid (ceil(m / 256), s), one row per thread.
__global__ void k_perm_inverse(const int64_t *perm, int64_t n, int *pinv) {
  for (int64_t c = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; c < n; c += (int64_t)gridDim.x * blockDim.x)
    pinv[perm[c]] = (int)c;
}

template <typename TW, int D>
__global__ void __launch_bounds__(256) k_transform_full(const TW *W, int64_t m, int64_t n, int64_t ldw,
                                                        const int8_t *dsign, const int *pinv, TW *Wp,
                                                        int64_t ldo) {
  constexpr int T = 1 << D;
  const int64_t s = n >> D;
  const int64_t f = blockIdx.y;
  const int64_t i = (int64_t)blockIdx.x * 256 + threadIdx.x;
  __shared__ double s_d[T];
  __shared__ int s_c[T];
  if (threadIdx.x < T) {
    s_d[threadIdx.x] = (double)dsign[f + threadIdx.x * s];
    s_c[threadIdx.x] = pinv[f + threadIdx.x * s];
  }
  __syncthreads();
  if (i >= m) return;
  // D[k_t] W[i, k_t] (exact: D = +-1); with t and u unrolled the Hadamard sign is a constant,
  // so each term is one fp64 add (products by +-1 are exact, the order is the oracle's)
  double v[T];
#pragma unroll
  for (int t = 0; t < T; ++t) v[t] = s_d[t] * (double)__ldcs(W + (f + t * s) * ldw + i);
#pragma unroll
  for (int u = 0; u < T; ++u) {
    double acc = 0.0;
#pragma unroll
    for (int t = 0; t < T; ++t) acc = __dadd_rn(acc, ((__popc(t & u) & 1) ? -v[t] : v[t]));
    __stcs(Wp + (int64_t)s_c[u] * ldo + i, (TW)acc);
  }
}

template <typename TW>
static cudaError_t launch_tf(const SketchArgs &a, const int *pinv, void *out, int64_t ldo, cudaStream_t st) {
  dim3 grid((unsigned)((a.m + 255) / 256), (unsigned)(a.n >> a.depth));
  const TW *W = reinterpret_cast<const TW *>(a.w);
  TW *Wp = reinterpret_cast<TW *>(out);
  switch (a.depth) {
    case 1: k_transform_full<TW, 1><<<grid, 256, 0, st>>>(W, a.m, a.n, a.ldw, a.dsign, pinv, Wp, ldo); break;
    case 2: k_transform_full<TW, 2><<<grid, 256, 0, st>>>(W, a.m, a.n, a.ldw, a.dsign, pinv, Wp, ldo); break;
    case 3: k_transform_full<TW, 3><<<grid, 256, 0, st>>>(W, a.m, a.n, a.ldw, a.dsign, pinv, Wp, ldo); break;
    case 4: k_transform_full<TW, 4><<<grid, 256, 0, st>>>(W, a.m, a.n, a.ldw, a.dsign, pinv, Wp, ldo); break;
    case 5: k_transform_full<TW, 5><<<grid, 256, 0, st>>>(W, a.m, a.n, a.ldw, a.dsign, pinv, Wp, ldo); break;
    default: return cudaErrorInvalidValue;
  }
  return cudaGetLastError();
}

cudaError_t launch_transform_full(const SketchArgs &a, int *pinv, void *out, int64_t ldo, cudaStream_t st, Prof *pf) {
  k_perm_inverse<<<(unsigned)((a.n + 255) / 256), 256, 0, st>>>(a.col, a.n, pinv);
  cudaError_t e = cudaGetLastError();
  if (e != cudaSuccess) return e;
  pf->begin("k_transform_full", st);
  e = a.dtype == LRA_F32 ? launch_tf<float>(a, pinv, out, ldo, st) : launch_tf<double>(a, pinv, out, ldo, st);
  pf->end(st);
  return e;
}

cudaError_t launch_sketch(const SketchArgs &a, int64_t nb, const double *omega, int64_t ldo,
                          cudaStream_t st, Prof *pf, void *tc_scratch, size_t tc_bytes) {
  if (a.kind == LRA_MUL_GAUSSIAN && tc_scratch) {
    const cudaError_t e = launch_sketch_tc(a, nb, omega, ldo, tc_scratch, tc_bytes, st, pf);
    if (e != cudaErrorInvalidConfiguration) return e;   // W strides TMA cannot map: the SIMT kernel
  }
  if (a.kind == LRA_MUL_GAUSSIAN) {
    pf->begin("k_sketch_gauss", st);
    const cudaError_t e = a.dtype == LRA_F32 ? launch_gauss<float>(a, nb, omega, ldo, st)
                                             : launch_gauss<double>(a, nb, omega, ldo, st);
    pf->end(st);
    return e;
  }
  dim3 grid((unsigned)((a.m + SK_ROWS - 1) / SK_ROWS), (unsigned)a.lbar, (unsigned)nb);
  const bool cplx = a.kind == LRA_MUL_ARFT;
  pf->begin(a.kind == LRA_MUL_SPARSE_PM1 ? "k_sketch_sparse" : (cplx ? "k_sketch_arft" : "k_sketch_arht"), st);
  if (a.dtype == LRA_F32) {
    if (cplx) k_sketch_structured<float, true><<<grid, SK_NT, 0, st>>>(a);
    else k_sketch_structured<float, false><<<grid, SK_NT, 0, st>>>(a);
  } else {
    if (cplx) k_sketch_structured<double, true><<<grid, SK_NT, 0, st>>>(a);
    else k_sketch_structured<double, false><<<grid, SK_NT, 0, st>>>(a);
  }
  pf->end(st);
  return cudaGetLastError();
}

// ------------------------------------------------------------- quasi-Gaussian multiplier
// Omega = G_q[:, col], G_q = M_0 ... M_{q-1}, M_i = B_i P_i (def11; reading C30):
// one CTA per sampled column c, the column vector in global scratch (two int32 buffers of n;
// entries are integers with |.| <= 2^q, q <= 30), the factors applied right to left:
//   U = P_i V:  U[perm_i[j]] = V[j];   V = B_i U:  V[r] = U[r] + sign_i[r-1] U[r-1]  (cyclic).
__global__ void __launch_bounds__(1024) k_qg_build(int64_t n, int q, const int8_t *sign, const int64_t *perm,
                                                   const int64_t *col, int *work, double *omega) {
  extern __shared__ int qsm[];                       // 2 n ints when they fit (else global work)
  const int64_t c = blockIdx.x;
  int *V = work ? work + (size_t)c * 2 * n : qsm, *U = V + n;
  const int64_t sc = col[c];
  for (int64_t j = threadIdx.x; j < n; j += blockDim.x) V[j] = j == sc ? 1 : 0;
  __syncthreads();
  for (int i = q - 1; i >= 0; --i) {
    const int64_t *pi = perm + (size_t)i * n;
    const int8_t *si = sign + (size_t)i * n;
    for (int64_t j = threadIdx.x; j < n; j += blockDim.x) U[pi[j]] = V[j];
    __syncthreads();
    for (int64_t r = threadIdx.x; r < n; r += blockDim.x) {
      const int64_t rm = r == 0 ? n - 1 : r - 1;
      V[r] = U[r] + (int)si[rm] * U[rm];
    }
    __syncthreads();
  }
  for (int64_t r = threadIdx.x; r < n; r += blockDim.x) omega[(size_t)c * n + r] = (double)V[r];
}

cudaError_t launch_qg_build(int64_t n, int q, int64_t lbar, const int8_t *sign, const int64_t *perm,
                            const int64_t *col, int *work, double *omega, cudaStream_t st, Prof *pf) {
  pf->begin("k_qg_build", st);
  const size_t smem = (size_t)2 * n * sizeof(int);
  const bool in_smem = smem <= 200 * 1024;
  if (in_smem) {
    cudaError_t e = cudaFuncSetAttribute(k_qg_build, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
    if (e != cudaSuccess) return e;
  }
  k_qg_build<<<(unsigned)lbar, 1024, in_smem ? smem : 0, st>>>(n, q, sign, perm, col, in_smem ? nullptr : work, omega);
  pf->end(st);
  return cudaGetLastError();
}

}  // namespace lra
