// ca_global.cu — global-memory tier of the real C-A (stages 2-3 of Alg 10.2 with C-A
// iterations, Remark rerfnhmt) for blocks whose C-matrix does not fit on chip
// (config 5: 131072 x 96 fp64 = 100 MB; any q <= 128).
//
// One cooperative persistent launch over all SMs per problem.  The block B (N x q, fp64,
// row-major) and the working C-matrix live in global memory (L2-resident at config-5
// size); CTA c owns the contiguous rows [c*rpc, (c+1)*rpc) and each row is processed by
// TPR threads (W = Q/TPR doubles each).  One pivot step = ONE pass over the CTA's rows that
// applies the previous step's update (cold LUP: B'[i,j] -= (B'[i,t-1]/B'[p,t-1]) B'[p,j],
// one IEEE multiply + one subtract as the oracle; swap: C <- C - C[:,j*](C[i*,:] - e_j*)/c)
// and, in the same pass, streams each thread's candidate (max |c| and the smallest linear
// index inside its tie window) -> warp -> CTA triple -> global slot -> ONE grid barrier ->
// every CTA decides redundantly and reads the winning row from global memory.  The tie
// rule is exact as in the cluster tier (a unit whose maximum lies in the tie window without
// equalling the global maximum, or a thread whose running maximum was overtaken inside its
// own window, flags the decision and an exact read-only pass decides it).
// C = B G^{-1} with G = B[S,:] inverted by the in-place Gauss-Jordan of the cluster tier in
// every CTA (fresh each maxvol call; no carried inverse in this tier).
#include <cooperative_groups.h>
#include <climits>

#include "kernels.cuh"

namespace cg = cooperative_groups;

namespace lra {
namespace cgm {

constexpr int NT = 512;
constexpr int NW = NT / 32;

struct __align__(16) Trip {
  unsigned long long key;
  unsigned idx;
  unsigned amb;
};

template <int Q>
struct Sh {
  long long S[2][Q];
  unsigned long long wkey[NW];
  unsigned widx[NW];
  unsigned wamb[NW];
  __align__(16) double prow[Q];
  __align__(16) double pm[Q];
  double rc;
  double dM;
  unsigned didx;
  int damb;
  unsigned long long gk[2][NW];
  int gr[2][NW];
  __align__(16) double gp[Q];
  double gd;
  int piv[Q], pinv[Q];
};

__device__ __forceinline__ unsigned long long dkey(double v) {
  return v > 0.0 ? (unsigned long long)__double_as_longlong(v) : 0ull;
}
__device__ __forceinline__ double kdbl(unsigned long long k) { return __longlong_as_double((long long)k); }
__device__ __forceinline__ unsigned long long wmaxk(unsigned long long k) {
  const unsigned hi = (unsigned)(k >> 32);
  const unsigned mhi = __reduce_max_sync(0xffffffffu, hi);
  const unsigned mlo = __reduce_max_sync(0xffffffffu, hi == mhi ? (unsigned)k : 0u);
  return ((unsigned long long)mhi << 32) | mlo;
}
__device__ __forceinline__ unsigned wminu(unsigned x) { return __reduce_min_sync(0xffffffffu, x); }

template <int OPK>
__device__ __forceinline__ double op_at(const OpView &op, int64_t i, int64_t j) {
  if (OPK == 0) return (double)__ldg((const float *)op.w + j * op.ldw + i);
  if (OPK == 1) return __ldg((const double *)op.w + j * op.ldw + i);
  return op.f.at(i, j);
}

// Streaming candidate of one thread over values visited in increasing linear index:
// M = running max, idx = smallest index with |c| >= (1-tau) M, amb if a new maximum arrived
// while the previous maximum was inside the new tie window (its earlier qualifying indices
// are not tracked) -> exact pass.
struct Cand {
  double M;
  unsigned idx;
  bool amb;
  __device__ __forceinline__ void init() {
    M = -1.0;
    idx = 0xffffffffu;
    amb = false;
  }
  __device__ __forceinline__ void add(double v, unsigned i, double tau) {
    if (v > M) {
      if (M >= 0.0 && M >= (1.0 - tau) * v) amb = true;
      M = v;
      idx = i;
    }
  }
};

struct GmArgs {
  double *gB, *gC;            // N x Q row-major (original block, working C-matrix)
  Trip *gtri;                 // [2][grid]
  unsigned *gx;               // [2][grid]
  unsigned char *inS;         // N flags (row currently selected)
};

// Gauss-Jordan in place on G (q x q, rows from gB at slots S), X = G^{-1} (row stride Q) in Xo.
template <int Q>
__device__ bool gj_global(Sh<Q> &sh, const long long *S, int q, const double *gB, double *Xo) {
  constexpr int KR = (Q + 15) / 16, MC = (Q + 31) / 32;
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  double x[KR][MC];
#pragma unroll
  for (int a = 0; a < KR; ++a) {
    const int r = warp + 16 * a;
    const double *src = gB + (size_t)(r < q ? S[r] : 0) * Q;
#pragma unroll
    for (int c = 0; c < MC; ++c) {
      const int col = lane + 32 * c;
      x[a][c] = (r < q && col < q) ? __ldcg(src + col) : 0.0;
    }
  }
  unsigned used = 0;
  for (int s = 0; s < q; ++s) {
    const int ls = s & 31, cs_ = s >> 5, sl = s & 1;
    double v[KR];
    unsigned long long key = 0ull;
    int arow = 0x7fffffff;
#pragma unroll
    for (int a = 0; a < KR; ++a) {
      double xv = x[a][0];
#pragma unroll
      for (int c = 1; c < MC; ++c) xv = (cs_ == c) ? x[a][c] : xv;
      v[a] = __shfl_sync(0xffffffffu, xv, ls);
      const int r = warp + 16 * a;
      if (r < q && !((used >> a) & 1u)) {
        const double av = fabs(v[a]);
        const unsigned long long kk = (av != av) ? 0x7ff8000000000000ull : dkey(av);
        if (arow == 0x7fffffff || kk > key) {
          key = kk;
          arow = r;
        }
      }
    }
    if (lane == 0) {
      sh.gk[sl][warp] = key;
      sh.gr[sl][warp] = arow;
    }
    __syncthreads();
    const unsigned long long ck = lane < NW ? sh.gk[sl][lane] : 0ull;
    const int cr = lane < NW ? sh.gr[sl][lane] : 0x7fffffff;
    const unsigned long long mk = wmaxk(ck);
    const int p = (int)__reduce_min_sync(0xffffffffu, (ck == mk && cr != 0x7fffffff) ? (unsigned)cr : 0xffffffffu);
    if (p >= q) return false;
    const int ap = p >> 4;
    if (threadIdx.x == 0) sh.piv[s] = p;
    if (warp == (p & 15)) {
      double d = v[0];
#pragma unroll
      for (int a = 1; a < KR; ++a) d = (ap == a) ? v[a] : d;
      const double rd = 1.0 / d;
#pragma unroll
      for (int c = 0; c < MC; ++c) {
        const int col = lane + 32 * c;
        double xv = x[0][c];
#pragma unroll
        for (int a = 1; a < KR; ++a) xv = (ap == a) ? x[a][c] : xv;
        if (col < Q) sh.gp[col] = (col == s) ? rd : xv * rd;
      }
      if (lane == 0) sh.gd = d;
    }
    __syncthreads();
    const double d = sh.gd;
    if (!(fabs(d) > 0.0) || !isfinite(d)) return false;
#pragma unroll
    for (int a = 0; a < KR; ++a) {
      const int r = warp + 16 * a;
      const bool isp = (r == p);
      if (isp) used |= 1u << a;
#pragma unroll
      for (int c = 0; c < MC; ++c) {
        const int col = lane + 32 * c;
        const double pv = col < Q ? sh.gp[col] : 0.0;
        x[a][c] = isp ? pv : ((col == s) ? fma(-v[a], pv, 0.0) : fma(-v[a], pv, x[a][c]));
      }
    }
  }
  if (threadIdx.x < q) sh.pinv[sh.piv[threadIdx.x]] = threadIdx.x;
  __syncthreads();
#pragma unroll
  for (int a = 0; a < KR; ++a) {
    const int r = warp + 16 * a;
    if (r >= q) continue;
    const int t = sh.pinv[r];
#pragma unroll
    for (int c = 0; c < MC; ++c) {
      const int col = lane + 32 * c;
      if (col < q) Xo[t * Q + sh.piv[col]] = x[a][c];
      else if (col < Q) Xo[t * Q + col] = 0.0;
    }
  }
  __syncthreads();
  return true;
}

// Grid-wide decision from the per-thread streaming candidates (see header).  Returns
// (M, idx, amb) identically in every thread of every CTA.
template <int Q>
__device__ __forceinline__ void decide(Sh<Q> &sh, const Cand &cd, double tau, const GmArgs &g, int &par) {
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const int p = par;
  par ^= 1;
  // warp
  const unsigned long long wk = wmaxk(dkey(cd.M));
  const double wthr = (1.0 - tau) * kdbl(wk);
  const bool top = wk != 0ull && dkey(cd.M) == wk;
  const unsigned wi = wminu(top ? cd.idx : 0xffffffffu);
  const bool wamb = __any_sync(0xffffffffu, (top && cd.amb) ||
                                                (!top && cd.M >= 0.0 && dkey(cd.M) != 0ull && cd.M >= wthr));
  if (lane == 0) {
    sh.wkey[warp] = wk;
    sh.widx[warp] = wi;
    sh.wamb[warp] = wamb;
  }
  __syncthreads();
  if (warp == 0) {
    const bool in = lane < NW;
    const unsigned long long ck = in ? sh.wkey[lane] : 0ull;
    const unsigned long long Ck = wmaxk(ck);
    const double Cthr = (1.0 - tau) * kdbl(Ck);
    const bool ctop = in && ck == Ck && Ck != 0ull;
    const unsigned Ci = wminu(ctop ? sh.widx[lane] : 0xffffffffu);
    const bool Camb = __any_sync(0xffffffffu, (ctop && sh.wamb[lane]) || (in && ck != Ck && ck != 0ull && kdbl(ck) >= Cthr));
    if (lane == 0) {
      Trip t{Ck, Ci, Camb ? 1u : 0u};
      Trip *dst = g.gtri + (size_t)p * gridDim.x + blockIdx.x;
      __stcg(reinterpret_cast<ulonglong2 *>(dst), *reinterpret_cast<ulonglong2 *>(&t));
    }
  }
  cg::this_grid().sync();
  if (warp == 0) {
    unsigned long long Mk = 0ull;
    for (int c = lane; c < (int)gridDim.x; c += 32) Mk = max(Mk, __ldcg(&g.gtri[(size_t)p * gridDim.x + c].key));
    const unsigned long long Gk = wmaxk(Mk);
    const double Gthr = (1.0 - tau) * kdbl(Gk);
    unsigned bi = 0xffffffffu;
    bool amb = false;
    for (int c = lane; c < (int)gridDim.x; c += 32) {
      const ulonglong2 raw = __ldcg(reinterpret_cast<const ulonglong2 *>(&g.gtri[(size_t)p * gridDim.x + c]));
      const unsigned long long k = raw.x;
      const unsigned idx = (unsigned)(raw.y & 0xffffffffu), a = (unsigned)(raw.y >> 32);
      if (k == Gk && Gk != 0ull) {
        bi = min(bi, idx);
        if (a) amb = true;
      } else if (k != 0ull && kdbl(k) >= Gthr) {
        amb = true;
      }
    }
    bi = wminu(bi);
    amb = __any_sync(0xffffffffu, amb);
    if (lane == 0) {
      sh.dM = kdbl(Gk);
      sh.didx = bi;
      sh.damb = amb;
    }
  }
  __syncthreads();
}

// exact round: smallest linear index with value >= thr over the problem (per-thread value
// supplied by the caller's pass as `mine`).
__device__ unsigned long long g_gm_exact;   // exact second rounds (diagnostics)

template <int Q>
__device__ __forceinline__ unsigned decide_exact(Sh<Q> &sh, unsigned mine, const GmArgs &g, int &par) {
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  if (threadIdx.x == 0 && blockIdx.x == 0) atomicAdd(&g_gm_exact, 1ull);
  const int p = par;
  par ^= 1;
  const unsigned wi = wminu(mine);
  if (lane == 0) sh.widx[warp] = wi;
  __syncthreads();
  if (warp == 0) {
    const unsigned ci = wminu(lane < NW ? sh.widx[lane] : 0xffffffffu);
    if (lane == 0) __stcg(&g.gx[(size_t)p * gridDim.x + blockIdx.x], ci);
  }
  cg::this_grid().sync();
  if (warp == 0) {
    unsigned bi = 0xffffffffu;
    for (int c = lane; c < (int)gridDim.x; c += 32) bi = min(bi, __ldcg(&g.gx[(size_t)p * gridDim.x + c]));
    bi = wminu(bi);
    if (lane == 0) sh.didx = bi;
  }
  __syncthreads();
  return sh.didx;
}

template <int Q, int TPR, int OPK, bool QEQ = false>
__global__ void __launch_bounds__(NT, 1) k_cagm(CAArgs a, GmArgs g) {
  if (a.skip && (a.skip[0] != 0 || a.skip[1] != 0)) return;   // row-sharded chain: step not needed
  constexpr int W = Q / TPR, RPP = NT / TPR;
  static_assert(W % 2 == 0, "W even");
  extern __shared__ __align__(16) double Xinv[];     // Q x Q
  __shared__ Sh<Q> sh;
  const int tid = threadIdx.x, lane = tid & 31;
  const int sub = tid % TPR, jb = sub * W, gl = lane & ~(TPR - 1);
  const int q = QEQ ? Q : a.q;           // QEQ: q == Q known at compile time
  const double tau = a.tau, tol = a.tol;
  OpView op = a.op;
  int par = 0;
  int32_t status = LRA_OK;
  int lu = 0, swaps = 0, caps = 0, sk_swaps = 0, loops = 0, sw_h = 0;
  double cert_r = 0.0, cert_c = 0.0;
  double mmin = 1.0;                     // diagnostics: min top-2 pivot margin (reading C35)
  const bool yreal = a.Y != nullptr && !a.y_complex;
  if (!yreal || a.y_warm) {
    if (tid < q) sh.S[0][tid] = a.I0[tid];
    if (a.yinfo) {
      status = a.yinfo[0];
      swaps = sk_swaps = a.yinfo[1];
      caps = a.yinfo[2];
      lu = a.yinfo[3];
    }
  }
  __syncthreads();
  const double *Y = yreal ? reinterpret_cast<const double *>(a.Y) : nullptr;
  const int last = 2 * a.sweeps;
  auto group_val = [&](const double (&c)[W], int col) -> double {   // column col of this row
    const int so = col / W, wo = col - so * W;
    double v = 0.0;
#pragma unroll
    for (int w = 0; w < W; ++w)
      if (w == wo) v = c[w];
    return __shfl_sync(0xffffffffu, v, gl | so);
  };
  for (int step = yreal ? 0 : 1; status == LRA_OK && step <= last; ++step) {
    const int kind = step == 0 ? 0 : ((step & 1) ? 1 : 2);   // 0 = Y, 1 = h, 2 = v
    const int64_t N = kind == 1 ? op.n : op.m;
    long long *S = kind == 1 ? sh.S[1] : sh.S[0];
    const bool cold = step <= 1 && !(step == 0 && a.y_warm);
    const int64_t rpc = (N + gridDim.x - 1) / gridDim.x;
    const int64_t r0 = (int64_t)blockIdx.x * rpc, r1 = min(N, r0 + rpc);
    const int iters = (int)((rpc + RPP - 1) / RPP);
    // ---- gather the block (and the LU working copy) for the owned rows; clear flags
    {
      const long long *I = sh.S[0], *J = sh.S[1];
      for (int64_t row = r0 + tid / TPR; row < r1; row += RPP) {
        double v[W];
#pragma unroll
        for (int w = 0; w < W; ++w) {
          const int j = jb + w;
          double x = 0.0;
          if (j < q) {
            if (kind == 0) x = __ldg(Y + (int64_t)j * a.ldy + row);
            else if (kind == 1) x = op_at<OPK>(op, I[j], row);
            else x = op_at<OPK>(op, row, J[j]);
          }
          v[w] = x;
        }
        double2 *dB = reinterpret_cast<double2 *>(g.gB + (size_t)row * Q + jb);
        double2 *dC = reinterpret_cast<double2 *>(g.gC + (size_t)row * Q + jb);
#pragma unroll
        for (int w = 0; w < W / 2; ++w) {
          const double2 t2 = make_double2(v[2 * w], v[2 * w + 1]);
          __stcg(dB + w, t2);
          if (cold) __stcg(dC + w, t2);
        }
        if (sub == 0) g.inS[row] = 0;
      }
    }
    __syncthreads();
    if (!cold) {   // mark the current slots (warm start)
      if (tid < q && S[tid] >= r0 && S[tid] < r1) g.inS[S[tid]] = 1;
    }
    cg::this_grid().sync();
    int nsw = 0;
    bool ok = true;
    double cert = 0.0;
    bool cap_hit = false;
    if (cold) {
      // ---- Alg D.2 stage 1: LUP (bit-identical arithmetic to the oracle)
      for (int t = 0; t < q && ok; ++t) {
        Cand cd;
        cd.init();
        for (int it = 0; it < iters; ++it) {
          const int64_t row = r0 + (int64_t)it * RPP + tid / TPR;
          const bool has = row < r1;
          double c[W];
#pragma unroll
          for (int w = 0; w < W; ++w) c[w] = 0.0;
          bool sel = true;
          if (has) {
            sel = g.inS[row] != 0;
            const double2 *src = reinterpret_cast<const double2 *>(g.gC + (size_t)row * Q + jb);
#pragma unroll
            for (int w = 0; w < W / 2; ++w) {
              const double2 t2 = __ldcg(src + w);
              c[2 * w] = t2.x;
              c[2 * w + 1] = t2.y;
            }
          }
          if (t > 0) {   // apply step t-1: B'[i,j] -= (B'[i,t-1]/B'[p,t-1]) B'[p,j], j > t-1
            const double x = group_val(c, t - 1);
            if (has && !sel) {
              const double f = x / sh.prow[t - 1];
#pragma unroll
              for (int w = 0; w < W; ++w) c[w] = rsub_mul(c[w], f, sh.pm[jb + w]);
              double2 *dst = reinterpret_cast<double2 *>(g.gC + (size_t)row * Q + jb);
#pragma unroll
              for (int w = 0; w < W / 2; ++w) __stcg(dst + w, make_double2(c[2 * w], c[2 * w + 1]));
            }
          }
          const double x = group_val(c, t);
          if (has && !sel && sub == 0) cd.add((x != x) ? INFINITY : fabs(x), (unsigned)row, tau);
        }
        decide<Q>(sh, cd, tau, g, par);
        double M = sh.dM;
        unsigned idx = sh.didx;
        if (sh.damb) {   // exact pass: smallest row with |B'[row,t]| >= (1-tau) M
          const double thr = (1.0 - tau) * M;
          unsigned mine = 0xffffffffu;
          for (int it = 0; it < iters; ++it) {
            const int64_t row = r0 + (int64_t)it * RPP + tid / TPR;
            if (row < r1 && sub == 0 && !g.inS[row]) {
              const double x = __ldcg(g.gC + (size_t)row * Q + t);
              const double v = (x != x) ? INFINITY : fabs(x);
              if (v >= thr && (unsigned)row < mine) mine = (unsigned)row;
            }
          }
          idx = decide_exact<Q>(sh, mine, g, par);
        }
        if (!(M > 0.0) || !isfinite(M)) { ok = false; break; }
        if (a.diag) {    // top-2 margin: the largest candidate other than the chosen row
          Cand c2;
          c2.init();
          for (int it = 0; it < iters; ++it) {
            const int64_t row = r0 + (int64_t)it * RPP + tid / TPR;
            if (row < r1 && sub == 0 && !g.inS[row] && (unsigned)row != idx) {
              const double x = __ldcg(g.gC + (size_t)row * Q + t);
              c2.add((x != x) ? INFINITY : fabs(x), (unsigned)row, tau);
            }
          }
          decide<Q>(sh, c2, tau, g, par);
          mmin = fmin(mmin, (M - fmax(sh.dM, 0.0)) / M);
        }
        // winning row (its column-t.. values are current) -> prow, pm (masked j > t)
        if (tid < Q) {
          const double xv = tid < q ? __ldcg(g.gC + (size_t)idx * Q + tid) : 0.0;
          sh.prow[tid] = xv;
          sh.pm[tid] = tid > t ? xv : 0.0;
        }
        if (tid == 0) S[t] = idx;
        if ((int64_t)idx >= r0 && (int64_t)idx < r1 && tid == 0) g.inS[idx] = 1;
        __syncthreads();
      }
      cg::this_grid().sync();           // inS flags of all CTAs visible
      if (!ok) { status = LRA_ESINGULAR; break; }
      lu += q;
    }
    // ---- G = B[S,:] -> G^{-1} (every CTA)
    if (!gj_global<Q>(sh, S, q, g.gB, Xinv)) { status = LRA_ESINGULAR; break; }
    // ---- product pass C = B G^{-1} (rows outside S), fused with the first candidate pass,
    // then the Alg D.1 swap loop (each pass applies the previous swap's update)
    int jstar = -1;
    long long istar = -1, sold = -1;
    for (;;) {
      Cand cd;
      cd.init();
      const bool first = jstar < 0 && nsw == 0;
      for (int it = 0; it < iters; ++it) {
        const int64_t row = r0 + (int64_t)it * RPP + tid / TPR;
        const bool has = row < r1;
        double c[W];
#pragma unroll
        for (int w = 0; w < W; ++w) c[w] = 0.0;
        bool sel = true;
        if (has) sel = g.inS[row] != 0;
        if (first) {
          if (has && !sel) {
            const double *brow = g.gB + (size_t)row * Q;
            for (int t = 0; t < q; ++t) {
              const double bt = __ldcg(brow + t);
              const double2 *xr = reinterpret_cast<const double2 *>(Xinv + t * Q + jb);
#pragma unroll
              for (int w = 0; w < W / 2; ++w) {
                const double2 xv = xr[w];
                c[2 * w] = fma(bt, xv.x, c[2 * w]);
                c[2 * w + 1] = fma(bt, xv.y, c[2 * w + 1]);
              }
            }
            double2 *dst = reinterpret_cast<double2 *>(g.gC + (size_t)row * Q + jb);
#pragma unroll
            for (int w = 0; w < W / 2; ++w) __stcg(dst + w, make_double2(c[2 * w], c[2 * w + 1]));
          }
        } else {
          const bool leaving = has && row == sold;      // explicit row e_{j*}, then updated
          if (has && (!sel || leaving)) {
            if (leaving) {
#pragma unroll
              for (int w = 0; w < W; ++w) c[w] = (jb + w == jstar) ? 1.0 : 0.0;
            } else {
              const double2 *src = reinterpret_cast<const double2 *>(g.gC + (size_t)row * Q + jb);
#pragma unroll
              for (int w = 0; w < W / 2; ++w) {
                const double2 t2 = __ldcg(src + w);
                c[2 * w] = t2.x;
                c[2 * w + 1] = t2.y;
              }
            }
          }
          const double xj = group_val(c, jstar);
          if (has && (!sel || leaving)) {
            const double gg = xj * sh.rc;
#pragma unroll
            for (int w = 0; w < W; ++w) c[w] = fma(-gg, sh.pm[jb + w], c[w]);
            double2 *dst = reinterpret_cast<double2 *>(g.gC + (size_t)row * Q + jb);
#pragma unroll
            for (int w = 0; w < W / 2; ++w) __stcg(dst + w, make_double2(c[2 * w], c[2 * w + 1]));
            if (leaving) {
              g.inS[row] = 0;       // (written by every group thread: same value)
              sel = false;
            }
          }
          if (has && row == istar) sel = true;
        }
        if (has && !sel) {
#pragma unroll
          for (int w = 0; w < W; ++w)
            if (jb + w < q) cd.add(fabs(c[w]), (unsigned)(row * q + jb + w), tau);
        }
      }
      // the entering row's flag (owner CTA)
      if (istar >= r0 && istar < r1 && tid == 0) g.inS[istar] = 1;
      decide<Q>(sh, cd, tau, g, par);
      const double M = sh.dM;
      unsigned idx = sh.didx;
      if (!(M == M)) { ok = false; break; }
      if (M <= 1.0 + tol || nsw >= a.cap) {
        cert = fmax(M, 0.0);
        cap_hit = M > 1.0 + tol;
        break;
      }
      if (sh.damb) {
        const double thr = (1.0 - tau) * M;
        unsigned mine = 0xffffffffu;
        for (int it = 0; it < iters; ++it) {
          const int64_t row = r0 + (int64_t)it * RPP + tid / TPR;
          if (row < r1 && !g.inS[row]) {
            const double *src = g.gC + (size_t)row * Q + jb;
            for (int w = 0; w < W; ++w)
              if (jb + w < q && fabs(__ldcg(src + w)) >= thr) {
                mine = min(mine, (unsigned)(row * q + jb + w));
                break;
              }
          }
        }
        idx = decide_exact<Q>(sh, mine, g, par);
      }
      if (a.diag) {      // top-2 margin over C' without the chosen entry
        Cand c2;
        c2.init();
        for (int it = 0; it < iters; ++it) {
          const int64_t row = r0 + (int64_t)it * RPP + tid / TPR;
          if (row < r1 && !g.inS[row]) {
            const double *src = g.gC + (size_t)row * Q + jb;
            for (int w = 0; w < W; ++w) {
              const unsigned li = (unsigned)(row * q + jb + w);
              if (jb + w < q && li != idx) c2.add(fabs(__ldcg(src + w)), li, tau);
            }
          }
        }
        decide<Q>(sh, c2, tau, g, par);
        mmin = fmin(mmin, (M - fmax(sh.dM, 0.0)) / M);
      }
      istar = idx / (unsigned)q;
      jstar = (int)(idx % (unsigned)q);
      sold = S[jstar];
      if (tid < Q) {
        const double xv = tid < q ? __ldcg(g.gC + (size_t)istar * Q + tid) : 0.0;
        sh.prow[tid] = xv;
        sh.pm[tid] = (tid == jstar) ? xv - 1.0 : xv;
        if (tid == jstar) sh.rc = 1.0 / xv;
      }
      __syncthreads();
      if (tid == 0) S[jstar] = istar;
      ++nsw;
      cg::this_grid().sync();     // every CTA read row istar before any CTA updates it
    }
    cg::this_grid().sync();
    if (!ok) { status = LRA_ESINGULAR; break; }
    swaps += nsw;
    caps += cap_hit;
    if (kind == 0) {
      sk_swaps = nsw;
      cert_r = cert;
    }
    if (kind == 1) { cert_c = cert; sw_h = nsw; }
    if (kind == 2) {
      cert_r = cert;
      ++loops;
      if (step > 2 && sw_h == 0 && nsw == 0) break;
    }
  }
  __syncthreads();
  if (blockIdx.x == 0) {
    if (tid < q) {
      a.I[tid] = sh.S[0][tid];
      a.J[tid] = sh.S[1][tid];
    }
    if (tid == 0) {
      a.status[0] = status;
      if (a.stats) {
        lra_ca_stats s;
        s.status = status;
        s.loops_done = loops;
        s.lu_steps = lu;
        s.swaps = swaps;
        s.cap_hits = caps;
        s.sketch_swaps = sk_swaps;
        s.cert_rows = cert_r;
        s.cert_cols = cert_c;
        s.logvol_final = __longlong_as_double(0x7ff8000000000000LL);   // filled by the nucleus
        s.min_pivot_margin = a.diag ? mmin : __longlong_as_double(0x7ff8000000000000LL);
        a.stats[0] = s;
      }
    }
  }
}

}  // namespace cgm

size_t ca_global_scratch_bytes(int64_t maxN, int q) {
  const int Q = q <= 32 ? 32 : (q <= 64 ? 64 : (q <= 96 ? 96 : 128));
  return (size_t)2 * maxN * Q * 8 + (size_t)maxN + 2 * 160 * (sizeof(cgm::Trip) + 4) + 1024;
}

static int num_sms_g() {
  static int n = 0;
  if (!n) {
    int dev = 0;
    cudaGetDevice(&dev);
    cudaDeviceGetAttribute(&n, cudaDevAttrMultiProcessorCount, dev);
  }
  return n;
}

template <int Q, int TPR>
static cudaError_t launch_gm_t(CAArgs a, int64_t nb, int64_t maxN, void *scratch, cudaStream_t st, Prof *pf) {
  using namespace cgm;
  char *p = reinterpret_cast<char *>((((uintptr_t)scratch) + 255) & ~(uintptr_t)255);
  GmArgs g{};
  g.gB = reinterpret_cast<double *>(p);
  p += (size_t)maxN * Q * 8;
  g.gC = reinterpret_cast<double *>(p);
  p += (size_t)maxN * Q * 8;
  g.gtri = reinterpret_cast<Trip *>(p);
  p += 2 * 160 * sizeof(Trip);
  g.gx = reinterpret_cast<unsigned *>(p);
  p += 2 * 160 * 4;
  g.inS = reinterpret_cast<unsigned char *>(p);
  const bool qeq = a.q == Q;
  void (*kern)(CAArgs, GmArgs) = a.op.kind == LRA_OP_FACTORED_CSR ? (qeq ? k_cagm<Q, TPR, 2, true> : k_cagm<Q, TPR, 2>)
                                 : (a.op.dtype == LRA_F64 ? (qeq ? k_cagm<Q, TPR, 1, true> : k_cagm<Q, TPR, 1>)
                                                          : (qeq ? k_cagm<Q, TPR, 0, true> : k_cagm<Q, TPR, 0>));
  const size_t smem = (size_t)Q * Q * 8;
  cudaError_t e = cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
  if (e != cudaSuccess) return e;
  int per_sm = 0;
  e = cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, kern, NT, smem);
  if (e != cudaSuccess) return e;
  if (per_sm < 1) return cudaErrorInvalidConfiguration;
  const int grid = num_sms_g() < 160 ? num_sms_g() : 160;
  for (int64_t b = 0; b < nb; ++b) {
    CAArgs rb = a;
    if (rb.op.kind == LRA_OP_DENSE) rb.op.w = (const char *)rb.op.w + b * rb.w_stride * (rb.op.dtype == LRA_F32 ? 4 : 8);
    if (rb.Y) rb.Y = (const char *)rb.Y + b * rb.y_stride * 8;
    if (rb.I0) rb.I0 += b * rb.i0_stride;
    rb.I += b * a.q;
    rb.J += b * a.q;
    if (rb.stats) rb.stats += b;
    rb.status += b;
    if (rb.yinfo) rb.yinfo += 4 * b;
    cudaLaunchConfig_t cfg = {};
    cfg.gridDim = dim3((unsigned)grid);
    cfg.blockDim = dim3(NT);
    cfg.dynamicSmemBytes = smem;
    cfg.stream = st;
    cudaLaunchAttribute attr[1];
    attr[0].id = cudaLaunchAttributeCooperative;
    attr[0].val.cooperative = 1;
    cfg.attrs = attr;
    cfg.numAttrs = 1;
    pf->begin("k_ca_global", st);
    e = cudaLaunchKernelEx(&cfg, kern, rb, g);
    pf->end(st);
    if (e != cudaSuccess) return e;
  }
  return cudaSuccess;
}

// Global-memory tier (any N, q <= 128).  scratch: ca_global_scratch_bytes(maxN, q).
cudaError_t launch_ca_global(CAArgs a, int64_t nb, int64_t maxN, void *scratch, cudaStream_t st, Prof *pf) {
  if (a.q <= 32) return launch_gm_t<32, 4>(a, nb, maxN, scratch, st, pf);
  if (a.q <= 64) return launch_gm_t<64, 8>(a, nb, maxN, scratch, st, pf);
  if (a.q <= 96) return launch_gm_t<96, 16>(a, nb, maxN, scratch, st, pf);
  if (a.q <= 128) return launch_gm_t<128, 16>(a, nb, maxN, scratch, st, pf);
  return cudaErrorInvalidConfiguration;
}

cudaError_t read_gm_exact(unsigned long long *out, bool reset) {
  cudaError_t e = cudaMemcpyFromSymbol(out, cgm::g_gm_exact, sizeof(unsigned long long));
  if (e == cudaSuccess && reset) {
    unsigned long long z = 0;
    e = cudaMemcpyToSymbol(cgm::g_gm_exact, &z, sizeof(z));
  }
  return e;
}

}  // namespace lra
