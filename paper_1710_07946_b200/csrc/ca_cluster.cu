// ca_cluster.cu — cluster tier of the real C-A kernel (stages 2-3 of Alg 10.2 with C-A
// iterations, Remark rerfnhmt), engineered for the latency of one pivot step.
//
// Method and arithmetic are those of ca.cu's register-row kernel, so outputs are identical:
// maxvol = Alg D.2 stage 1 (LUP cold start with the slack pivot rule, reading C11, one IEEE
// multiply + one subtract per update so the pivots are bit-identical to the oracle's,
// P:6550-6556) or a warm start from the current slots, then the Alg D.1 swap loop
// with the rank-1 update C <- C - C[:,j*](C[i*,:] - e_j*)/c_{i*j*}.
// C = B * G^{-1} (G = B[S,:]) with G^{-1} from a Gauss-Jordan inverse (cold) or from the
// carried inverse of the previous C-A step, transposed and Newton-refined (warm).
//
// What is new is the schedule.  One cluster of CS CTAs per problem, one block row per TPR
// threads held in registers (W = Q/TPR doubles per thread).  A pivot decision costs
//   warp max (redux) + warp first index -> ONE __syncthreads -> every warp forms the CTA
//   triple (max key, first index, ambiguity flag) -> warp 0 pushes it into every CTA's
//   shared memory while the owner threads publish their row -> ONE cluster barrier ->
//   every warp decides redundantly -> warp 0 pulls the winning row -> ONE __syncthreads.
// The smallest-index rule among |c| >= (1-tau) max is exact: a unit (warp or CTA) whose
// own maximum lies inside the tie window of the global maximum without being equal to it
// may hold a smaller qualifying index than its candidate; that flags the decision
// ambiguous and a second, exact round with the global threshold is run (rare).
// The inverse work (Gauss-Jordan in place, Newton products) uses a q x q register/shared
// layout with no padding beyond the next multiple of 16 rows / 32 columns.
#include <cooperative_groups.h>
#include <climits>
#include <cstdlib>

#include "kernels.cuh"

namespace cg = cooperative_groups;

#ifndef CC_PAIR_PRODUCT
#define CC_PAIR_PRODUCT 1   // k_cacl2: row-pair blocked C = B G^{-1}
#endif

namespace lra {

// phase counters (clock64 cycles of CTA 0 / thread 0, summed over problems):
// 0 loads, 1 cold LU, 2 warm gather + Newton, 3 Gauss-Jordan, 4 product, 5 swap loops,
// 6 whole kernel, 7 pivot steps (count), 8 exact second rounds (count)
__device__ unsigned long long g_cc_cyc[16];
#define CC_MARK(kk) do { if (threadIdx.x == 0 && k.rank == 0) { long long _n = clock64(); atomicAdd(&g_cc_cyc[kk], (unsigned long long)(_n - _tm)); _tm = _n; } } while (0)

namespace ccl {

constexpr int NT = 512;
constexpr int NW = NT / 32;

struct __align__(16) Trip {
  unsigned long long key;   // max key of the CTA
  unsigned idx;             // CTA candidate (smallest linear index >= (1-tau) * CTA max)
  unsigned amb;             // the candidate may be inexact under a lower (global) threshold
};

template <int Q>
struct Sh {
  long long S[2][Q];                  // [0]: I slots, [1]: J slots
  unsigned long long wkey[2][NW];
  unsigned widx[2][NW];
  Trip xin[2][16];                    // pushed by every CTA of the cluster (slot = rank)
  unsigned xi2[2][16];                // second (exact) round
  __align__(16) double pub[2][Q];     // this CTA's candidate row
  __align__(16) double prow[Q];       // winning row
  __align__(16) double pm[Q];         // update row (LU: masked; swap: prow - e_j*)
  double rc;                          // 1 / c_{i*j*}
  unsigned long long gk[2][NW];       // Gauss-Jordan pivot candidates
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
__device__ __forceinline__ void cluster_sync_all() {
  asm volatile("barrier.cluster.arrive.release.aligned;\n\tbarrier.cluster.wait.acquire.aligned;\n" ::: "memory");
}
template <typename T>
__device__ __forceinline__ T *rmap(T *p, int rank) {
  return cg::this_cluster().map_shared_rank(p, rank);
}
// r[w] for a warp-uniform w (jump table: no select chain over the register array)
template <int W>
__device__ __forceinline__ double rsel(const double (&r)[W], int w) {
  double v = 0.0;
#pragma unroll
  for (int i = 0; i < W; ++i)
    if (i == w) v = r[i];
  return v;
}

template <int Q>
struct Kx {
  Sh<Q> *sh;
  int cs, rank, lane, warp, par;
  double tau;
};

struct Dec {
  double M;
  unsigned idx;
  int owner;
  bool amb;
};

// Round 1 of a pivot decision (see the header).  mloc < 0: no candidate in this thread.
template <int Q, class First, class Pub>
__device__ __forceinline__ Dec pick(Kx<Q> &k, double mloc, First first, Pub publish, int &p) {
  Sh<Q> &sh = *k.sh;
  long long _tm = clock64();
  p = k.par;
  k.par ^= 1;
  const unsigned long long wk = wmaxk(dkey(mloc));
  unsigned ci = 0xffffffffu;
  if (wk) {
    const double thr = (1.0 - k.tau) * kdbl(wk);
    if (mloc >= thr) ci = first(thr);
  }
  ci = wminu(ci);
  if (k.lane == 0) {
    sh.wkey[p][k.warp] = wk;
    sh.widx[p][k.warp] = ci;
  }
  __syncthreads();
  const unsigned long long ck = k.lane < NW ? sh.wkey[p][k.lane] : 0ull;
  const unsigned cx = k.lane < NW ? sh.widx[p][k.lane] : 0xffffffffu;
  const unsigned long long Ck = wmaxk(ck);
  const double Cthr = (1.0 - k.tau) * kdbl(Ck);
  const unsigned Cidx = wminu(ck == Ck ? cx : 0xffffffffu);
  const bool Camb = __any_sync(0xffffffffu, ck != Ck && ck != 0ull && kdbl(ck) >= Cthr);
  publish(p, Cidx);
  Dec d;
  CC_MARK(9);
  if (k.cs > 1) {
    if (k.warp == 0 && k.lane < k.cs) *rmap(&sh.xin[p][k.rank], k.lane) = Trip{Ck, Cidx, Camb ? 1u : 0u};
    cluster_sync_all();
    CC_MARK(10);
    const bool in = k.lane < k.cs;
    const Trip t = in ? sh.xin[p][k.lane] : Trip{0ull, 0xffffffffu, 0u};
    const unsigned long long Gk = wmaxk(t.key);
    const double Gthr = (1.0 - k.tau) * kdbl(Gk);
    const bool top = in && t.key == Gk;
    d.idx = wminu(top ? t.idx : 0xffffffffu);
    d.amb = __any_sync(0xffffffffu, (top && t.amb) || (in && t.key != Gk && t.key != 0ull && kdbl(t.key) >= Gthr));
    const unsigned bal = __ballot_sync(0xffffffffu, top && t.idx == d.idx);
    d.owner = bal ? __ffs(bal) - 1 : 0;
    d.M = kdbl(Gk);
    CC_MARK(11);
  } else {
    __syncthreads();
    d.M = kdbl(Ck);
    d.idx = Cidx;
    d.amb = Camb;
    d.owner = 0;
  }
  return d;
}

// Exact second round: smallest linear index with value >= (1-tau) M over the whole problem.
template <int Q, class First, class Pub>
__device__ __forceinline__ Dec pick_exact(Kx<Q> &k, double mloc, double M, First first, Pub publish, int &p) {
  Sh<Q> &sh = *k.sh;
  p = k.par;
  k.par ^= 1;
  const double thr = (1.0 - k.tau) * M;
  unsigned ci = mloc >= thr ? first(thr) : 0xffffffffu;
  ci = wminu(ci);
  if (k.lane == 0) sh.widx[p][k.warp] = ci;
  __syncthreads();
  const unsigned Cidx = wminu(k.lane < NW ? sh.widx[p][k.lane] : 0xffffffffu);
  publish(p, Cidx);
  Dec d;
  d.M = M;
  d.amb = false;
  if (k.cs > 1) {
    if (k.warp == 0 && k.lane < k.cs) *rmap(&sh.xi2[p][k.rank], k.lane) = Cidx;
    cluster_sync_all();
    const unsigned t = k.lane < k.cs ? sh.xi2[p][k.lane] : 0xffffffffu;
    d.idx = wminu(t);
    const unsigned bal = __ballot_sync(0xffffffffu, k.lane < k.cs && t == d.idx);
    d.owner = bal ? __ffs(bal) - 1 : 0;
  } else {
    __syncthreads();
    d.idx = Cidx;
    d.owner = 0;
  }
  if (threadIdx.x == 0 && k.rank == 0) atomicAdd(&g_cc_cyc[8], 1ull);
  return d;
}

// warp 0 copies the winning row (owner CTA's pub[p]) into prow and prepares pm / rc.
template <int Q, class Prep>
__device__ __forceinline__ void take_row(Kx<Q> &k, const Dec &d, int p, int q, Prep prep) {
  long long _tm = clock64();
  if (k.warp == 0) {
    const double *src = k.cs > 1 ? rmap(&k.sh->pub[p][0], d.owner) : &k.sh->pub[p][0];
    double x[(Q + 31) / 32];
#pragma unroll
    for (int u = 0; u < (Q + 31) / 32; ++u) {
      const int j = k.lane + 32 * u;
      x[u] = j < q ? src[j] : 0.0;
    }
#pragma unroll
    for (int u = 0; u < (Q + 31) / 32; ++u) {
      const int j = k.lane + 32 * u;
      if (j < Q) {
        k.sh->prow[j] = x[u];
        prep(j, x[u]);
      }
    }
  }
  __syncthreads();
  CC_MARK(12);
}

template <int OPK>
__device__ __forceinline__ double op_at(const OpView &op, int64_t i, int64_t j) {
  if (OPK == 0) return (double)__ldg((const float *)op.w + j * op.ldw + i);
  if (OPK == 1) return __ldg((const double *)op.w + j * op.ldw + i);
  return op.f.at(i, j);
}

#define CC_T0() long long _t0 = clock64()
#define CC_T1(kk) do { if (threadIdx.x == 0 && k.rank == 0) atomicAdd(&g_cc_cyc[kk], (unsigned long long)(clock64() - _t0)); } while (0)

// Gauss-Jordan inverse in place (bit-identical to the augmented [G | I] elimination of
// ca.cu): thread (warp w, lane l) holds G[w + 16 a][l + 32 c].  Step s picks the unused row
// p_s of max |G[., s]| (first on ties, NaN largest), scales it and eliminates column s;
// slot s then holds the right-part column p_s.  Result X = G^{-1} (row stride Q, columns
// >= q zero) in Xo.  False if singular.
template <int Q>
__device__ __forceinline__ bool gj_inplace(Kx<Q> &k, const long long *S, int q, int rpc, const double *Cs, int QP,
                                           double *Xo) {
  constexpr int KR = (Q + 15) / 16, MC = (Q + 31) / 32;
  Sh<Q> &sh = *k.sh;
  double x[KR][MC];
#pragma unroll
  for (int a = 0; a < KR; ++a) {
    const int r = k.warp + 16 * a;
    const long long sr = r < q ? S[r] : 0;
    const double *src = Cs + (size_t)(sr % rpc) * QP;
    if (k.cs > 1 && r < q) src = rmap(const_cast<double *>(src), (int)(sr / rpc));
#pragma unroll
    for (int c = 0; c < MC; ++c) {
      const int col = k.lane + 32 * c;
      x[a][c] = (r < q && col < q) ? src[col] : 0.0;
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
      const int r = k.warp + 16 * a;
      if (r < q && !((used >> a) & 1u)) {
        const double av = fabs(v[a]);
        const unsigned long long kk = (av != av) ? 0x7ff8000000000000ull : dkey(av);
        if (arow == 0x7fffffff || kk > key) {
          key = kk;
          arow = r;
        }
      }
    }
    if (k.lane == 0) {
      sh.gk[sl][k.warp] = key;
      sh.gr[sl][k.warp] = arow;
    }
    __syncthreads();
    const unsigned long long ck = k.lane < NW ? sh.gk[sl][k.lane] : 0ull;
    const int cr = k.lane < NW ? sh.gr[sl][k.lane] : 0x7fffffff;
    const unsigned long long mk = wmaxk(ck);
    const int p = (int)__reduce_min_sync(0xffffffffu, (ck == mk && cr != 0x7fffffff) ? (unsigned)cr : 0xffffffffu);
    if (p >= q) return false;
    const int ap = p >> 4;
    if (threadIdx.x == 0) sh.piv[s] = p;
    if (k.warp == (p & 15)) {
      double d = v[0];
#pragma unroll
      for (int a = 1; a < KR; ++a) d = (ap == a) ? v[a] : d;
      const double rd = 1.0 / d;
#pragma unroll
      for (int c = 0; c < MC; ++c) {
        const int col = k.lane + 32 * c;
        double xv = x[0][c];
#pragma unroll
        for (int a = 1; a < KR; ++a) xv = (ap == a) ? x[a][c] : xv;
        if (col < Q) sh.gp[col] = (col == s) ? rd : xv * rd;
      }
      if (k.lane == 0) sh.gd = d;
    }
    __syncthreads();
    const double d = sh.gd;
    if (!(fabs(d) > 0.0) || !isfinite(d)) return false;
#pragma unroll
    for (int a = 0; a < KR; ++a) {
      const int r = k.warp + 16 * a;
      const bool isp = (r == p);
      if (isp) used |= 1u << a;
#pragma unroll
      for (int c = 0; c < MC; ++c) {
        const int col = k.lane + 32 * c;
        const double pv = col < Q ? sh.gp[col] : 0.0;
        x[a][c] = isp ? pv : ((col == s) ? fma(-v[a], pv, 0.0) : fma(-v[a], pv, x[a][c]));
      }
    }
  }
  // X[t][piv[t']] = M[piv[t]][t']
  if (threadIdx.x < q) sh.pinv[sh.piv[threadIdx.x]] = threadIdx.x;
  __syncthreads();
#pragma unroll
  for (int a = 0; a < KR; ++a) {
    const int r = k.warp + 16 * a;
    if (r >= q) continue;
    const int t = sh.pinv[r];
#pragma unroll
    for (int c = 0; c < MC; ++c) {
      const int col = k.lane + 32 * c;
      if (col < q) Xo[t * Q + sh.piv[col]] = x[a][c];
      else if (col < Q) Xo[t * Q + col] = 0.0;
    }
  }
  __syncthreads();
  return true;
}

// out = base + sg * (L * R) on q x q parts (row stride Q); base = I if bp == nullptr.
// acc is the fma chain over t ascending from 0, then out = fma(sg, acc, base) (as ca.cu).
template <int Q>
__device__ __forceinline__ void mm_part(Kx<Q> &k, int q, double *out, const double *L, const double *R,
                                        const double *bp, double sg) {
  constexpr int KR = (Q + 15) / 16, MC = (Q + 31) / 32;
  double acc[KR][MC];
#pragma unroll
  for (int a = 0; a < KR; ++a)
#pragma unroll
    for (int c = 0; c < MC; ++c) acc[a][c] = 0.0;
  for (int t = 0; t < q; ++t) {
    double rv[MC];
#pragma unroll
    for (int c = 0; c < MC; ++c) {
      const int col = k.lane + 32 * c;
      rv[c] = col < Q ? R[t * Q + col] : 0.0;
    }
#pragma unroll
    for (int a = 0; a < KR; ++a) {
      const int r = k.warp + 16 * a;
      const double l = r < Q ? L[r * Q + t] : 0.0;
#pragma unroll
      for (int c = 0; c < MC; ++c) acc[a][c] = fma(l, rv[c], acc[a][c]);
    }
  }
  __syncthreads();    // out may alias an input part
#pragma unroll
  for (int a = 0; a < KR; ++a) {
    const int r = k.warp + 16 * a;
    if (r >= q) continue;
#pragma unroll
    for (int c = 0; c < MC; ++c) {
      const int col = k.lane + 32 * c;
      if (col >= Q) continue;
      double v = 0.0;
      if (col < q) {
        const double bv = bp ? bp[r * Q + col] : (r == col ? 1.0 : 0.0);
        v = fma(sg, acc[a][c], bv);
      }
      out[r * Q + col] = v;
    }
  }
  __syncthreads();
}

// Steps: 0 = stage 2 on a real sketch Y (cold); then 2L+1 = horizontal step of loop L
// (J <- maxvol(W[I,:]^T), cold in loop 0), 2L+2 = vertical step (I <- maxvol(W[:,J]), warm).
template <int Q, int TPR, int OPK, bool QEQ = false>
__global__ void __launch_bounds__(NT, 1) k_cacl(CAArgs a) {
  if (a.skip && (a.skip[0] != 0 || a.skip[1] != 0)) return;   // row-sharded chain: step not needed
  constexpr int W = Q / TPR, QP = Q | 1;
  static_assert(W % 2 == 0 || W == 1, "W even");
  extern __shared__ __align__(16) unsigned char dsm[];
  __shared__ Sh<Q> sh;
  const int rpc = a.rpc;
  double *Cs = reinterpret_cast<double *>(dsm);
  double *Xp = Cs + (((size_t)rpc * QP + 1) & ~(size_t)1);
  Kx<Q> k;
  k.sh = &sh;
  k.cs = a.cs;
  k.rank = a.cs > 1 ? (int)cg::this_cluster().block_rank() : 0;
  k.lane = threadIdx.x & 31;
  k.warp = threadIdx.x >> 5;
  k.par = 0;
  k.tau = a.tau;
  const double tol = a.tol;
  const int q = QEQ ? Q : a.q;           // QEQ: q == Q known at compile time (loops fold)
  const int64_t b = blockIdx.x / a.cs;
  OpView op = a.op;
  if (op.kind == LRA_OP_DENSE) op.w = (const char *)op.w + b * a.w_stride * (op.dtype == LRA_F32 ? 4 : 8);
  const int ri = threadIdx.x / TPR, sub = threadIdx.x % TPR, jb = sub * W;
  const int64_t r0 = (int64_t)k.rank * rpc;
  int32_t status = LRA_OK;
  int lu = 0, swaps = 0, caps = 0, sk_swaps = 0, loops = 0, sw_h = 0;
  double cert_r = 0.0, cert_c = 0.0;
  const bool yreal = a.Y != nullptr && !a.y_complex;
  if (!yreal || a.y_warm) {
    if (threadIdx.x < q) sh.S[0][threadIdx.x] = a.I0[b * a.i0_stride + threadIdx.x];
    if (a.yinfo) {
      status = a.yinfo[4 * b + 0];
      swaps = sk_swaps = a.yinfo[4 * b + 1];
      caps = a.yinfo[4 * b + 2];
      lu = a.yinfo[4 * b + 3];
    }
  }
  if (threadIdx.x < Q) sh.pm[threadIdx.x] = 0.0;
  // zero the inverse parts (padding columns stay zero)
  for (int e = threadIdx.x; e < 3 * Q * Q; e += NT) Xp[e] = 0.0;
  __syncthreads();
  const double *Y = yreal ? reinterpret_cast<const double *>(a.Y) + b * a.y_stride : nullptr;
  const int last = 2 * a.sweeps;
  int ib = 0;                 // part holding the carried G^{-1}
  long long _tk = clock64();
  for (int step = yreal ? 0 : 1; status == LRA_OK && step <= last; ++step) {
    const int kind = step == 0 ? 0 : ((step & 1) ? 1 : 2);   // 0 = Y, 1 = h, 2 = v
    const int64_t N = kind == 1 ? op.n : op.m;
    long long *S = kind == 1 ? sh.S[1] : sh.S[0];
    const bool fresh = step <= 1;                     // G^{-1} by Gauss-Jordan (no carried inverse)
    const bool cold = fresh && !(step == 0 && a.y_warm);   // LUP cold start
    // the inverse is carried only into a following warm step
    const bool carry = step >= 1 && step < last;
    const int nloc = (int)max((int64_t)0, min((int64_t)rpc, N - r0));
    if (k.cs > 1) cluster_sync_all(); else __syncthreads();    // previous block no longer read
    {
      CC_T0();
      const long long *I = sh.S[0], *J = sh.S[1];
      const int tot = nloc * q;
      for (int e0 = threadIdx.x; e0 < tot; e0 += 8 * NT) {
        double v[8];
#pragma unroll
        for (int u = 0; u < 8; ++u) {
          const int e = e0 + u * NT;
          v[u] = 0.0;
          if (e < tot) {
            const int i = e % nloc, j = e / nloc;
            if (kind == 0) v[u] = __ldg(Y + (int64_t)j * a.ldy + r0 + i);
            else if (kind == 1) {
              long long ii = I[j];
              LRA_CHKIDX(5, b, ii, op.m);
              v[u] = op_at<OPK>(op, ii, r0 + i);
            } else {
              long long jj = J[j];
              LRA_CHKIDX(6, b, jj, op.n);
              v[u] = op_at<OPK>(op, r0 + i, jj);
            }
          }
        }
#pragma unroll
        for (int u = 0; u < 8; ++u) {
          const int e = e0 + u * NT;
          if (e < tot) Cs[(size_t)(e % nloc) * QP + e / nloc] = v[u];
        }
      }
      __syncthreads();
      CC_T1(0);
    }
    const bool has = ri < nloc;
    const long long grow = r0 + ri;
    const double *Crow = Cs + (size_t)ri * QP;
    double row[W];
    int myslot = -1;
    int nsw = 0;
    bool ok = true;
    double cert = 0.0;
    bool cap_hit = false;
    if (cold) {
      CC_T0();
#pragma unroll
      for (int w = 0; w < W; ++w) row[w] = (has && jb + w < q) ? Crow[jb + w] : 0.0;
      // ---- Alg D.2 stage 1: LUP with the slack pivot rule (bit-identical to the oracle)
      for (int t = 0; t < q && ok; ++t) {
        const int st = t / W, wt = t - st * W;
        double x = rsel<W>(row, wt);
        if (TPR > 1) x = __shfl_sync(0xffffffffu, x, (k.lane & ~(TPR - 1)) | st);
        const double val = (has && myslot < 0) ? ((x != x) ? INFINITY : fabs(x)) : -1.0;
        auto first = [&](double) -> unsigned { return (unsigned)grow; };
        auto publish = [&](int p, unsigned cidx) {
          if (has && (unsigned)grow == cidx) {
#pragma unroll
            for (int w = 0; w < W; ++w) sh.pub[p][jb + w] = row[w];
          }
        };
        int p;
        Dec d = pick(k, val, first, publish, p);
        if (d.amb) d = pick_exact(k, val, d.M, first, publish, p);
        if (!(d.M > 0.0) || !isfinite(d.M)) { ok = false; break; }
        take_row(k, d, p, q, [&](int j, double xv) { sh.pm[j] = j > t ? xv : 0.0; });
        const long long piv = d.idx;
        if (threadIdx.x == 0) S[t] = piv;
        if (has && grow == piv) myslot = t;
        if (has && myslot < 0) {
          const double f = x / sh.prow[t];
#pragma unroll
          for (int w = 0; w < W; ++w) row[w] = rsub_mul(row[w], f, sh.pm[jb + w]);
        }
      }
      __syncthreads();
      CC_T1(1);
      if (!ok) { status = LRA_ESINGULAR; break; }
      lu += q;
    } else if (has) {
      for (int s2 = 0; s2 < q; ++s2)
        if (S[s2] == grow) myslot = s2;
    }
    if (fresh) {
      // ---- G = B[S,:] (original rows, owners' shared memory) -> G^{-1} in part 0
      if (!cold && k.cs > 1) cluster_sync_all();        // every CTA's block rows are loaded
      {
        CC_T0();
        ib = 0;
        ok = gj_inplace<Q>(k, S, q, rpc, Cs, QP, Xp);
        CC_T1(3);
      }
      if (!ok) { status = LRA_ESINGULAR; break; }
    } else {
      CC_T0();
      // carried X0 = (G_prev^{-1})^T, one Newton step against the freshly gathered G
      const int cur = ib, pa = (ib + 1) % 3, pb = (ib + 2) % 3;
      double *Xc = Xp + cur * Q * Q, *Xa = Xp + pa * Q * Q, *Xb = Xp + pb * Q * Q;
      for (int e = threadIdx.x; e < q * q; e += NT) {
        const int r = e / q, c = e % q;
        Xa[r * Q + c] = Xc[c * Q + r];
      }
      if (k.cs > 1) cluster_sync_all(); else __syncthreads();  // every CTA's block rows are loaded
      constexpr int KR = (Q + 15) / 16, MC = (Q + 31) / 32;
#pragma unroll
      for (int aa = 0; aa < KR; ++aa) {
        const int r = k.warp + 16 * aa;
        if (r >= q) continue;
        const long long sr = S[r];
        const double *src = Cs + (size_t)(sr % rpc) * QP;
        if (k.cs > 1) src = rmap(const_cast<double *>(src), (int)(sr / rpc));
#pragma unroll
        for (int c = 0; c < MC; ++c) {
          const int col = k.lane + 32 * c;
          if (col < q) Xb[r * Q + col] = src[col];
        }
      }
      __syncthreads();
      mm_part<Q>(k, q, Xc, Xb, Xa, nullptr, -1.0);      // R  = I - G X0   -> cur
      mm_part<Q>(k, q, Xb, Xa, Xc, Xa, 1.0);            // X1 = X0 + X0 R  -> pb
      ib = pb;
      CC_T1(2);
    }
    // ---- C = B G^{-1} for the rows outside S
    {
      CC_T0();
      const double *X = Xp + ib * Q * Q;
#if CC_PAIR_PRODUCT
      if constexpr (W >= 4 && W % 4 == 0) {
        // row pairs (ri, ri ^ 1), as in k_cacl2: each X value from shared memory feeds two FMAs,
        // the halves are swapped with the pair partner (lane ^ TPR); same FMA chains
        constexpr int H = W / 2;
        const int h = (k.lane / TPR) & 1;
        const int rp = ri ^ 1;
        const bool hp = rp < nloc;
        const double *Prow = Cs + (size_t)(hp ? rp : 0) * QP;
        double a0[H], a1[H];
#pragma unroll
        for (int w = 0; w < H; ++w) a0[w] = a1[w] = 0.0;
        for (int t = 0; t < q; ++t) {
          const double b0 = has ? Crow[t] : 0.0, b1 = hp ? Prow[t] : 0.0;
          const double2 *xr = reinterpret_cast<const double2 *>(X + t * Q + jb + h * H);
#pragma unroll
          for (int w = 0; w < H / 2; ++w) {
            const double2 xv = xr[w];
            a0[2 * w] = fma(b0, xv.x, a0[2 * w]);
            a0[2 * w + 1] = fma(b0, xv.y, a0[2 * w + 1]);
            a1[2 * w] = fma(b1, xv.x, a1[2 * w]);
            a1[2 * w + 1] = fma(b1, xv.y, a1[2 * w + 1]);
          }
        }
        const bool live = has && myslot < 0;
#pragma unroll
        for (int w = 0; w < H; ++w) {
          const double o = __shfl_xor_sync(0xffffffffu, a1[w], TPR);
          row[w] = live ? (h == 0 ? a0[w] : o) : 0.0;
          row[H + w] = live ? (h == 0 ? o : a0[w]) : 0.0;
        }
      } else
#endif
      {
#pragma unroll
      for (int w = 0; w < W; ++w) row[w] = 0.0;
      if (has && myslot < 0) {
        for (int t = 0; t < q; ++t) {
          const double bt = Crow[t];
          if (W >= 2) {
            const double2 *xr = reinterpret_cast<const double2 *>(X + t * Q + jb);
#pragma unroll
            for (int w = 0; w < W / 2; ++w) {
              const double2 xv = xr[w];
              row[2 * w] = fma(bt, xv.x, row[2 * w]);
              row[2 * w + 1] = fma(bt, xv.y, row[2 * w + 1]);
            }
          } else {
            row[0] = fma(bt, X[t * Q + jb], row[0]);
          }
        }
      }
      }
      CC_T1(4);
    }
    double rmx = 0.0;
#pragma unroll
    for (int w = 0; w < W; ++w) rmx = fmax(rmx, fabs(row[w]));
    // ---- Alg D.1 swap loop
    {
      CC_T0();
      double *Xi = Xp + ib * Q * Q;
      for (;;) {
        const double mloc = (has && myslot < 0) ? rmx : -1.0;
        auto first = [&](double thr) -> unsigned {
          unsigned res = 0xffffffffu;
#pragma unroll
          for (int w = W - 1; w >= 0; --w)
            if (jb + w < q && fabs(row[w]) >= thr) res = (unsigned)(grow * q + jb + w);
          return res;
        };
        auto publish = [&](int p, unsigned cidx) {
          if (has && cidx != 0xffffffffu && (unsigned)grow == cidx / (unsigned)q) {
#pragma unroll
            for (int w = 0; w < W; ++w) sh.pub[p][jb + w] = row[w];
          }
        };
        int p;
        Dec d = pick(k, mloc, first, publish, p);
        if (!(d.M == d.M)) { ok = false; break; }
        if (d.M <= 1.0 + tol || nsw >= a.cap) {
          cert = fmax(d.M, 0.0);
          cap_hit = d.M > 1.0 + tol;
          break;
        }
        if (d.amb) d = pick_exact(k, mloc, d.M, first, publish, p);
        const long long istar = d.idx / (unsigned)q;
        const int jstar = (int)(d.idx % (unsigned)q);
        take_row(k, d, p, q, [&](int j, double xv) {
          sh.pm[j] = (j == jstar) ? xv - 1.0 : xv;
          if (j == jstar) sh.rc = 1.0 / xv;
        });
        long long _tm = clock64();
        if (threadIdx.x == 0) S[jstar] = istar;
        if (has && myslot == jstar) {                    // leaves S: explicit row e_{j*}
          myslot = -1;
#pragma unroll
          for (int w = 0; w < W; ++w) row[w] = (jb + w == jstar) ? 1.0 : 0.0;
        }
        if (has && grow == istar) myslot = jstar;        // enters S
        const int sj = jstar / W, wj = jstar - sj * W;
        double xj = rsel<W>(row, wj);
        if (TPR > 1) xj = __shfl_sync(0xffffffffu, xj, (k.lane & ~(TPR - 1)) | sj);
        const double rc = sh.rc;
        rmx = 0.0;
        if (has && myslot < 0) {            // C <- C - C[:,j*] (C[i*,:] - e_j*) / c
          const double g = xj * rc;
#pragma unroll
          for (int w = 0; w < W; ++w) {
            row[w] = fma(-g, sh.pm[jb + w], row[w]);
            rmx = fmax(rmx, fabs(row[w]));
          }
        }
        if (carry) {                          // the same update of the carried G^{-1}
          constexpr int KR = (Q + 15) / 16, MC = (Q + 31) / 32;
#pragma unroll
          for (int aa = 0; aa < KR; ++aa) {
            const int r = k.warp + 16 * aa;
            if (r >= q) continue;
            double *ir = Xi + r * Q;
            const double gg = ir[jstar] * rc;
            __syncwarp();
#pragma unroll
            for (int c = 0; c < MC; ++c) {
              const int col = k.lane + 32 * c;
              if (col < q) ir[col] = fma(-gg, sh.pm[col], ir[col]);
            }
          }
        }
        CC_MARK(13);
        ++nsw;
      }
      if (threadIdx.x == 0 && k.rank == 0) atomicAdd(&g_cc_cyc[7], (unsigned long long)(nsw + (cold ? q : 0)));
      CC_T1(5);
    }
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
      if (step > 2 && sw_h == 0 && nsw == 0) break;           // fixed point (reading C13)
    }
  }
  __syncthreads();
  if (threadIdx.x == 0 && k.rank == 0) atomicAdd(&g_cc_cyc[6], (unsigned long long)(clock64() - _tk));
  if (k.rank == 0) {
    if (threadIdx.x < q) {
      a.I[b * q + threadIdx.x] = sh.S[0][threadIdx.x];
      a.J[b * q + threadIdx.x] = sh.S[1][threadIdx.x];
    }
    if (threadIdx.x == 0) {
      a.status[b] = status;
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
        s.min_pivot_margin = __longlong_as_double(0x7ff8000000000000LL);
        a.stats[b] = s;
      }
    }
  }
  if (k.cs > 1) cluster_sync_all();   // keep every CTA's shared memory alive until done
}


// ============================================================================================
// k_cacl2: the same method, schedule and arithmetic with TWO rows per row-group of threads —
// slot A in registers (as k_cacl) and slot B in shared memory — so a CTA holds 2 NT / TPR
// rows and a problem needs half the CTAs (config 2: 8-CTA clusters instead of 16: 15 problems
// co-resident instead of 7).  The block B itself is no longer staged in shared memory: its
// entries are read from global memory / L2 where needed (cold LUP start, G = B[S,:], and the
// product C = B G^{-1}).  Every decision, update and tie rule is that of k_cacl, applied to
// the union of both slots (slot A rows precede slot B rows in index order inside a CTA), so
// the pivots are bit-identical.
// --------------------------------------------------------------------------------------------

// entry (row, col) of the current block: kind 0 = sketch Y, 1 = W[I,:]^T, 2 = W[:,J]
template <int OPK>
struct BSrc {
  int kind;
  const double *Y;
  int64_t ldy;
  OpView op;
  const long long *I, *J;
  __device__ __forceinline__ double operator()(int64_t row, int col) const {
    if (kind == 0) return __ldg(Y + (int64_t)col * ldy + row);
    if (kind == 1) return op_at<OPK>(op, I[col], row);
    return op_at<OPK>(op, row, J[col]);
  }
};

// Gauss-Jordan in place as gj_inplace, with G = B[S,:] read through the block source.
template <int Q, class Src>
__device__ __forceinline__ bool gj_src(Kx<Q> &k, const long long *S, int q, const Src &bsrc, double *Xo) {
  constexpr int KR = (Q + 15) / 16, MC = (Q + 31) / 32;
  Sh<Q> &sh = *k.sh;
  double x[KR][MC];
#pragma unroll
  for (int a = 0; a < KR; ++a) {
    const int r = k.warp + 16 * a;
    const long long sr = r < q ? S[r] : 0;
#pragma unroll
    for (int c = 0; c < MC; ++c) {
      const int col = k.lane + 32 * c;
      x[a][c] = (r < q && col < q) ? bsrc(sr, col) : 0.0;
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
      const int r = k.warp + 16 * a;
      if (r < q && !((used >> a) & 1u)) {
        const double av = fabs(v[a]);
        const unsigned long long kk = (av != av) ? 0x7ff8000000000000ull : dkey(av);
        if (arow == 0x7fffffff || kk > key) {
          key = kk;
          arow = r;
        }
      }
    }
    if (k.lane == 0) {
      sh.gk[sl][k.warp] = key;
      sh.gr[sl][k.warp] = arow;
    }
    __syncthreads();
    const unsigned long long ck = k.lane < NW ? sh.gk[sl][k.lane] : 0ull;
    const int cr = k.lane < NW ? sh.gr[sl][k.lane] : 0x7fffffff;
    const unsigned long long mk = wmaxk(ck);
    const int p = (int)__reduce_min_sync(0xffffffffu, (ck == mk && cr != 0x7fffffff) ? (unsigned)cr : 0xffffffffu);
    if (p >= q) return false;
    const int ap = p >> 4;
    if (threadIdx.x == 0) sh.piv[s] = p;
    if (k.warp == (p & 15)) {
      double d = v[0];
#pragma unroll
      for (int a = 1; a < KR; ++a) d = (ap == a) ? v[a] : d;
      const double rd = 1.0 / d;
#pragma unroll
      for (int c = 0; c < MC; ++c) {
        const int col = k.lane + 32 * c;
        double xv = x[0][c];
#pragma unroll
        for (int a = 1; a < KR; ++a) xv = (ap == a) ? x[a][c] : xv;
        if (col < Q) sh.gp[col] = (col == s) ? rd : xv * rd;
      }
      if (k.lane == 0) sh.gd = d;
    }
    __syncthreads();
    const double d = sh.gd;
    if (!(fabs(d) > 0.0) || !isfinite(d)) return false;
#pragma unroll
    for (int a = 0; a < KR; ++a) {
      const int r = k.warp + 16 * a;
      const bool isp = (r == p);
      if (isp) used |= 1u << a;
#pragma unroll
      for (int c = 0; c < MC; ++c) {
        const int col = k.lane + 32 * c;
        const double pv = col < Q ? sh.gp[col] : 0.0;
        x[a][c] = isp ? pv : ((col == s) ? fma(-v[a], pv, 0.0) : fma(-v[a], pv, x[a][c]));
      }
    }
  }
  if (threadIdx.x < q) sh.pinv[sh.piv[threadIdx.x]] = threadIdx.x;
  __syncthreads();
#pragma unroll
  for (int a = 0; a < KR; ++a) {
    const int r = k.warp + 16 * a;
    if (r >= q) continue;
    const int t = sh.pinv[r];
#pragma unroll
    for (int c = 0; c < MC; ++c) {
      const int col = k.lane + 32 * c;
      if (col < q) Xo[t * Q + sh.piv[col]] = x[a][c];
      else if (col < Q) Xo[t * Q + col] = 0.0;
    }
  }
  __syncthreads();
  return true;
}

template <int Q, int TPR, int OPK, bool QEQ = false>
__global__ void __launch_bounds__(NT, 1) k_cacl2(CAArgs a) {
  if (a.skip && (a.skip[0] != 0 || a.skip[1] != 0)) return;   // row-sharded chain: step not needed
  constexpr int W = Q / TPR, RPH = NT / TPR;                  // RPH rows per slot per CTA
  static_assert(W % 2 == 0 || W == 1, "W even");
  extern __shared__ __align__(16) unsigned char dsm[];
  __shared__ Sh<Q> sh;
  double *SB = reinterpret_cast<double *>(dsm);               // slot B rows: SB[w * NT + tid]
  double *Xp = SB + (size_t)W * NT;                           // 3 q x q parts (row stride Q)
  Kx<Q> k;
  k.sh = &sh;
  k.cs = a.cs;
  k.rank = a.cs > 1 ? (int)cg::this_cluster().block_rank() : 0;
  k.lane = threadIdx.x & 31;
  k.warp = threadIdx.x >> 5;
  k.par = 0;
  k.tau = a.tau;
  const double tol = a.tol;
  const int q = QEQ ? Q : a.q;
  const int64_t b = blockIdx.x / a.cs;
  OpView op = a.op;
  if (op.kind == LRA_OP_DENSE) op.w = (const char *)op.w + b * a.w_stride * (op.dtype == LRA_F32 ? 4 : 8);
  const int tid = threadIdx.x;
  const int ri = tid / TPR, sub = tid % TPR, jb = sub * W;
  const int64_t r0 = (int64_t)k.rank * (2 * RPH);
  const long long growA = r0 + ri, growB = r0 + RPH + ri;   // slot A rows precede slot B rows
  int32_t status = LRA_OK;
  int lu = 0, swaps = 0, caps = 0, sk_swaps = 0, loops = 0, sw_h = 0;
  double cert_r = 0.0, cert_c = 0.0;
  const bool yreal = a.Y != nullptr && !a.y_complex;
  if (!yreal || a.y_warm) {
    if (tid < q) sh.S[0][tid] = a.I0[b * a.i0_stride + tid];
    if (a.yinfo) {
      status = a.yinfo[4 * b + 0];
      swaps = sk_swaps = a.yinfo[4 * b + 1];
      caps = a.yinfo[4 * b + 2];
      lu = a.yinfo[4 * b + 3];
    }
  }
  if (tid < Q) sh.pm[tid] = 0.0;
  for (int e = tid; e < 3 * Q * Q; e += NT) Xp[e] = 0.0;
  __syncthreads();
  const double *Yb = yreal ? reinterpret_cast<const double *>(a.Y) + b * a.y_stride : nullptr;
  const int last = 2 * a.sweeps;
  int ib = 0;
  long long _tk = clock64();
  for (int step = yreal ? 0 : 1; status == LRA_OK && step <= last; ++step) {
    const int kind = step == 0 ? 0 : ((step & 1) ? 1 : 2);   // 0 = Y, 1 = h, 2 = v
    const int64_t N = kind == 1 ? op.n : op.m;
    long long *S = kind == 1 ? sh.S[1] : sh.S[0];
    const bool fresh = step <= 1;
    const bool cold = fresh && !(step == 0 && a.y_warm);
    const bool carry = step >= 1 && step < last;
    BSrc<OPK> bsrc{kind, Yb, a.ldy, op, sh.S[0], sh.S[1]};
    const bool hasA = growA < N, hasB = growB < N;
    // every CTA is done with the previous block's slots / rows before they change
    if (k.cs > 1) cluster_sync_all(); else __syncthreads();
    double row[W];
    int myA = -1, myB = -1;
    int nsw = 0;
    bool ok = true;
    double cert = 0.0;
    bool cap_hit = false;
    if (cold) {
      // ---- Alg D.2 stage 1: LUP with the slack pivot rule over the rows of both slots
      CC_T0();
#pragma unroll
      for (int w = 0; w < W; ++w) {
        row[w] = (hasA && jb + w < q) ? bsrc(growA, jb + w) : 0.0;
        SB[w * NT + tid] = (hasB && jb + w < q) ? bsrc(growB, jb + w) : 0.0;
      }
      __syncthreads();
      for (int t = 0; t < q && ok; ++t) {
        const int st = t / W, wt = t - st * W;
        double xA = rsel<W>(row, wt);
        if (TPR > 1) xA = __shfl_sync(0xffffffffu, xA, (k.lane & ~(TPR - 1)) | st);
        const double xB = SB[wt * NT + ri * TPR + st];
        const double vA = (hasA && myA < 0) ? ((xA != xA) ? INFINITY : fabs(xA)) : -1.0;
        const double vB = (hasB && myB < 0) ? ((xB != xB) ? INFINITY : fabs(xB)) : -1.0;
        const double val = fmax(vA, vB);
        auto first = [&](double thr) -> unsigned {
          return vA >= thr ? (unsigned)growA : (unsigned)growB;
        };
        auto publish = [&](int p, unsigned cidx) {
          if (hasA && (unsigned)growA == cidx) {
#pragma unroll
            for (int w = 0; w < W; ++w) sh.pub[p][jb + w] = row[w];
          } else if (hasB && (unsigned)growB == cidx) {
#pragma unroll
            for (int w = 0; w < W; ++w) sh.pub[p][jb + w] = SB[w * NT + tid];
          }
        };
        int p;
        Dec d = pick(k, val, first, publish, p);
        if (d.amb) d = pick_exact(k, val, d.M, first, publish, p);
        if (!(d.M > 0.0) || !isfinite(d.M)) { ok = false; break; }
        take_row(k, d, p, q, [&](int j, double xv) { sh.pm[j] = j > t ? xv : 0.0; });
        const long long piv = d.idx;
        if (threadIdx.x == 0) S[t] = piv;
        if (hasA && growA == piv) myA = t;
        if (hasB && growB == piv) myB = t;
        if (hasA && myA < 0) {
          const double f = xA / sh.prow[t];
#pragma unroll
          for (int w = 0; w < W; ++w) row[w] = rsub_mul(row[w], f, sh.pm[jb + w]);
        }
        if (hasB && myB < 0) {
          const double f = xB / sh.prow[t];
#pragma unroll
          for (int w = 0; w < W; ++w) SB[w * NT + tid] = rsub_mul(SB[w * NT + tid], f, sh.pm[jb + w]);
        }
        __syncwarp();   // slot B columns are read across the row group (one warp) in the next step
      }
      __syncthreads();
      CC_T1(1);
      if (!ok) { status = LRA_ESINGULAR; break; }
      lu += q;
    } else {
      for (int s2 = 0; s2 < q; ++s2) {
        if (hasA && S[s2] == growA) myA = s2;
        if (hasB && S[s2] == growB) myB = s2;
      }
    }
    if (fresh) {
      // ---- G = B[S,:] -> G^{-1} in part 0 (read through the block source)
      ib = 0;
      CC_T0();
      ok = gj_src<Q>(k, S, q, bsrc, Xp);
      CC_T1(3);
      if (!ok) { status = LRA_ESINGULAR; break; }
    } else {
      // carried X0 = (G_prev^{-1})^T, one Newton step against the freshly gathered G
      CC_T0();
      const int cur = ib, pa = (ib + 1) % 3, pb = (ib + 2) % 3;
      double *Xc = Xp + cur * Q * Q, *Xa = Xp + pa * Q * Q, *Xb = Xp + pb * Q * Q;
      for (int e = tid; e < q * q; e += NT) {
        const int r = e / q, c = e % q;
        Xa[r * Q + c] = Xc[c * Q + r];
      }
      constexpr int KR = (Q + 15) / 16, MC = (Q + 31) / 32;
#pragma unroll
      for (int aa = 0; aa < KR; ++aa) {
        const int r = k.warp + 16 * aa;
        if (r >= q) continue;
        const long long sr = S[r];
#pragma unroll
        for (int c = 0; c < MC; ++c) {
          const int col = k.lane + 32 * c;
          if (col < q) Xb[r * Q + col] = bsrc(sr, col);
        }
      }
      __syncthreads();
      mm_part<Q>(k, q, Xc, Xb, Xa, nullptr, -1.0);      // R  = I - G X0   -> cur
      mm_part<Q>(k, q, Xb, Xa, Xc, Xa, 1.0);            // X1 = X0 + X0 R  -> pb
      ib = pb;
      CC_T1(2);
    }
    // ---- C = B G^{-1} for the rows outside S (both slots; B rows read from global / L2)
    double rmxA = 0.0, rmxB = 0.0;
    {
      CC_T0();
      const double *X = Xp + ib * Q * Q;
      const bool doA = hasA && myA < 0, doB = hasB && myB < 0;
      // Each thread loads the W entries B[row][jb..jb+W) of its half-row (all loads in flight
      // together) into its own columns of SB; the row group then reads the whole row from SB
      // (entry t lives with the thread of sub t / W).  Slot A first (accumulated in row[]), then
      // slot B (accumulated in accB[], written back after the row group has read its B row).
      auto load_half = [&](long long grow, bool live) {
        double v[W];
#pragma unroll
        for (int w = 0; w < W; ++w) v[w] = (live && jb + w < q) ? bsrc(grow, jb + w) : 0.0;
#pragma unroll
        for (int w = 0; w < W; ++w) SB[w * NT + tid] = v[w];
        __syncwarp();
      };
      auto product = [&](double (&acc)[W]) {
#if CC_PAIR_PRODUCT
        if constexpr (W >= 4 && W % 4 == 0) {
          // Row pairs (ri, ri ^ 1): each thread computes BOTH rows of the pair over half of its
          // W columns, so every X value read from shared memory feeds two FMAs (the product was
          // shared-memory bound: one 8-byte X read per DFMA), then swaps the other row's half
          // with the pair partner (lane ^ TPR).  Every output is the same FMA chain over t
          // ascending as before (bit-identical).
          constexpr int H = W / 2;
          const int h = (k.lane / TPR) & 1;
          const int rp = ri ^ 1;
          double a0[H], a1[H];
#pragma unroll
          for (int w = 0; w < H; ++w) a0[w] = a1[w] = 0.0;
          for (int t = 0; t < q; ++t) {
            const int st = t / W, wt = t - st * W;
            const double b0 = SB[wt * NT + ri * TPR + st];
            const double b1 = SB[wt * NT + rp * TPR + st];
            const double2 *xr = reinterpret_cast<const double2 *>(X + t * Q + jb + h * H);
#pragma unroll
            for (int w = 0; w < H / 2; ++w) {
              const double2 xv = xr[w];
              a0[2 * w] = fma(b0, xv.x, a0[2 * w]);
              a0[2 * w + 1] = fma(b0, xv.y, a0[2 * w + 1]);
              a1[2 * w] = fma(b1, xv.x, a1[2 * w]);
              a1[2 * w + 1] = fma(b1, xv.y, a1[2 * w + 1]);
            }
          }
#pragma unroll
          for (int w = 0; w < H; ++w) {
            const double o = __shfl_xor_sync(0xffffffffu, a1[w], TPR);   // row ri, the other half
            acc[w] = h == 0 ? a0[w] : o;
            acc[H + w] = h == 0 ? o : a0[w];
          }
          return;
        }
#endif
#pragma unroll
        for (int w = 0; w < W; ++w) acc[w] = 0.0;
        for (int t = 0; t < q; ++t) {
          const int st = t / W, wt = t - st * W;
          const double bt = SB[wt * NT + ri * TPR + st];
          if (W >= 2) {
            const double2 *xr = reinterpret_cast<const double2 *>(X + t * Q + jb);
#pragma unroll
            for (int w = 0; w < W / 2; ++w) {
              const double2 xv = xr[w];
              acc[2 * w] = fma(bt, xv.x, acc[2 * w]);
              acc[2 * w + 1] = fma(bt, xv.y, acc[2 * w + 1]);
            }
          } else {
            acc[0] = fma(bt, X[t * Q + jb], acc[0]);
          }
        }
      };
      load_half(growA, doA);
      product(row);
      __syncwarp();
      double accB[W];
      load_half(growB, doB);
      product(accB);
      __syncwarp();
      if (!doA) {
#pragma unroll
        for (int w = 0; w < W; ++w) row[w] = 0.0;
      }
#pragma unroll
      for (int w = 0; w < W; ++w) {
        const double v = doB ? accB[w] : 0.0;
        SB[w * NT + tid] = v;
        rmxA = fmax(rmxA, fabs(row[w]));
        rmxB = fmax(rmxB, fabs(v));
      }
      CC_T1(4);
    }
    __syncthreads();
    // ---- Alg D.1 swap loop over the rows of both slots
    {
      CC_T0();
      double *Xi = Xp + ib * Q * Q;
      for (;;) {
        const double cA = (hasA && myA < 0) ? rmxA : -1.0;
        const double cB = (hasB && myB < 0) ? rmxB : -1.0;
        const double mloc = fmax(cA, cB);
        auto first = [&](double thr) -> unsigned {
          unsigned res = 0xffffffffu;
          if (cB >= thr) {
#pragma unroll
            for (int w = W - 1; w >= 0; --w)
              if (jb + w < q && fabs(SB[w * NT + tid]) >= thr) res = (unsigned)(growB * q + jb + w);
          }
          if (cA >= thr) {
#pragma unroll
            for (int w = W - 1; w >= 0; --w)
              if (jb + w < q && fabs(row[w]) >= thr) res = (unsigned)(growA * q + jb + w);
          }
          return res;
        };
        auto publish = [&](int p, unsigned cidx) {
          if (cidx == 0xffffffffu) return;
          const unsigned rr = cidx / (unsigned)q;
          if (hasA && (unsigned)growA == rr) {
#pragma unroll
            for (int w = 0; w < W; ++w) sh.pub[p][jb + w] = row[w];
          } else if (hasB && (unsigned)growB == rr) {
#pragma unroll
            for (int w = 0; w < W; ++w) sh.pub[p][jb + w] = SB[w * NT + tid];
          }
        };
        int p;
        Dec d = pick(k, mloc, first, publish, p);
        if (!(d.M == d.M)) { ok = false; break; }
        if (d.M <= 1.0 + tol || nsw >= a.cap) {
          cert = fmax(d.M, 0.0);
          cap_hit = d.M > 1.0 + tol;
          break;
        }
        if (d.amb) d = pick_exact(k, mloc, d.M, first, publish, p);
        const long long istar = d.idx / (unsigned)q;
        const int jstar = (int)(d.idx % (unsigned)q);
        take_row(k, d, p, q, [&](int j, double xv) {
          sh.pm[j] = (j == jstar) ? xv - 1.0 : xv;
          if (j == jstar) sh.rc = 1.0 / xv;
        });
        if (threadIdx.x == 0) S[jstar] = istar;
        if (hasA && myA == jstar) {                    // leaves S: explicit row e_{j*}
          myA = -1;
#pragma unroll
          for (int w = 0; w < W; ++w) row[w] = (jb + w == jstar) ? 1.0 : 0.0;
        }
        if (hasB && myB == jstar) {
          myB = -1;
#pragma unroll
          for (int w = 0; w < W; ++w) SB[w * NT + tid] = (jb + w == jstar) ? 1.0 : 0.0;
        }
        if (hasA && growA == istar) myA = jstar;        // enters S
        if (hasB && growB == istar) myB = jstar;
        __syncwarp();
        const int sj = jstar / W, wj = jstar - sj * W;
        double xjA = rsel<W>(row, wj);
        if (TPR > 1) xjA = __shfl_sync(0xffffffffu, xjA, (k.lane & ~(TPR - 1)) | sj);
        const double xjB = SB[wj * NT + ri * TPR + sj];
        const double rc = sh.rc;
        __syncwarp();
        rmxA = 0.0;
        rmxB = 0.0;
        if (hasA && myA < 0) {            // C <- C - C[:,j*] (C[i*,:] - e_j*) / c
          const double g = xjA * rc;
#pragma unroll
          for (int w = 0; w < W; ++w) {
            row[w] = fma(-g, sh.pm[jb + w], row[w]);
            rmxA = fmax(rmxA, fabs(row[w]));
          }
        }
        if (hasB && myB < 0) {
          const double g = xjB * rc;
#pragma unroll
          for (int w = 0; w < W; ++w) {
            const double v = fma(-g, sh.pm[jb + w], SB[w * NT + tid]);
            SB[w * NT + tid] = v;
            rmxB = fmax(rmxB, fabs(v));
          }
        }
        if (carry) {
          constexpr int KR = (Q + 15) / 16, MC = (Q + 31) / 32;
#pragma unroll
          for (int aa = 0; aa < KR; ++aa) {
            const int r = k.warp + 16 * aa;
            if (r >= q) continue;
            double *ir = Xi + r * Q;
            const double gg = ir[jstar] * rc;
            __syncwarp();
#pragma unroll
            for (int c = 0; c < MC; ++c) {
              const int col = k.lane + 32 * c;
              if (col < q) ir[col] = fma(-gg, sh.pm[col], ir[col]);
            }
          }
        }
        ++nsw;
      }
      if (threadIdx.x == 0 && k.rank == 0) atomicAdd(&g_cc_cyc[7], (unsigned long long)(nsw + (cold ? q : 0)));
      CC_T1(5);
    }
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
      if (step > 2 && sw_h == 0 && nsw == 0) break;           // fixed point (reading C13)
    }
  }
  __syncthreads();
  if (threadIdx.x == 0 && k.rank == 0) atomicAdd(&g_cc_cyc[6], (unsigned long long)(clock64() - _tk));
  if (k.rank == 0) {
    if (threadIdx.x < q) {
      a.I[b * q + threadIdx.x] = sh.S[0][threadIdx.x];
      a.J[b * q + threadIdx.x] = sh.S[1][threadIdx.x];
    }
    if (threadIdx.x == 0) {
      a.status[b] = status;
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
        s.min_pivot_margin = __longlong_as_double(0x7ff8000000000000LL);
        a.stats[b] = s;
      }
    }
  }
  if (k.cs > 1) cluster_sync_all();   // keep every CTA's shared memory alive until done
}

}  // namespace ccl

static size_t cc_smem(int rpc, int Q) {
  const int QP = Q | 1;
  return ((((size_t)rpc * QP + 1) & ~(size_t)1) + (size_t)3 * Q * Q) * 8;
}

template <int Q, int TPR>
static cudaError_t launch_cc_t(CAArgs a, int64_t nb, int64_t maxN, cudaStream_t st, int *cs_out, Prof *pf) {
  constexpr int RPC = ccl::NT / TPR;
  int cs = 1;
  while ((int64_t)cs * RPC < maxN) cs *= 2;
  if (cs > 16) return cudaErrorInvalidConfiguration;
  const int rpc = (int)((maxN + cs - 1) / cs);
  const size_t smem = cc_smem(rpc, Q);
  if (smem + sizeof(ccl::Sh<Q>) > 227 * 1024) return cudaErrorInvalidConfiguration;
  a.cs = cs;
  a.rpc = rpc;
  a.grid = 0;
  if (cs_out) *cs_out = cs;
  const bool qeq = a.q == Q;
  void (*kern)(CAArgs) = a.op.kind == LRA_OP_FACTORED_CSR ? (qeq ? ccl::k_cacl<Q, TPR, 2, true> : ccl::k_cacl<Q, TPR, 2>)
                         : (a.op.dtype == LRA_F64 ? (qeq ? ccl::k_cacl<Q, TPR, 1, true> : ccl::k_cacl<Q, TPR, 1>)
                                                  : (qeq ? ccl::k_cacl<Q, TPR, 0, true> : ccl::k_cacl<Q, TPR, 0>));
  cudaError_t e = cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
  if (e != cudaSuccess) return e;
  if (cs > 8) {
    e = cudaFuncSetAttribute(kern, cudaFuncAttributeNonPortableClusterSizeAllowed, 1);
    if (e != cudaSuccess) return e;
  }
  cudaLaunchConfig_t cfg = {};
  cfg.gridDim = dim3((unsigned)(nb * cs));
  cfg.blockDim = dim3(ccl::NT);
  cfg.dynamicSmemBytes = smem;
  cfg.stream = st;
  cudaLaunchAttribute attr[1];
  attr[0].id = cudaLaunchAttributeClusterDimension;
  attr[0].val.clusterDim.x = cs;
  attr[0].val.clusterDim.y = 1;
  attr[0].val.clusterDim.z = 1;
  cfg.attrs = attr;
  static const bool cl1 = getenv("LRA_CA_CLUSTER1") != nullptr;   // diagnostics: cluster attribute for cs = 1
  cfg.numAttrs = (cs > 1 || cl1) ? 1 : 0;
  pf->begin("k_ca", st);
  e = cudaLaunchKernelEx(&cfg, kern, a);
  pf->end(st);
  return e;
}

static size_t cc2_smem(int Q, int W) { return ((size_t)W * ccl::NT + (size_t)3 * Q * Q) * 8; }

// two-slot kernel: 2 NT / TPR rows per CTA
template <int Q, int TPR>
static cudaError_t launch_cc2_t(CAArgs a, int64_t nb, int64_t maxN, cudaStream_t st, int *cs_out, Prof *pf) {
  constexpr int RPC2 = 2 * ccl::NT / TPR, W = Q / TPR;
  int cs = 1;
  while ((int64_t)cs * RPC2 < maxN) cs *= 2;
  if (cs > 16) return cudaErrorInvalidConfiguration;
  const size_t smem = cc2_smem(Q, W);
  if (smem + sizeof(ccl::Sh<Q>) > 227 * 1024) return cudaErrorInvalidConfiguration;
  a.cs = cs;
  a.rpc = RPC2;
  a.grid = 0;
  if (cs_out) *cs_out = cs;
  const bool qeq = a.q == Q;
  void (*kern)(CAArgs) = a.op.kind == LRA_OP_FACTORED_CSR ? (qeq ? ccl::k_cacl2<Q, TPR, 2, true> : ccl::k_cacl2<Q, TPR, 2>)
                         : (a.op.dtype == LRA_F64 ? (qeq ? ccl::k_cacl2<Q, TPR, 1, true> : ccl::k_cacl2<Q, TPR, 1>)
                                                  : (qeq ? ccl::k_cacl2<Q, TPR, 0, true> : ccl::k_cacl2<Q, TPR, 0>));
  cudaError_t e = cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
  if (e != cudaSuccess) return e;
  if (cs > 8) {
    e = cudaFuncSetAttribute(kern, cudaFuncAttributeNonPortableClusterSizeAllowed, 1);
    if (e != cudaSuccess) return e;
  }
  cudaLaunchConfig_t cfg = {};
  cfg.gridDim = dim3((unsigned)(nb * cs));
  cfg.blockDim = dim3(ccl::NT);
  cfg.dynamicSmemBytes = smem;
  cfg.stream = st;
  cudaLaunchAttribute attr[1];
  attr[0].id = cudaLaunchAttributeClusterDimension;
  attr[0].val.clusterDim.x = cs;
  attr[0].val.clusterDim.y = 1;
  attr[0].val.clusterDim.z = 1;
  cfg.attrs = attr;
  cfg.numAttrs = cs > 1 ? 1 : 0;
  pf->begin("k_ca", st);
  e = cudaLaunchKernelEx(&cfg, kern, a);
  pf->end(st);
  return e;
}

template <int Q, int TPR>
static int cc2_active_t(int64_t maxN) {
  constexpr int RPC2 = 2 * ccl::NT / TPR, W = Q / TPR;
  int cs = 1;
  while ((int64_t)cs * RPC2 < maxN) cs *= 2;
  if (cs > 16) return 0;
  const size_t smem = cc2_smem(Q, W);
  void (*kern)(CAArgs) = ccl::k_cacl2<Q, TPR, 0>;
  if (cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem) != cudaSuccess) return 0;
  if (cs > 8 && cudaFuncSetAttribute(kern, cudaFuncAttributeNonPortableClusterSizeAllowed, 1) != cudaSuccess) return 0;
  cudaLaunchConfig_t cfg = {};
  cfg.gridDim = dim3((unsigned)(cs * 64));
  cfg.blockDim = dim3(ccl::NT);
  cfg.dynamicSmemBytes = smem;
  cudaLaunchAttribute attr[1];
  attr[0].id = cudaLaunchAttributeClusterDimension;
  attr[0].val.clusterDim.x = cs;
  attr[0].val.clusterDim.y = 1;
  attr[0].val.clusterDim.z = 1;
  cfg.attrs = attr;
  cfg.numAttrs = 1;
  int n = 0;
  if (cudaOccupancyMaxActiveClusters(&n, kern, &cfg) != cudaSuccess) {
    cudaGetLastError();
    return 0;
  }
  return n;
}

// The two-slot kernel is used whenever the one-slot kernel would need a cluster of 2 or more.
static bool use_two_slot(int64_t maxN, int q) {
  static const int env = getenv("LRA_CA_SLOTS") ? atoi(getenv("LRA_CA_SLOTS")) : 2;   // diagnostics (A/B)
  if (env == 1) return false;
  const int rpc1 = q <= 24 ? ccl::NT : ccl::NT / 2;
  return maxN > rpc1;
}

template <int Q, int TPR>
static int cc_active_t(int64_t maxN) {
  constexpr int RPC = ccl::NT / TPR;
  int cs = 1;
  while ((int64_t)cs * RPC < maxN) cs *= 2;
  if (cs > 16) return 0;
  const int rpc = (int)((maxN + cs - 1) / cs);
  const size_t smem = cc_smem(rpc, Q);
  void (*kern)(CAArgs) = ccl::k_cacl<Q, TPR, 0>;
  if (cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem) != cudaSuccess) return 0;
  if (cs > 8 && cudaFuncSetAttribute(kern, cudaFuncAttributeNonPortableClusterSizeAllowed, 1) != cudaSuccess) return 0;
  cudaLaunchConfig_t cfg = {};
  cfg.gridDim = dim3((unsigned)(cs * 64));
  cfg.blockDim = dim3(ccl::NT);
  cfg.dynamicSmemBytes = smem;
  cudaLaunchAttribute attr[1];
  attr[0].id = cudaLaunchAttributeClusterDimension;
  attr[0].val.clusterDim.x = cs;
  attr[0].val.clusterDim.y = 1;
  attr[0].val.clusterDim.z = 1;
  cfg.attrs = attr;
  cfg.numAttrs = 1;
  int n = 0;
  if (cudaOccupancyMaxActiveClusters(&n, kern, &cfg) != cudaSuccess) {
    cudaGetLastError();
    return 0;
  }
  return n;
}

// Problems of this shape the cluster tier runs concurrently (co-resident clusters; 0 if the
// tier does not apply).  B200, config 2 (16-CTA clusters): 7.
int ca_cluster_max_active(int64_t maxN, int q) {
  if (use_two_slot(maxN, q)) {
    if (q <= 8) return cc2_active_t<8, 1>(maxN);
    if (q <= 16) return cc2_active_t<16, 1>(maxN);
    if (q <= 24) return cc2_active_t<24, 1>(maxN);
    if (q <= 32) return cc2_active_t<32, 2>(maxN);
    if (q <= 48) return cc2_active_t<48, 2>(maxN);
    return 0;
  }
  if (q <= 8) return cc_active_t<8, 1>(maxN);
  if (q <= 16) return cc_active_t<16, 1>(maxN);
  if (q == 20) return cc_active_t<20, 1>(maxN);    // config 3 (k = l = 20): q as a compile-time constant
  if (q <= 24) return cc_active_t<24, 1>(maxN);
  if (q <= 32) return cc_active_t<32, 2>(maxN);
  if (q <= 48) return cc_active_t<48, 2>(maxN);
  return 0;
}

// Cluster tier of the real C-A (q <= 48, at most 16 CTAs of NT / TPR rows): returns
// cudaErrorInvalidConfiguration when the problem does not fit (caller falls back).
cudaError_t launch_ca_cluster(CAArgs a, int64_t nb, int64_t maxN, cudaStream_t st, int *cs_out, Prof *pf) {
  if (use_two_slot(maxN, a.q)) {
    if (a.q <= 8) return launch_cc2_t<8, 1>(a, nb, maxN, st, cs_out, pf);
    if (a.q <= 16) return launch_cc2_t<16, 1>(a, nb, maxN, st, cs_out, pf);
    if (a.q <= 24) return launch_cc2_t<24, 1>(a, nb, maxN, st, cs_out, pf);
    if (a.q <= 32) return launch_cc2_t<32, 2>(a, nb, maxN, st, cs_out, pf);
    if (a.q <= 48) return launch_cc2_t<48, 2>(a, nb, maxN, st, cs_out, pf);
    return cudaErrorInvalidConfiguration;
  }
  if (a.q <= 8) return launch_cc_t<8, 1>(a, nb, maxN, st, cs_out, pf);
  if (a.q <= 16) return launch_cc_t<16, 1>(a, nb, maxN, st, cs_out, pf);
  if (a.q == 20) return launch_cc_t<20, 1>(a, nb, maxN, st, cs_out, pf);
  if (a.q <= 24) return launch_cc_t<24, 1>(a, nb, maxN, st, cs_out, pf);
  if (a.q <= 32) return launch_cc_t<32, 2>(a, nb, maxN, st, cs_out, pf);
  if (a.q <= 48) return launch_cc_t<48, 2>(a, nb, maxN, st, cs_out, pf);
  return cudaErrorInvalidConfiguration;
}

cudaError_t read_idx_err_cc(long long *out, bool reset) {
  cudaError_t e = cudaMemcpyFromSymbol(out, g_idx_err, sizeof(g_idx_err));
  if (e == cudaSuccess && reset) {
    long long z[4] = {0, 0, 0, 0};
    e = cudaMemcpyToSymbol(g_idx_err, z, sizeof(z));
  }
  return e;
}

cudaError_t read_cc_counters(unsigned long long *out, bool reset) {
  cudaError_t e = cudaMemcpyFromSymbol(out, g_cc_cyc, sizeof(g_cc_cyc));
  if (e == cudaSuccess && reset) {
    unsigned long long z[16] = {0};
    e = cudaMemcpyToSymbol(g_cc_cyc, z, sizeof(z));
  }
  return e;
}

}  // namespace lra
