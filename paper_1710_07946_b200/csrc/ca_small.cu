// ca_small.cu — the C-A iterations (Alg 10.2 stages 2-3 with Remark rerfnhmt, P:4048-4057;
// maxvol = Alg D.2 stage 1 + Alg D.1) for SMALL blocks: one 128-thread CTA per
// problem, several problems per SM (config 3: 512 x 20 blocks; config 1: 256 x 8).
//
// The cluster tier spends a 512-thread CTA (one per SM) on a 512-row block, and every phase
// of it is synchronisation latency (tools/ca_phases_cfg3.py: 252 us per config-3 block).  Here
// a thread owns RPT rows (r = tid + 128 u) with all their q values in registers, so a pivot
// decision is two 4-warp reductions, and two or three problems share an SM.
//
// Arithmetic (the oracle's decisions, readings C10-C12):
//   * cold start (Alg D.2 stage 1): LUP with the slack rule — column t's candidates |B'[i,t]|
//     over unchosen rows (NaN counts as +inf), M = max, pivot = the smallest row index with
//     |B'[i,t]| >= (1 - tau) M; every unchosen row: f = B'[i,t] / B'[p,t] (IEEE divide) and
//     B'[i,j] = B'[i,j] - f B'[p,j] for j > t (one multiply, one subtract, no FMA), as the
//     oracle's lup_pivots;
//   * C = B G^{-1} for the rows outside S, G = B[S,:] inverted by Gauss-Jordan with partial
//     pivoting (smallest row on ties), each C entry an FMA chain over t ascending;
//   * Alg D.1 swaps: M = max |C'| over the rows outside S; stop when M <= 1 + tol or at the
//     swap cap; else (i*, j*) = the smallest row-major index i q + j with |C| >= (1 - tau) M,
//     S[j*] = i*, C <- C - C[:, j*] (C[i*,:] - e_j*) / C[i*, j*] (the leaving row restarts as
//     e_j*, the entering row leaves the candidate set).
// Every decision is an exact two-pass reduction (the max, then the first qualifying index over
// the values as computed), so no ambiguity round is needed.
#include "kernels.cuh"

namespace lra {
namespace cas {

constexpr int NT = 128;          // threads per problem
constexpr int NW = NT / 32;

template <int OPK>
__device__ __forceinline__ double opv(const OpView &op, int64_t i, int64_t j) {
  if (OPK == 0) return (double)__ldg((const float *)op.w + j * op.ldw + i);
  if (OPK == 1) return __ldg((const double *)op.w + j * op.ldw + i);
  return op.f.at(i, j);
}

__device__ __forceinline__ unsigned long long dkey(double v) {   // order-preserving key of v >= 0
  return v > 0.0 ? (unsigned long long)__double_as_longlong(v) : 0ull;
}

template <int Q>
struct Sh {
  long long S[2][Q];                 // [0]: I slots, [1]: J slots
  unsigned long long wk[2][NW];      // per-warp max keys (double-buffered by decision parity)
  unsigned wi[2][NW];                // per-warp first indices
  double cand[2][NW][Q];             // each warp's candidate row (the winner's is read back)
  double X[Q * Q];                   // G^{-1} (row-major, stride Q)
  double G[Q * Q];                   // G = B[S,:]; Gauss-Jordan pivot rows
  double gd;
};

// One decision: the CTA max of the threads' keys, then the smallest of the threads' first
// indices at the threshold (1 - tau) M.  The thread holding a warp's first index publishes its
// candidate row into cand[p][warp] before the second barrier; *wwin = the winning warp.
template <int Q, class FirstF, class PubF>
__device__ __forceinline__ int decide(Sh<Q> &sh, int &par, unsigned long long key, double tau, FirstF firstv,
                                      PubF pub, double &M, unsigned &idx, int &wwin) {
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const int p = par;
  par ^= 1;
  const unsigned hi = (unsigned)(key >> 32);
  const unsigned mhi = __reduce_max_sync(0xffffffffu, hi);
  const unsigned mlo = __reduce_max_sync(0xffffffffu, hi == mhi ? (unsigned)key : 0u);
  if (lane == 0) sh.wk[p][warp] = ((unsigned long long)mhi << 32) | mlo;
  __syncthreads();
  unsigned long long g = 0ull;
#pragma unroll
  for (int w = 0; w < NW; ++w) g = sh.wk[p][w] > g ? sh.wk[p][w] : g;
  M = __longlong_as_double((long long)g);
  const double thr = (1.0 - tau) * M;
  const unsigned mine = g ? firstv(thr) : 0xffffffffu;
  const unsigned wmin = __reduce_min_sync(0xffffffffu, mine);
  if (wmin != 0xffffffffu && mine == wmin) pub(p, warp, mine);
  if (lane == 0) sh.wi[p][warp] = wmin;
  __syncthreads();
  idx = 0xffffffffu;
  wwin = 0;
#pragma unroll
  for (int w = 0; w < NW; ++w)
    if (sh.wi[p][w] < idx) {
      idx = sh.wi[p][w];
      wwin = w;
    }
  return p;
}

// Gauss-Jordan inverse of the q x q matrix sh.G (row-major, stride Q) into sh.X with partial
// pivoting (largest |.| among the unused rows, smallest row on ties, NaN largest); false if
// singular.  Thread (warp w, lane l) keeps column l of the rows w + 4k of [G | I].
template <int Q>
__device__ __forceinline__ bool gauss_jordan(Sh<Q> &sh, int q) {
  constexpr int KR = (Q + NW - 1) / NW;
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  double ga[KR], gx[KR];
#pragma unroll
  for (int k = 0; k < KR; ++k) {
    const int r = warp + NW * k;
    ga[k] = (r < q && lane < q) ? sh.G[r * Q + lane] : 0.0;
    gx[k] = (r < q && lane == r) ? 1.0 : 0.0;
  }
  unsigned used = 0;
  int pstep[KR];                                 // the step at which each owned row was the pivot
#pragma unroll
  for (int k = 0; k < KR; ++k) pstep[k] = 0;
  for (int s = 0; s < q; ++s) {
    unsigned long long bk = 0ull;
    int br = 0x7fffffff;
#pragma unroll
    for (int k = 0; k < KR; ++k) {
      const int r = warp + NW * k;
      const double v = __shfl_sync(0xffffffffu, ga[k], s);
      if (r < q && !((used >> k) & 1u)) {
        const double av = fabs(v);
        const unsigned long long kk = (av != av) ? 0x7ff8000000000000ull : dkey(av);
        if (br == 0x7fffffff || kk > bk) {
          bk = kk;
          br = r;
        }
      }
    }
    if (lane == 0) {
      sh.wk[0][warp] = bk;
      sh.wi[0][warp] = (unsigned)br;
    }
    __syncthreads();
    unsigned long long gk = 0ull;
    int pr = 0x7fffffff;
#pragma unroll
    for (int w = 0; w < NW; ++w) {
      const int r = (int)sh.wi[0][w];
      if (r == 0x7fffffff) continue;
      if (pr == 0x7fffffff || sh.wk[0][w] > gk || (sh.wk[0][w] == gk && r < pr)) {
        gk = sh.wk[0][w];
        pr = r;
      }
    }
    if (pr >= q) return false;
    if (warp == pr % NW) {                       // the pivot row, scaled, into shared memory
      const int kp = pr / NW;
      double pa = ga[0], px = gx[0];
#pragma unroll
      for (int k = 1; k < KR; ++k)
        if (k == kp) {
          pa = ga[k];
          px = gx[k];
        }
      const double d = __shfl_sync(0xffffffffu, pa, s);
      const double rd = 1.0 / d;
      if (lane < Q) {
        sh.G[pr * Q + lane] = pa * rd;
        sh.X[pr * Q + lane] = px * rd;
      }
      if (lane == 0) sh.gd = d;
    }
    __syncthreads();
    const double d = sh.gd;
    if (!(fabs(d) > 0.0) || !isfinite(d)) return false;
    const double pa = lane < Q ? sh.G[pr * Q + lane] : 0.0, px = lane < Q ? sh.X[pr * Q + lane] : 0.0;
#pragma unroll
    for (int k = 0; k < KR; ++k) {
      const int r = warp + NW * k;
      const double f = __shfl_sync(0xffffffffu, ga[k], s);
      if (r == pr) {
        used |= 1u << k;
        pstep[k] = s;
        ga[k] = pa;
        gx[k] = px;
      } else if (r < q) {
        ga[k] = fma(-f, pa, ga[k]);
        gx[k] = fma(-f, px, gx[k]);
      }
    }
    __syncthreads();                             // sh.G / sh.X pivot rows are rewritten next step
  }
  // [G | I] -> [P | P G^{-1}] with P[pivot of step s] = e_s: row s of G^{-1} is the right part
  // of the row that was the pivot of step s
#pragma unroll
  for (int k = 0; k < KR; ++k) {
    const int r = warp + NW * k;
    if (r < q && lane < Q) sh.X[pstep[k] * Q + lane] = lane < q ? gx[k] : 0.0;
  }
  __syncthreads();
  return true;
}

template <int Q>
__device__ __forceinline__ double selj(const double (&r)[Q], int j) {   // r[j], j warp-uniform
  double v = 0.0;
#pragma unroll
  for (int jj = 0; jj < Q; ++jj)
    if (jj == j) v = r[jj];
  return v;
}

// Steps: 0 = stage 2 on a real sketch Y (cold); then 2L+1 = horizontal step of loop L
// (J <- maxvol(W[I,:]^T), cold in loop 0), 2L+2 = vertical step (I <- maxvol(W[:,J]), warm).
template <int Q, int RPT, int OPK>
__global__ void __launch_bounds__(NT, 2) k_cas(CAArgs a) {
  if (a.skip && (a.skip[0] != 0 || a.skip[1] != 0)) return;   // row-sharded chain: step not needed
  __shared__ Sh<Q> sh;
  const int tid = threadIdx.x;
  const int64_t b = blockIdx.x;
  const int q = a.q;
  const double tau = a.tau, tol = a.tol;
  OpView op = a.op;
  if (op.kind == LRA_OP_DENSE) op.w = (const char *)op.w + b * a.w_stride * (op.dtype == LRA_F32 ? 4 : 8);
  int par = 0;
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
  __syncthreads();
  const double *Y = yreal ? reinterpret_cast<const double *>(a.Y) + b * a.y_stride : nullptr;
  const int last = 2 * a.sweeps;
  double row[RPT][Q];
  int slot[RPT];                      // slot of the row in S, -1 outside
  for (int step = yreal ? 0 : 1; status == LRA_OK && step <= last; ++step) {
    const int kind = step == 0 ? 0 : ((step & 1) ? 1 : 2);   // 0 = Y, 1 = h, 2 = v
    const int64_t N = kind == 1 ? op.n : op.m;
    long long *S = kind == 1 ? sh.S[1] : sh.S[0];
    const bool cold = step <= 1 && !(step == 0 && a.y_warm);
    const long long *Ig = sh.S[0], *Jg = sh.S[1];
    auto bval = [&](int64_t r, int j) -> double {            // entry (r, j) of this step's N x q block
      if (kind == 0) return __ldg(Y + (int64_t)j * a.ldy + r);
      if (kind == 1) return opv<OPK>(op, Ig[j], r);
      return opv<OPK>(op, r, Jg[j]);
    };
    auto load_rows = [&]() {
#pragma unroll
      for (int u = 0; u < RPT; ++u) {
        const int64_t r = tid + NT * u;
#pragma unroll
        for (int j = 0; j < Q; ++j) row[u][j] = (r < N && j < q) ? bval(r, j) : 0.0;
      }
    };
    __syncthreads();                  // S of the previous step is final everywhere
    load_rows();
#pragma unroll
    for (int u = 0; u < RPT; ++u) slot[u] = -1;
    int nsw = 0;
    bool ok = true;
    double cert = 0.0;
    bool cap_hit = false;
    if (cold) {
      // ---- Alg D.2 stage 1: LUP with the slack pivot rule (the oracle's arithmetic)
      for (int t = 0; t < q && ok; ++t) {
        double val[RPT];
        unsigned long long key = 0ull;
#pragma unroll
        for (int u = 0; u < RPT; ++u) {
          const int64_t r = tid + NT * u;
          const double x = selj<Q>(row[u], t);
          val[u] = (r < N && slot[u] < 0) ? ((x != x) ? INFINITY : fabs(x)) : -1.0;
          if (val[u] >= 0.0) {
            const unsigned long long kk = val[u] == INFINITY ? 0x7ff0000000000000ull : dkey(val[u]);
            key = kk > key ? kk : key;
          }
        }
        double M;
        unsigned idx;
        int ww;
        const int p = decide(
            sh, par, key, tau,
            [&](double thr) -> unsigned {
              unsigned res = 0xffffffffu;
#pragma unroll
              for (int u = RPT - 1; u >= 0; --u)
                if (val[u] >= 0.0 && val[u] >= thr) res = (unsigned)(tid + NT * u);
              return res;
            },
            [&](int pp, int w, unsigned mine) {
              const int u = (int)(mine / NT);
#pragma unroll
              for (int uu = 0; uu < RPT; ++uu)
                if (uu == u)
#pragma unroll
                  for (int j = 0; j < Q; ++j) sh.cand[pp][w][j] = row[uu][j];
            },
            M, idx, ww);
        if (!(M > 0.0) || !isfinite(M) || idx == 0xffffffffu) { ok = false; break; }
        if (tid == 0) S[t] = (long long)idx;
        const double *prw = sh.cand[p][ww];
        const double pt = prw[t];
#pragma unroll
        for (int u = 0; u < RPT; ++u) {
          const int64_t r = tid + NT * u;
          if ((unsigned)r == idx) slot[u] = t;
          if (r < N && slot[u] < 0) {
            const double f = selj<Q>(row[u], t) / pt;
#pragma unroll
            for (int j = 0; j < Q; ++j)
              if (j > t && j < q) row[u][j] = rsub_mul(row[u][j], f, prw[j]);
          }
        }
      }
      if (!ok) { status = LRA_ESINGULAR; break; }
      lu += q;
      __syncthreads();                // S complete
      load_rows();                    // the original block rows (C = B G^{-1} uses them)
    } else {
#pragma unroll
      for (int u = 0; u < RPT; ++u)
        for (int s2 = 0; s2 < q; ++s2)
          if (S[s2] == (long long)(tid + NT * u)) slot[u] = s2;
    }
    // ---- G = B[S,:] (original rows) -> X = G^{-1}
    for (int e = tid; e < q * q; e += NT) {
      const int r = e / q, c = e % q;
      sh.G[r * Q + c] = bval(S[r], c);
    }
    __syncthreads();
    if (!gauss_jordan<Q>(sh, q)) { status = LRA_ESINGULAR; break; }
    // ---- C = B X for the rows outside S (FMA chain over t ascending)
    double rmx[RPT];
#pragma unroll
    for (int u = 0; u < RPT; ++u) {
      const int64_t r = tid + NT * u;
      double c[Q];
#pragma unroll
      for (int j = 0; j < Q; ++j) c[j] = 0.0;
      if (r < N && slot[u] < 0) {
#pragma unroll
        for (int t = 0; t < Q; ++t) {
          if (t < q) {
            const double bt = row[u][t];
#pragma unroll
            for (int j = 0; j < Q; ++j) c[j] = fma(bt, sh.X[t * Q + j], c[j]);
          }
        }
      }
      rmx[u] = 0.0;
#pragma unroll
      for (int j = 0; j < Q; ++j) {
        row[u][j] = j < q ? c[j] : 0.0;
        rmx[u] = fmax(rmx[u], fabs(row[u][j]));
      }
    }
    // ---- Alg D.1 swap loop
    for (;;) {
      unsigned long long key = 0ull;
#pragma unroll
      for (int u = 0; u < RPT; ++u) {
        const int64_t r = tid + NT * u;
        if (r < N && slot[u] < 0) {
          const unsigned long long kk = dkey(rmx[u]);
          key = kk > key ? kk : key;
        }
      }
      double M;
      unsigned idx;
      int ww;
      const int p = decide(
          sh, par, key, tau,
          [&](double thr) -> unsigned {
            unsigned res = 0xffffffffu;
#pragma unroll
            for (int u = RPT - 1; u >= 0; --u) {
              const int64_t r = tid + NT * u;
              if (r < N && slot[u] < 0 && rmx[u] >= thr) {
#pragma unroll
                for (int j = Q - 1; j >= 0; --j)
                  if (j < q && fabs(row[u][j]) >= thr) res = (unsigned)(r * q + j);
              }
            }
            return res;
          },
          [&](int pp, int w, unsigned mine) {
            const int u = (int)((mine / (unsigned)q) / NT);
#pragma unroll
            for (int uu = 0; uu < RPT; ++uu)
              if (uu == u)
#pragma unroll
                for (int j = 0; j < Q; ++j) sh.cand[pp][w][j] = row[uu][j];
          },
          M, idx, ww);
      if (!(M == M)) { ok = false; break; }
      if (M <= 1.0 + tol || nsw >= a.cap || idx == 0xffffffffu) {
        cert = fmax(M, 0.0);
        cap_hit = M > 1.0 + tol;
        break;
      }
      const unsigned istar = idx / (unsigned)q;
      const int jstar = (int)(idx % (unsigned)q);
      const double *crow = sh.cand[p][ww];          // C[i*, :]
      const double rc = 1.0 / crow[jstar];
      if (tid == 0) S[jstar] = (long long)istar;
#pragma unroll
      for (int u = 0; u < RPT; ++u) {
        const int64_t r = tid + NT * u;
        if (r >= N) continue;
        if (slot[u] == jstar) {                      // leaves S: explicit row e_{j*}
          slot[u] = -1;
#pragma unroll
          for (int j = 0; j < Q; ++j) row[u][j] = j == jstar ? 1.0 : 0.0;
        }
        if ((unsigned)r == istar) slot[u] = jstar;   // enters S
        rmx[u] = 0.0;
        if (slot[u] < 0) {                           // C <- C - C[:,j*] (C[i*,:] - e_j*) / c
          const double g = selj<Q>(row[u], jstar) * rc;
#pragma unroll
          for (int j = 0; j < Q; ++j) {
            if (j < q) {
              const double pm = j == jstar ? crow[j] - 1.0 : crow[j];
              row[u][j] = fma(-g, pm, row[u][j]);
              rmx[u] = fmax(rmx[u], fabs(row[u][j]));
            }
          }
        }
      }
      ++nsw;
    }
    if (!ok) { status = LRA_ESINGULAR; break; }
    swaps += nsw;
    caps += cap_hit;
    if (kind == 0) {
      sk_swaps = nsw;
      cert_r = cert;
    }
    if (kind == 1) {
      cert_c = cert;
      sw_h = nsw;
    }
    if (kind == 2) {
      cert_r = cert;
      ++loops;
      if (step > 2 && sw_h == 0 && nsw == 0) break;           // fixed point (reading C13)
    }
  }
  __syncthreads();
  if (tid < q) {
    a.I[b * q + tid] = sh.S[0][tid];
    a.J[b * q + tid] = sh.S[1][tid];
  }
  if (tid == 0) {
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

template <int Q, int RPT>
static cudaError_t launch_t(const CAArgs &a, int64_t nb, cudaStream_t st, Prof *pf) {
  void (*k)(CAArgs) = a.op.kind == LRA_OP_FACTORED_CSR ? k_cas<Q, RPT, 2>
                                                       : (a.op.dtype == LRA_F64 ? k_cas<Q, RPT, 1> : k_cas<Q, RPT, 0>);
  pf->begin("k_ca_small", st);
  k<<<(unsigned)nb, NT, 0, st>>>(a);
  pf->end(st);
  return cudaGetLastError();
}

}  // namespace cas

// The small tier: q <= 20 with up to 512 rows (RPT x Q doubles of rows per thread in
// registers).  Opt-in (LRA_CA_SMALL=1): measured slower than the cluster tier on config 3
// (905 us vs ~300 us per wave of 148 blocks, 14.3 vs 8.6 ms per 4096-block batch) — with
// 4 warps per problem and 1-2 problems per SM, each scheduler holds 1-2 warps and every
// dependent fp64 / shared-memory latency is exposed.  Pivots are bit-identical
// to the other tiers on every GPU parity test (run with LRA_CA_SMALL=1).
bool ca_small_fits(int64_t maxN, int q, int y_complex, int y_warm) {
  static const bool on = [] { const char *e = getenv("LRA_CA_SMALL"); return e && e[0] == '1'; }();
  if (!on || y_complex || y_warm) return false;
  return q >= 1 && q <= 20 && maxN <= 4 * cas::NT;
}

int ca_small_max_active(int64_t maxN, int q) {
  int n = 0, dev = 0, sms = 148;
  cudaGetDevice(&dev);
  cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev);
  cudaError_t e;
  if (q <= 8) e = cudaOccupancyMaxActiveBlocksPerMultiprocessor(&n, cas::k_cas<8, 4, 0>, cas::NT, 0);
  else e = cudaOccupancyMaxActiveBlocksPerMultiprocessor(&n, cas::k_cas<20, 4, 0>, cas::NT, 0);
  if (e != cudaSuccess) {
    cudaGetLastError();
    n = 1;
  }
  (void)maxN;
  return n * sms;
}

cudaError_t launch_ca_small(CAArgs a, int64_t nb, int64_t maxN, cudaStream_t st, int *cs_out, Prof *pf) {
  if (!ca_small_fits(maxN, a.q, a.y_complex, a.y_warm)) return cudaErrorInvalidConfiguration;
  if (cs_out) *cs_out = 1;
  const int rpt = (int)((maxN + cas::NT - 1) / cas::NT);
  if (a.q <= 8) {
    if (rpt <= 2) return cas::launch_t<8, 2>(a, nb, st, pf);
    return cas::launch_t<8, 4>(a, nb, st, pf);
  }
  if (rpt <= 2) return cas::launch_t<20, 2>(a, nb, st, pf);
  return cas::launch_t<20, 4>(a, nb, st, pf);
}

}  // namespace lra
