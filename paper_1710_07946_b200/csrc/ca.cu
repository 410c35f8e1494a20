// ca.cu — stages 2-3 of Alg 10.2 with C-A iterations (Remark rerfnhmt),
// each C-A step a maxvol on a tall-skinny N x q block: Alg D.2 stage 1 (LUP cold start,
// P:6550-6556) or a warm start from the current slots, then the Alg D.1 swap loop
// with the rank-1 update C <- C - C[:,j*](C[i*,:] - e_j*^T)/c_{i*j*}.
//
// One thread-block CLUSTER per problem, ONE ROW OF THE BLOCK PER THREAD.  The row of the
// C-matrix lives in that thread's registers (compile-time width Q >= q, zero padded), so
// the LU and swap updates never touch shared memory.  Each pivot decision is
//   CTA max  ->  CTA smallest index with |c| >= (1-tau) max  ->  ONE cluster exchange
// of (max, index, value) triples through DSMEM, together with the CTA winner's row, which
// the winning CTA publishes in its shared memory before the cluster barrier; every CTA
// then copies the winning row (ld.shared::cluster).  The smallest-index rule (reading C11)
// is exact: a CTA whose candidate value falls inside the tie window of the global max
// (< 1e-12 relative) triggers a second, exact exchange (deterministic in every CTA).
// C = B * X^{-1} is formed by an in-shared-memory Gauss-Jordan inverse of the q x q X
// (X = B[S,:] for a warm start, X = L_S after the cold LUP, where the rows hold their LU
// multipliers) followed by a register-accumulated product (fp64 FMA bound).  The selected
// rows are implicit identity rows of C = (I_q | C') (reading C12b).  Blocks are gathered
// straight from W (vertical W[:,J]: coalesced columns; horizontal W[I,:]^T: one sector
// per element, 16 loads in flight per thread).  The whole C-A (all sweeps, early exit)
// is one launch.  The complex (ARFT) stage-2 maxvol uses a shared-memory row variant.
#include <cooperative_groups.h>
#include <climits>
#include <cstdlib>

#include "kernels.cuh"

namespace cg = cooperative_groups;

namespace lra {

// Phase timers (clock64 cycles of CTA 0, thread 0 of every problem; read by
// lra_debug_counters): 0 load, 1 cold LU, 2 warm gather, 3 Gauss-Jordan, 4 product,
// 5 swap loop, 6 whole kernel, 7 pivot steps (count).
__device__ unsigned long long g_ca_cyc[16];
#define CA_MARK(k) do { if (threadIdx.x == 0 && c.rank == 0) { long long _n = clock64(); atomicAdd(&g_ca_cyc[k], (unsigned long long)(_n - _tm)); _tm = _n; } } while (0)
#define CA_T0() long long _t0 = clock64()
#define CA_T1(k) do { if (threadIdx.x == 0 && c.rank == 0) atomicAdd(&g_ca_cyc[k], (unsigned long long)(clock64() - _t0)); } while (0)

struct Tri {
  double M;
  long long idx;
  double v;
};

struct CAShared {
  long long Isl[LRA_QMAX], Jsl[LRA_QMAX];
  unsigned long long rk[2][32];
  unsigned ri[2][32];
  double rv[2][32];
  Tri xt[2];
  Tri xin[2][16];              // triples pushed by every CTA of the cluster (slot = rank)
  __align__(16) double pub[2][LRA_QMAX * 2];   // published candidate row (complex: 2x)
  __align__(16) double prow[LRA_QMAX * 2];
  __align__(16) double pm[LRA_QMAX];           // pivot row prepared for the update
  double rc;                                   // 1 / pivot (swap steps)
  double fcol[LRA_QMAX];
  double xd[2];
  long long xi[2];
  double bd;
  long long bi;
  int piv[LRA_QMAX];
  int sing;
  unsigned long long gk[2][32];   // Gauss-Jordan: per-warp pivot candidates
  int gr[2][32];
  __align__(16) double gp[2][128];   // Gauss-Jordan: scaled pivot row
  double gd[2];
  double dM;                   // exchange decision (written by warp 0)
  long long dbest;
  int damb;
};

struct Ctx {
  CAShared *sh;
  void *Cs;                    // rpc x qp (block rows; complex path: the C rows)
  double *X;                   // q x QX (Gauss-Jordan), or packed L_S (complex path)
  double *rmax;                // rpc   (complex path)
  unsigned char *inS;          // rpc   (complex path)
  int rank, cs, rpc, qp, q, QX, R0, AS, tid, lane, warp, nt, nw;
  int par;                     // exchange slot parity (identical in every CTA)
  int ib;                      // column offset of the carried G^{-1} inside aug (0 or Q)
  int rb;                      // CTA reduction buffer parity
  double tau, tol;
  // grid tier (one problem spread over the whole grid, cooperative launch): exchanges go
  // through global memory instead of DSMEM
  int grid;
  Tri *gtri;                   // [2][cs]  CTA triples
  double *grow;                // [2][cs][LRA_QMAX]  CTA candidate rows
  double *gG;                  // [LRA_QMAX][LRA_QMAX]  rows B[S,:] for warm starts
};

__device__ __forceinline__ void cluster_barrier(const Ctx &c) {
  if (c.grid) cg::this_grid().sync();
  else if (c.cs > 1) cg::this_cluster().sync();
  else __syncthreads();
}
// where this CTA publishes its candidate row for exchange parity p
__device__ __forceinline__ double *pub_slot(const Ctx &c, int p) {
  return c.grid ? c.grow + ((size_t)p * c.cs + c.rank) * LRA_QMAX : &c.sh->pub[p][0];
}
template <typename T>
__device__ __forceinline__ T *remote(const Ctx &c, T *p, int rank) {
  if (c.cs == 1) return p;
  return cg::this_cluster().map_shared_rank(p, rank);
}
// grid tier: owners copy the block rows B[S[a],:] of their CTA to gG before the barrier
__device__ __forceinline__ void publish_S_rows(const Ctx &c, const long long *S, int64_t r0, int nloc) {
  if (!c.grid) return;
  for (int a = c.warp; a < c.q; a += c.nw) {
    const long long sr = S[a];
    if (sr < r0 || sr >= r0 + nloc) continue;
    const double *src = reinterpret_cast<const double *>(c.Cs) + (size_t)(sr - r0) * c.qp;
    for (int e = c.lane; e < c.q; e += 32) __stcg(c.gG + (size_t)a * LRA_QMAX + e, src[e]);
  }
}
// element e of B[S[a],:] after the barrier (DSMEM read in the cluster tier, L2 in the grid tier)
__device__ __forceinline__ double S_row_elem(const Ctx &c, const long long *S, int a, int e) {
  if (c.grid) return __ldcg(c.gG + (size_t)a * LRA_QMAX + e);
  const long long sr = S[a];
  const double *src = reinterpret_cast<const double *>(c.Cs) + (size_t)(sr % c.rpc) * c.qp;
  return remote(c, src, (int)(sr / c.rpc))[e];
}

// ------------------------------------------------------ CTA reductions (1 barrier each)
// Non-negative doubles order like their bit patterns, so maxima are taken on 64-bit keys
// with two redux.sync.max.u32 (high word, then low word among the high-word winners);
// negative sentinels map to key 0.  Index minima use redux.sync.min.u32 (indices < 2^31),
// the value riding along from the winning lane by one shuffle.
__device__ __forceinline__ unsigned long long dkey(double v) {
  return v > 0.0 ? (unsigned long long)__double_as_longlong(v) : 0ull;
}
__device__ __forceinline__ unsigned long long warp_max_key(unsigned long long k) {
  const unsigned hi = (unsigned)(k >> 32);
  const unsigned mhi = __reduce_max_sync(0xffffffffu, hi);
  const unsigned mlo = __reduce_max_sync(0xffffffffu, hi == mhi ? (unsigned)k : 0u);
  return ((unsigned long long)mhi << 32) | mlo;
}
__device__ __forceinline__ void warp_min_idx(unsigned &i, double &v) {
  const unsigned m = __reduce_min_sync(0xffffffffu, i);
  const int src = __ffs(__ballot_sync(0xffffffffu, i == m)) - 1;
  v = __shfl_sync(0xffffffffu, v, src);
  i = m;
}
__device__ double cta_max1(Ctx &c, double v) {
  unsigned long long k = warp_max_key(dkey(v));
  const int b = c.rb;
  c.rb ^= 1;
  if (c.lane == 0) c.sh->rk[b][c.warp] = k;
  __syncthreads();
  k = warp_max_key(c.lane < c.nw ? c.sh->rk[b][c.lane] : 0ull);
  return __longlong_as_double((long long)k);
}
__device__ void cta_minidx1(Ctx &c, unsigned &i, double &v) {
  warp_min_idx(i, v);
  const int b = c.rb;
  c.rb ^= 1;
  if (c.lane == 0) { c.sh->ri[b][c.warp] = i; c.sh->rv[b][c.warp] = v; }
  __syncthreads();
  i = c.lane < c.nw ? c.sh->ri[b][c.lane] : 0xffffffffu;
  v = c.lane < c.nw ? c.sh->rv[b][c.lane] : 0.0;
  warp_min_idx(i, v);
}

// Cluster exchange of the CTA triples (M_c, idx_c, v_c); the CTA winner's row has been
// written to pub[p] by its owner thread.  Returns the global max M and the winning index
// (smallest index with value >= (1-tau) M), `amb` if a tie-window candidate makes the CTA
// candidates inexact; on success the winning row is copied into sh->prow (nwords doubles).
struct Pick {
  double M;
  long long idx;
  bool amb;
};
// mode 0: plain (prow only).  mode 1 (LU step t = arg): pm[j] = j > t ? prow[j] : 0.
// mode 2 (swap): jstar = winner % q, pm = prow - e_jstar, rc = 1 / prow[jstar].
__device__ Pick exchange(Ctx &c, int p, double Mc, long long idxc, double vc, int nwords, int mode = 0,
                         int arg = 0) {
  long long _tm = clock64();
  // push this CTA's triple into slot `rank` of every CTA (remote stores; ordered by the
  // cluster barrier's release/acquire), so the decision needs no remote load round trip
  if (c.grid) {
    if (c.tid == 0) {
      Tri *dst = c.gtri + (size_t)p * c.cs + c.rank;
      __stcg(&dst->M, Mc);
      __stcg(&dst->idx, idxc);
      __stcg(&dst->v, vc);
    }
  } else if (c.warp == 0 && c.lane < c.cs) {
    *remote(c, &c.sh->xin[p][c.rank], c.lane) = Tri{Mc, idxc, vc};
  }
  cluster_barrier(c);
  CA_MARK(11);
  if (c.warp == 0) {
    // per lane: the best of CTAs lane, lane+32, ... (grid tier: up to 148 CTAs)
    double tM = -INFINITY;
    long long tcand = LLONG_MAX;
    int tamb = 0, twr = -1;
    double Mloc = -INFINITY;
    for (int r = c.lane; r < c.cs; r += 32) {
      Tri t;
      if (c.grid) {
        const Tri *src = c.gtri + (size_t)p * c.cs + r;
        t = Tri{__ldcg(&src->M), __ldcg(&src->idx), __ldcg(&src->v)};
      } else {
        t = c.sh->xin[p][r];
      }
      Mloc = fmax(Mloc, t.M);
    }
    const double M = __longlong_as_double((long long)warp_max_key(dkey(Mloc)));
    const double thr = (1.0 - c.tau) * M;
    for (int r = c.lane; r < c.cs; r += 32) {
      Tri t;
      if (c.grid) {
        const Tri *src = c.gtri + (size_t)p * c.cs + r;
        t = Tri{__ldcg(&src->M), __ldcg(&src->idx), __ldcg(&src->v)};
      } else {
        t = c.sh->xin[p][r];
      }
      if (t.M >= thr && t.v >= thr && t.idx < tcand) { tcand = t.idx; twr = r; }
      if (t.M >= thr && t.v < thr) tamb = 1;
    }
    (void)tM;
    const int amb = __any_sync(0xffffffffu, tamb);
    const long long best = warp_min_ll(tcand);
    const int wl = __ffs(__ballot_sync(0xffffffffu, tcand == best && best != LLONG_MAX)) - 1;
    const int wr = wl >= 0 ? __shfl_sync(0xffffffffu, twr, wl) : -1;
    if (!amb && wr >= 0) {
      const double *src = c.grid ? c.grow + ((size_t)p * c.cs + wr) * LRA_QMAX : remote(c, &c.sh->pub[p][0], wr);
      const int js = (mode == 2) ? (int)(best % c.q) : -1;
      for (int j = c.lane; j < nwords; j += 32) {
        const double x = c.grid ? __ldcg(src + j) : src[j];
        c.sh->prow[j] = x;
        if (mode == 1) c.sh->pm[j] = (j > arg) ? x : 0.0;
        if (mode == 2) {
          c.sh->pm[j] = (j == js) ? x - 1.0 : x;
          if (j == js) c.sh->rc = 1.0 / x;
        }
      }
    }
    if (c.lane == 0) {
      c.sh->dM = M;
      c.sh->dbest = best;
      c.sh->damb = amb;
    }
  }
  __syncthreads();
  CA_MARK(12);
  return Pick{c.sh->dM, c.sh->dbest, c.sh->damb != 0};
}

// ------------------------------------------------------------------ register rows
// A block row is held by TPR consecutive lanes ("group"), lane s of the group owning the
// W = Q/TPR contiguous columns [s*W, s*W + W).  Per-row quantities are combined with
// xor-shuffles inside the group; selects / maxima use log-depth trees.
template <int W>
__device__ __forceinline__ double tsel(const double (&r)[W], int w) {   // r[w], runtime w
  double v[W];
#pragma unroll
  for (int i = 0; i < W; ++i) v[i] = r[i];
#pragma unroll
  for (int span = 1; span < W; span <<= 1) {
#pragma unroll
    for (int i = 0; i + span < W; i += 2 * span) v[i] = (w & span) ? v[i + span] : v[i];
  }
  return v[0];
}
template <int W>
__device__ __forceinline__ double tmaxabs(const double (&r)[W]) {
  double v[W];
#pragma unroll
  for (int i = 0; i < W; ++i) v[i] = fabs(r[i]);
#pragma unroll
  for (int span = 1; span < W; span <<= 1) {
#pragma unroll
    for (int i = 0; i + span < W; i += 2 * span) v[i] = fmax(v[i], v[i + span]);
  }
  return v[0];
}
// smallest local column w with |r[w]| >= thr (and global column < q), else W; value in v
template <int W>
__device__ __forceinline__ int tfirst(const double (&r)[W], double thr, int jbase, int q, double &v) {
  unsigned mask = 0;
#pragma unroll
  for (int i = 0; i < W; ++i) mask |= ((jbase + i < q) && fabs(r[i]) >= thr) ? (1u << i) : 0u;
  if (!mask) return W;
  const int w = __ffs(mask) - 1;
  v = fabs(tsel<W>(r, w));
  return w;
}
template <int TPR>
__device__ __forceinline__ double gmax(double v) {
#pragma unroll
  for (int o = 1; o < TPR; o <<= 1) v = fmax(v, __shfl_xor_sync(0xffffffffu, v, o));
  return v;
}
template <int TPR>
__device__ __forceinline__ void gminpair(int &j, double &v) {
#pragma unroll
  for (int o = 1; o < TPR; o <<= 1) {
    int oj = __shfl_xor_sync(0xffffffffu, j, o);
    double ov = __shfl_xor_sync(0xffffffffu, v, o);
    if (oj < j) { j = oj; v = ov; }
  }
}
template <int TPR>
__device__ __forceinline__ double gbcast(double v, int lane, int s) {
  return TPR == 1 ? v : __shfl_sync(0xffffffffu, v, (lane & ~(TPR - 1)) | s);
}

// ------------------------------------------------------------------ block loads
// Row i of the CTA (global block row r0 + i) is loaded by its TPR lanes, 8 loads in flight.
template <int TPR, typename F>
__device__ __forceinline__ void load_rows(Ctx &c, int nloc, F &&at) {
  double *Cs = reinterpret_cast<double *>(c.Cs);
  const int i = c.tid / TPR, s = c.tid % TPR;
  if (i >= nloc) return;
  for (int j0 = s; j0 < c.q; j0 += 8 * TPR) {
    double v[8];
#pragma unroll
    for (int u = 0; u < 8; ++u)
      if (j0 + u * TPR < c.q) v[u] = at(i, j0 + u * TPR);
#pragma unroll
    for (int u = 0; u < 8; ++u)
      if (j0 + u * TPR < c.q) Cs[(size_t)i * c.qp + j0 + u * TPR] = v[u];
  }
}

// Operand access specialised at compile time (keeps the kernel's code small).
template <int OPK>
__device__ __forceinline__ double op_at(const OpView &op, int64_t i, int64_t j) {
  if (OPK == 0) return (double)__ldg((const float *)op.w + j * op.ldw + i);
  if (OPK == 1) return __ldg((const double *)op.w + j * op.ldw + i);
  return op.f.at(i, j);
}

// ------------------------------------------------------------------ Gauss-Jordan inverse
// The q x q matrix X sits in the left part of the augmented [X | I] (row stride AS, right
// part at column R0 = Q, zero padded to width Q).  Gauss-Jordan with partial pivoting
// WITHOUT physical row swaps: step t picks the row p_t (not yet a pivot) of max |X[a][t]|
// (first on ties), scales it and eliminates column t from every other row.  The matrix
// is held in registers (warp w: rows w + 16k; lane l: columns l + 32m), so a step costs
// two barriers and ~100 bytes of shared traffic: per-warp pivot candidates, then the
// scaled pivot row.  Afterwards row t of X^{-1} is the right part of row piv[t], which is
// copied to the left part (rows t).  Every CTA computes the same result.  False if singular.
__device__ __noinline__ bool gj_inverse(CAShared *sh, double *A, int q, int R0, int AS, int nt) {
  const int WD = 2 * R0;                     // [X | I] width (row stride AS >= WD)
  const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5, nw = nt >> 5;
  double x[4][4];
#pragma unroll
  for (int k = 0; k < 4; ++k)
#pragma unroll
    for (int m = 0; m < 4; ++m) {
      const int a = warp + k * nw, bc = lane + 32 * m;
      x[k][m] = (a < q && bc < WD) ? A[a * AS + bc] : 0.0;
    }
  unsigned usedk = 0;                        // my rows already used as pivots (bit k)
  for (int t = 0; t < q; ++t) {
    const int mt = t >> 5, lt = t & 31, sl = t & 1;
    double v[4];
    unsigned long long key = 0ull;
    int arow = 0x7fffffff;
#pragma unroll
    for (int k = 0; k < 4; ++k) {
      double xv = x[k][0];
#pragma unroll
      for (int m = 1; m < 4; ++m) xv = (mt == m) ? x[k][m] : xv;
      v[k] = __shfl_sync(0xffffffffu, xv, lt);
      const int a = warp + k * nw;
      if (a < q && !((usedk >> k) & 1u)) {
        const double av = fabs(v[k]);
        const unsigned long long kk = (av != av) ? 0x7ff8000000000000ull : dkey(av);
        if (arow == 0x7fffffff || kk > key) { key = kk; arow = a; }
      }
    }
    if (lane == 0) { sh->gk[sl][warp] = key; sh->gr[sl][warp] = arow; }
    __syncthreads();
    unsigned long long ck = lane < nw ? sh->gk[sl][lane] : 0ull;
    const int cr = lane < nw ? sh->gr[sl][lane] : 0x7fffffff;
    const unsigned long long mk = warp_max_key(ck);
    const int p = (int)__reduce_min_sync(0xffffffffu, (ck == mk && cr != 0x7fffffff) ? (unsigned)cr : 0xffffffffu);
    if (p >= q) return false;
    const int kp = p / nw;
    if (tid == 0) sh->piv[t] = p;
    if (warp == p % nw) {                    // owner of the pivot row publishes it scaled
      const double d = v[kp == 0 ? 0 : (kp == 1 ? 1 : (kp == 2 ? 2 : 3))];
      const double rd = 1.0 / d;
#pragma unroll
      for (int m = 0; m < 4; ++m) {
        const int bc = lane + 32 * m;
        double xv = x[0][m];
#pragma unroll
        for (int k = 1; k < 4; ++k) xv = (kp == k) ? x[k][m] : xv;
        sh->gp[sl][bc] = (bc == t) ? 1.0 : xv * rd;
      }
      if (lane == 0) sh->gd[sl] = d;
    }
    __syncthreads();
    const double d = sh->gd[sl];
    if (!(fabs(d) > 0.0) || !isfinite(d)) return false;
#pragma unroll
    for (int k = 0; k < 4; ++k) {
      const int a = warp + k * nw;
      const bool isp = (a == p);
      if (isp) usedk |= 1u << k;
#pragma unroll
      for (int m = 0; m < 4; ++m) {
        const int bc = lane + 32 * m;
        const double pv = sh->gp[sl][bc];
        x[k][m] = isp ? pv : ((bc == t) ? 0.0 : fma(-v[k], pv, x[k][m]));
      }
    }
  }
#pragma unroll
  for (int k = 0; k < 4; ++k)
#pragma unroll
    for (int m = 0; m < 4; ++m) {
      const int a = warp + k * nw, bc = lane + 32 * m;
      if (a < q && bc < WD) A[a * AS + bc] = x[k][m];
    }
  __syncthreads();
  return true;
}

// out = base + sg * L * R on q x q blocks of aug (parts are column offsets, stride AS):
// base = I (bp < 0) or part bp.  Warp w: rows w + 16k; lanes: columns lane, lane + 32.
__device__ __forceinline__ void mm_small(const Ctx &c, int out, int lp, int rp, int bp, double sg) {
  const int q = c.q, AS = c.AS;
  double acc[4][2];
#pragma unroll
  for (int k = 0; k < 4; ++k) acc[k][0] = acc[k][1] = 0.0;
  for (int t = 0; t < q; ++t) {
    const double r0v = (c.lane < q) ? c.X[t * AS + rp + c.lane] : 0.0;
    const double r1v = (c.lane + 32 < q) ? c.X[t * AS + rp + c.lane + 32] : 0.0;
#pragma unroll
    for (int k = 0; k < 4; ++k) {
      const int i = c.warp + k * c.nw;
      const double l = (i < q) ? c.X[i * AS + lp + t] : 0.0;
      acc[k][0] = fma(l, r0v, acc[k][0]);
      acc[k][1] = fma(l, r1v, acc[k][1]);
    }
  }
  __syncthreads();                           // out may alias an input part
#pragma unroll
  for (int k = 0; k < 4; ++k) {
    const int i = c.warp + k * c.nw;
    if (i >= q) continue;
#pragma unroll
    for (int h = 0; h < 2; ++h) {
      const int j = c.lane + 32 * h;
      if (j >= c.QX) continue;
      double v = 0.0;
      if (j < q) {
        const double b = bp < 0 ? (i == j ? 1.0 : 0.0) : c.X[i * AS + bp + j];
        v = fma(sg, acc[k][h], b);
      }
      c.X[i * AS + out + j] = v;
    }
  }
  __syncthreads();
}

// own W columns of (row input in Cs) * G^{-1};  G^{-1} = aug[t][ib .. ib+Q)
template <int W>
__device__ __forceinline__ void product(const Ctx &c, int i, int jb, int ib, double (&row)[W]) {
  const double *Cs = reinterpret_cast<const double *>(c.Cs) + (size_t)i * c.qp;
#pragma unroll
  for (int w = 0; w < W; ++w) row[w] = 0.0;
  for (int t = 0; t < c.q; ++t) {
    const double b = Cs[t];
    const double2 *xr = reinterpret_cast<const double2 *>(c.X + t * c.AS + ib + jb);
#pragma unroll
    for (int w = 0; w < W / 2; ++w) {
      const double2 x = xr[w];
      row[2 * w] = fma(b, x.x, row[2 * w]);
      row[2 * w + 1] = fma(b, x.y, row[2 * w + 1]);
    }
  }
}

struct MVOut {
  int swaps, lu_steps;
  bool cap_hit;
  double cert;
};

// ------------------------------------------------------------------ real maxvol (registers)
// Block rows are in Cs (unchanged).  S: slot array (smem; cold: output, warm: input/output).
// G^{-1} (G = B[S,:]) lives in aug (q rows of width 2Q, at column offset c.ib): a cold step
// forms it by Gauss-Jordan on the gathered B[S,:]; every swap updates it with the same
// rank-1 formula as C (it is C for the "rows" of I_q), and since each C-A step's
// generator is the transpose of the previous step's final generator (W[I,J] vs W[I,J]^T),
// a warm start only transposes the carried inverse.
template <int Q, int TPR>
__device__ __forceinline__ bool maxvol_real(Ctx &c, int64_t N, long long *S, bool cold, bool carried, int cap,
                                            MVOut &o) {
  constexpr int W = Q / TPR;
  const int64_t r0 = (int64_t)c.rank * c.rpc;
  const int nloc = (int)max((int64_t)0, min((int64_t)c.rpc, N - r0));
  const int q = c.q;
  const int ri = c.tid / TPR, sub = c.tid % TPR, jb = sub * W;
  const bool has = ri < nloc;
  const long long grow = r0 + ri;
  const double *Cs = reinterpret_cast<const double *>(c.Cs) + (size_t)ri * c.qp;
  double row[W];
  int myslot = -1;
  o = MVOut{0, 0, false, 0.0};
  CA_T0();
  if (cold) {
#pragma unroll
    for (int w = 0; w < W; ++w) row[w] = (has && jb + w < q) ? Cs[jb + w] : 0.0;
    // ---- Alg D.2 stage 1: LUP with the slack pivot rule; bit-identical to the oracle
    for (int t = 0; t < q; ++t) {
      const int st = t / W, wt = t - st * W;
      const double x = gbcast<TPR>(tsel<W>(row, wt), c.lane, st);   // B'[row, t]
      double val = -1.0;
      if (has && myslot < 0) val = (x != x) ? INFINITY : fabs(x);
      const double Mc = cta_max1(c, val);
      const double thrc = (1.0 - c.tau) * Mc;
      unsigned ui = (has && myslot < 0 && val >= thrc) ? (unsigned)grow : 0xffffffffu;
      double v = val;
      cta_minidx1(c, ui, v);
      const long long idx = ui == 0xffffffffu ? LLONG_MAX : (long long)ui;
      int p = c.par;
      c.par ^= 1;
      if (has && grow == idx) {
        double *pb = pub_slot(c, p);
#pragma unroll
        for (int w = 0; w < W; ++w) pb[jb + w] = row[w];
      }
      Pick pk = exchange(c, p, Mc, idx, v, Q, 1, t);
      if (!(pk.M > 0.0) || !isfinite(pk.M)) return false;
      if (pk.amb) {                                  // exact second round (tie window)
        if (threadIdx.x == 0 && c.rank == 0) atomicAdd(&g_ca_cyc[8], 1ull);
        const double thr = (1.0 - c.tau) * pk.M;
        unsigned u2 = (has && myslot < 0 && val >= thr) ? (unsigned)grow : 0xffffffffu;
        double v2 = val;
        cta_minidx1(c, u2, v2);
        const long long i2 = u2 == 0xffffffffu ? LLONG_MAX : (long long)u2;
        p = c.par;
        c.par ^= 1;
        if (has && grow == i2) {
          double *pb = pub_slot(c, p);
#pragma unroll
          for (int w = 0; w < W; ++w) pb[jb + w] = row[w];
        }
        pk = exchange(c, p, pk.M, i2, v2, Q, 1, t);
      }
      const long long piv = pk.idx;
      if (c.tid == 0) S[t] = piv;
      if (has && grow == piv) myslot = t;
      if (has && myslot < 0) {            // B'[i, j] -= (B'[i,t]/B'[p,t]) B'[p,j], j > t
        const double f = x / c.sh->prow[t];
        const double2 *pm2 = reinterpret_cast<const double2 *>(c.sh->pm + jb);
#pragma unroll
        for (int w = 0; w < W / 2; ++w) {   // pm = 0 for j <= t: those entries are unchanged
          const double2 pv = pm2[w];
          row[2 * w] = rsub_mul(row[2 * w], f, pv.x);
          row[2 * w + 1] = rsub_mul(row[2 * w + 1], f, pv.y);
        }
      }
    }
    o.lu_steps = q;
    __syncthreads();
    CA_T1(1);
  } else if (has) {
    for (int s2 = 0; s2 < q; ++s2)
      if (S[s2] == grow) myslot = s2;
  }
  {
    CA_T0();
    if (cold || !carried) {
      // ---- G = B[S,:] gathered from the owners' shared memory, G^{-1} by Gauss-Jordan
      publish_S_rows(c, S, r0, nloc);
      cluster_barrier(c);                            // every CTA's block rows are loaded
      for (int a = c.warp; a < q; a += c.nw) {       // [G | I]
        for (int e = c.lane; e < 2 * Q; e += 32) {
          double xv;
          if (e < Q) xv = (e < q) ? S_row_elem(c, S, a, e) : 0.0;
          else xv = (e - Q == a) ? 1.0 : 0.0;
          c.X[a * c.AS + e] = xv;
        }
      }
      __syncthreads();
      CA_T1(2);
      CA_T0();
      if (!gj_inverse(c.sh, c.X, q, Q, c.AS, c.nt)) return false;
      // rows of G^{-1}: row t is the right part of row piv[t] -> left part, row t
      for (int a = c.warp; a < q; a += c.nw) {
        const int pr = c.sh->piv[a];
        for (int e = c.lane; e < Q; e += 32) c.X[a * c.AS + e] = c.X[pr * c.AS + Q + e];
      }
      c.ib = 0;
      __syncthreads();
      CA_T1(3);
    } else {
      // ---- carried inverse X0 = (G_prev^{-1})^T = G^{-1} up to the rounding accumulated by
      // the previous step's rank-1 updates; one Newton step X1 = X0 + X0 (I - G X0) against
      // the freshly gathered G restores a fresh-solve accuracy.
      const int cur = c.ib, pa = (cur + Q) % (3 * Q), pb = (cur + 2 * Q) % (3 * Q);
      for (int a = c.warp; a < q; a += c.nw)         // X0 = cur^T -> part pa
        for (int e = c.lane; e < Q; e += 32) c.X[a * c.AS + pa + e] = (e < q) ? c.X[e * c.AS + cur + a] : 0.0;
      publish_S_rows(c, S, r0, nloc);
      cluster_barrier(c);                            // every CTA's block rows are loaded
      for (int a = c.warp; a < q; a += c.nw)         // G = B[S,:] -> part pb
        for (int e = c.lane; e < Q; e += 32) c.X[a * c.AS + pb + e] = (e < q) ? S_row_elem(c, S, a, e) : 0.0;
      __syncthreads();
      mm_small(c, cur, pb, pa, -1, -1.0);            // R  = I - G X0   -> part cur
      mm_small(c, pb, pa, cur, pa, 1.0);             // X1 = X0 + X0 R  -> part pb
      c.ib = pb;
      CA_T1(2);
    }
  }
  {
    CA_T0();
    if (has && myslot < 0) product<W>(c, ri, jb, c.ib, row);
    __syncthreads();
    CA_T1(4);
  }
  double rmx = gmax<TPR>(tmaxabs<W>(row));
  if (!(has && myslot < 0)) rmx = -1.0;
  long long _ts = clock64();
  // ---- Alg D.1 swap loop
  for (int round = 0;; ++round) {
    long long _tm = clock64();
    const double Mc = cta_max1(c, rmx);
    CA_MARK(8);
    const double thrc = (1.0 - c.tau) * Mc;
    int jl = Q;
    double v = 0.0;
    if (has && myslot < 0 && rmx >= thrc) {
      const int w = tfirst<W>(row, thrc, jb, q, v);
      jl = (w < W) ? jb + w : Q;
    }
    gminpair<TPR>(jl, v);
    unsigned ui = (jl < q) ? (unsigned)(grow * q + jl) : 0xffffffffu;
    cta_minidx1(c, ui, v);
    const long long idx = ui == 0xffffffffu ? LLONG_MAX : (long long)ui;
    CA_MARK(9);
    int p = c.par;
    c.par ^= 1;
    if (has && idx != LLONG_MAX && grow == idx / q) {
      double *pb = pub_slot(c, p);
#pragma unroll
      for (int w = 0; w < W; ++w) pb[jb + w] = row[w];
    }
    CA_MARK(10);
    Pick pk = exchange(c, p, Mc, idx, v, Q, 2);
    _tm = clock64();
    if (!(pk.M == pk.M)) return false;
    if (pk.M <= 1.0 + c.tol || o.swaps >= cap) {
      o.cert = fmax(pk.M, 0.0);
      o.cap_hit = pk.M > 1.0 + c.tol;
      if (threadIdx.x == 0 && c.rank == 0) {
        atomicAdd(&g_ca_cyc[5], (unsigned long long)(clock64() - _ts));
        atomicAdd(&g_ca_cyc[7], (unsigned long long)(o.swaps + o.lu_steps));
      }
      return true;
    }
    if (pk.amb) {
      if (threadIdx.x == 0 && c.rank == 0) atomicAdd(&g_ca_cyc[8], 1ull);
      const double thr = (1.0 - c.tau) * pk.M;
      int j2 = Q;
      double v2 = 0.0;
      if (has && myslot < 0 && rmx >= thr) {
        const int w = tfirst<W>(row, thr, jb, q, v2);
        j2 = (w < W) ? jb + w : Q;
      }
      gminpair<TPR>(j2, v2);
      unsigned u2 = (j2 < q) ? (unsigned)(grow * q + j2) : 0xffffffffu;
      cta_minidx1(c, u2, v2);
      const long long i2 = u2 == 0xffffffffu ? LLONG_MAX : (long long)u2;
      p = c.par;
      c.par ^= 1;
      if (has && i2 != LLONG_MAX && grow == i2 / q) {
        double *pb = pub_slot(c, p);
#pragma unroll
        for (int w = 0; w < W; ++w) pb[jb + w] = row[w];
      }
      pk = exchange(c, p, pk.M, i2, v2, Q, 2);
    }
    const long long istar = pk.idx / q;
    const int jstar = (int)(pk.idx % q);
    const int sj = jstar / W, wj = jstar - sj * W;
    if (c.tid == 0) S[jstar] = istar;
    if (has && myslot == jstar) {                    // leaves S: explicit row e_{j*}
      myslot = -1;
#pragma unroll
      for (int w = 0; w < W; ++w) row[w] = (jb + w == jstar) ? 1.0 : 0.0;
    }
    if (has && grow == istar) myslot = jstar;        // enters S
    const double xj = gbcast<TPR>(tsel<W>(row, wj), c.lane, sj);
    const double rc = c.sh->rc;
    if (has && myslot < 0) {           // C <- C - C[:,j*] (C[i*,:] - e_j*) / c
      const double g = xj * rc;
      const double2 *pm2 = reinterpret_cast<const double2 *>(c.sh->pm + jb);
#pragma unroll
      for (int w = 0; w < W / 2; ++w) {
        const double2 pv = pm2[w];
        row[2 * w] = fma(-g, pv.x, row[2 * w]);
        row[2 * w + 1] = fma(-g, pv.y, row[2 * w + 1]);
      }
    }
    // the same update of the carried G^{-1} (every CTA keeps an identical copy)
    for (int a = c.warp; a < q; a += c.nw) {
      double *ir = c.X + a * c.AS + c.ib;
      const double g = ir[jstar] * rc;
      __syncwarp();
      for (int e = c.lane; e < q; e += 32) ir[e] = fma(-g, c.sh->pm[e], ir[e]);
    }
    rmx = gmax<TPR>(tmaxabs<W>(row));
    if (!(has && myslot < 0)) rmx = -1.0;
    ++o.swaps;
    CA_MARK(14);
  }
}

// ------------------------------------------------- complex maxvol (ARFT sketch, smem rows)
__device__ double cta_max_c(Ctx &c, double v) { return cta_max1(c, v); }
__device__ long long cta_min_c(Ctx &c, long long v) {
  double dummy = 0.0;
  unsigned u = v == LLONG_MAX ? 0xffffffffu : (unsigned)v;
  cta_minidx1(c, u, dummy);
  return u == 0xffffffffu ? LLONG_MAX : (long long)u;
}
__device__ double cluster_max_c(Ctx &c, double v) {
  v = cta_max_c(c, v);
  if (c.cs == 1) return v;
  cg::cluster_group cl = cg::this_cluster();
  const int p = c.par;
  c.par ^= 1;
  if (c.tid == 0) c.sh->xd[p] = v;
  cl.sync();
  double x = c.lane < c.cs ? *cl.map_shared_rank(&c.sh->xd[p], c.lane) : -INFINITY;
  return warp_max(x);
}
__device__ long long cluster_min_c(Ctx &c, long long v) {
  v = cta_min_c(c, v);
  if (c.cs == 1) return v;
  cg::cluster_group cl = cg::this_cluster();
  const int p = c.par;
  c.par ^= 1;
  if (c.tid == 0) c.sh->xi[p] = v;
  cl.sync();
  long long x = c.lane < c.cs ? *cl.map_shared_rank(&c.sh->xi[p], c.lane) : LLONG_MAX;
  return warp_min_ll(x);
}
__device__ const cplx *remote_row_c(const Ctx &c, int owner, int row_loc) {
  cplx *base = reinterpret_cast<cplx *>(c.Cs) + (size_t)row_loc * c.qp;
  return remote(c, base, owner);
}

__device__ __noinline__ bool maxvol_complex(Ctx &c, int64_t N, long long *S, int cap, MVOut &o) {
  using K = Sc<cplx>;
  cplx *Cs = reinterpret_cast<cplx *>(c.Cs);
  cplx *prow = reinterpret_cast<cplx *>(c.sh->prow);
  cplx *Ls = reinterpret_cast<cplx *>(c.X);
  const int64_t r0 = (int64_t)c.rank * c.rpc;
  const int nloc = (int)max((int64_t)0, min((int64_t)c.rpc, N - r0));
  const int q = c.q;
  o = MVOut{0, q, false, 0.0};
  for (int i = c.tid; i < c.rpc; i += c.nt) c.inS[i] = 0;
  __syncthreads();
  for (int t = 0; t < q; ++t) {
    double lm = -1.0;
    for (int i = c.tid; i < nloc; i += c.nt)
      if (!c.inS[i]) {
        double a = K::abs(Cs[(size_t)i * c.qp + t]);
        lm = fmax(lm, a != a ? INFINITY : a);
      }
    const double M = cluster_max_c(c, lm);
    if (!(M > 0.0) || !isfinite(M)) return false;
    const double thr = (1.0 - c.tau) * M;
    long long li = LLONG_MAX;
    for (int i = c.tid; i < nloc; i += c.nt)
      if (!c.inS[i] && K::abs(Cs[(size_t)i * c.qp + t]) >= thr) { li = r0 + i; break; }
    const long long p = cluster_min_c(c, li);
    const int owner = (int)(p / c.rpc), ploc = (int)(p % c.rpc);
    if (c.tid < q) prow[c.tid] = remote_row_c(c, owner, ploc)[c.tid];
    if (c.tid == 0) {
      S[t] = p;
      if (owner == c.rank) c.inS[ploc] = 1;
    }
    __syncthreads();
    if (c.tid < t) Ls[t * (t - 1) / 2 + c.tid] = prow[c.tid];
    const cplx piv = prow[t];
    for (int i = c.tid; i < nloc; i += c.nt) {
      if (c.inS[i]) continue;
      cplx *row = Cs + (size_t)i * c.qp;
      const cplx f = K::div(row[t], piv);
      row[t] = f;
      for (int j = t + 1; j < q; ++j) row[j] = K::sub_mul(row[j], f, prow[j]);
    }
    __syncthreads();
  }
  for (int i = c.tid; i < nloc; i += c.nt) {
    if (c.inS[i]) continue;
    cplx *row = Cs + (size_t)i * c.qp;
    double mx = 0.0;
    for (int j = q - 1; j >= 0; --j) {
      cplx acc = row[j];
      for (int t = j + 1; t < q; ++t) acc = K::fsub_mul(acc, row[t], Ls[t * (t - 1) / 2 + j]);
      row[j] = acc;
      mx = fmax(mx, K::abs(acc));
    }
    c.rmax[i] = mx;
  }
  __syncthreads();
  for (;;) {
    double lm = 0.0;
    for (int i = c.tid; i < nloc; i += c.nt)
      if (!c.inS[i]) lm = fmax(lm, c.rmax[i]);
    const double M = cluster_max_c(c, lm);
    if (!(M == M)) return false;
    if (M <= 1.0 + c.tol || o.swaps >= cap) {
      o.cert = M;
      o.cap_hit = M > 1.0 + c.tol;
      return true;
    }
    const double thr = (1.0 - c.tau) * M;
    long long li = LLONG_MAX;
    for (int i = c.tid; i < nloc && li == LLONG_MAX; i += c.nt) {
      if (c.inS[i] || c.rmax[i] < thr) continue;
      const cplx *row = Cs + (size_t)i * c.qp;
      for (int j = 0; j < q; ++j)
        if (K::abs(row[j]) >= thr) { li = (r0 + i) * (long long)q + j; break; }
    }
    const long long L = cluster_min_c(c, li);
    const long long istar = L / q;
    const int jstar = (int)(L % q);
    const int owner = (int)(istar / c.rpc);
    if (c.tid < q) prow[c.tid] = remote_row_c(c, owner, (int)(istar % c.rpc))[c.tid];
    const long long sold = S[jstar];
    __syncthreads();
    if (c.tid == 0) {
      S[jstar] = istar;
      if (owner == c.rank) c.inS[istar % c.rpc] = 1;
      if (sold / c.rpc == c.rank) {
        int sl = (int)(sold % c.rpc);
        c.inS[sl] = 0;
        cplx *row = Cs + (size_t)sl * c.qp;
        for (int j = 0; j < q; ++j) row[j] = (j == jstar) ? K::one() : K::zero();
      }
    }
    __syncthreads();
    const cplx piv = prow[jstar];
    for (int i = c.tid; i < nloc; i += c.nt) {
      if (c.inS[i]) continue;
      cplx *row = Cs + (size_t)i * c.qp;
      const cplx g = K::div(row[jstar], piv);
      double mx = 0.0;
      for (int j = 0; j < q; ++j) {
        cplx v = (j == jstar) ? g : K::fsub_mul(row[j], g, prow[j]);
        row[j] = v;
        mx = fmax(mx, K::abs(v));
      }
      c.rmax[i] = mx;
    }
    __syncthreads();
    ++o.swaps;
  }
}

// ------------------------------------------------------------------ context setup
template <int Q, int NT>
__device__ __forceinline__ void ctx_init(Ctx &c, CAShared *sh, unsigned char *dsm, const CAArgs &a) {
  c.sh = sh;
  c.cs = a.cs;
  c.rank = (a.cs > 1) ? (int)cg::this_cluster().block_rank() : 0;
  c.rpc = a.rpc;
  c.qp = a.qp;
  c.q = a.q;
  c.QX = Q;
  c.R0 = Q;
  c.AS = 3 * Q;
  c.ib = 0;
  c.tid = threadIdx.x;
  c.lane = threadIdx.x & 31;
  c.warp = threadIdx.x >> 5;
  c.nt = NT;
  c.nw = NT / 32;
  c.par = 0;
  c.rb = 0;
  c.tau = a.tau;
  c.tol = a.tol;
  c.grid = a.grid;
  c.gtri = reinterpret_cast<Tri *>(a.gscratch);
  c.grow = a.gscratch ? reinterpret_cast<double *>(c.gtri + 2 * (size_t)a.cs) : nullptr;
  c.gG = a.gscratch ? c.grow + 2 * (size_t)a.cs * LRA_QMAX : nullptr;
  if (a.grid) c.rank = blockIdx.x;
  const size_t esz = a.y_complex ? 16 : 8;
  size_t off = 0;
  c.Cs = dsm;
  off += (size_t)a.rpc * a.qp * esz;
  off = (off + 15) & ~(size_t)15;
  c.X = reinterpret_cast<double *>(dsm + off);
  off += a.y_complex ? (size_t)a.q * (a.q - 1) / 2 * 16 : (size_t)a.q * 3 * Q * 8;
  c.rmax = reinterpret_cast<double *>(dsm + off);
  off += (size_t)a.rpc * 8;
  c.inS = dsm + off;
}

// Stage 2 on a complex (ARFT) sketch: I0 <- maxvol(Y), written to a.I; its counters go
// to a.yinfo[4b..4b+3] = (status, swaps, cap_hit, lu_steps) for the C-A kernel.
template <int NT>
__global__ void __launch_bounds__(NT, 1) k_ca_ycplx(CAArgs a) {
  extern __shared__ __align__(16) unsigned char dsm[];
  __shared__ CAShared sh;
  Ctx c;
  ctx_init<LRA_QMAX, NT>(c, &sh, dsm, a);
  const int64_t b = blockIdx.x / a.cs;
  const int64_t r0 = (int64_t)c.rank * c.rpc;
  const int64_t m = a.op.m;
  const int nloc = (int)max((int64_t)0, min((int64_t)c.rpc, m - r0));
  const cplx *Y = reinterpret_cast<const cplx *>(a.Y) + b * a.y_stride;
  cplx *Cs = reinterpret_cast<cplx *>(c.Cs);
  for (int e = c.tid; e < nloc * a.q; e += NT) {
    int j = e / nloc, i = e % nloc;
    Cs[(size_t)i * c.qp + j] = Y[(int64_t)j * a.ldy + r0 + i];
  }
  __syncthreads();
  MVOut o;
  const bool ok = maxvol_complex(c, m, sh.Isl, a.cap, o);
  __syncthreads();
  if (c.rank == 0) {
    if (c.tid < a.q) a.I[b * a.q + c.tid] = sh.Isl[c.tid];
    if (c.tid == 0) {
      a.yinfo[4 * b + 0] = ok ? LRA_OK : LRA_ESINGULAR;
      a.yinfo[4 * b + 1] = o.swaps;
      a.yinfo[4 * b + 2] = o.cap_hit;
      a.yinfo[4 * b + 3] = o.lu_steps;
    }
  }
  cluster_barrier(c);
}

// ------------------------------------------------------------------ the C-A kernel
// Steps: 0 = stage 2 on a real Y (cold); then 2L+1 = horizontal step of loop L
// (J <- maxvol(W[I,:]^T), cold in loop 0), 2L+2 = vertical step (I <- maxvol(W[:,J]), warm).
template <int Q, int TPR, int NT, int OPK>
__global__ void __launch_bounds__(NT, 1) k_ca(CAArgs a) {
  if (a.skip && (a.skip[0] != 0 || a.skip[1] != 0)) return;   // row-sharded chain: step not needed
  extern __shared__ __align__(16) unsigned char dsm[];
  __shared__ CAShared sh;
  Ctx c;
  ctx_init<Q, NT>(c, &sh, dsm, a);
  const int64_t b = a.grid ? 0 : blockIdx.x / a.cs;
  OpView op = a.op;
  if (op.kind == LRA_OP_DENSE)
    op.w = (const char *)op.w + b * a.w_stride * (op.dtype == LRA_F32 ? 4 : 8);
  const int q = a.q;
  int32_t status = LRA_OK;
  int lu = 0, swaps = 0, caps = 0, sk_swaps = 0, loops = 0, sw_h = 0;
  double cert_r = 0.0, cert_c = 0.0;
  const int64_t r0 = (int64_t)c.rank * c.rpc;
  const bool yreal = a.Y != nullptr && !a.y_complex;
  if (!yreal) {
    if (c.tid < q) sh.Isl[c.tid] = a.I0[b * a.i0_stride + c.tid];
    if (a.yinfo) {
      status = a.yinfo[4 * b + 0];
      swaps = sk_swaps = a.yinfo[4 * b + 1];
      caps = a.yinfo[4 * b + 2];
      lu = a.yinfo[4 * b + 3];
    }
    __syncthreads();
  }
  const double *Y = yreal ? reinterpret_cast<const double *>(a.Y) + b * a.y_stride : nullptr;
  const int last = 2 * a.sweeps;
  long long _tk = clock64();
  for (int step = yreal ? 0 : 1; status == LRA_OK && step <= last; ++step) {
    const int kind = step == 0 ? 0 : ((step & 1) ? 1 : 2);        // 0 = Y, 1 = h, 2 = v
    const int64_t N = kind == 1 ? op.n : op.m;
    long long *S = kind == 1 ? sh.Jsl : sh.Isl;
    const bool cold = step <= 1;
    cluster_barrier(c);                                             // previous block no longer read
    CA_T0();
    {
      const int nloc = (int)max((int64_t)0, min((int64_t)c.rpc, N - r0));
      const long long *I = sh.Isl, *J = sh.Jsl;
      load_rows<TPR>(c, nloc, [&](int i, int j) -> double {
        if (kind == 0) return __ldg(Y + (int64_t)j * a.ldy + r0 + i);
        if (kind == 1) return op_at<OPK>(op, I[j], r0 + i);
        return op_at<OPK>(op, r0 + i, J[j]);
      });
    }
    __syncthreads();
    CA_T1(0);
    MVOut o;
    if (!maxvol_real<Q, TPR>(c, N, S, cold, step >= 2, a.cap, o)) {
      status = LRA_ESINGULAR;
      break;
    }
    lu += o.lu_steps;
    swaps += o.swaps;
    caps += o.cap_hit;
    if (kind == 0) sk_swaps = o.swaps;
    if (kind == 1) { cert_c = o.cert; sw_h = o.swaps; }
    if (kind == 2) {
      cert_r = o.cert;
      ++loops;
      if (step > 2 && sw_h == 0 && o.swaps == 0) break;           // fixed point (reading C13)
    }
  }
  __syncthreads();
  if (threadIdx.x == 0 && c.rank == 0) atomicAdd(&g_ca_cyc[6], (unsigned long long)(clock64() - _tk));
  if (c.rank == 0) {
    if (c.tid < q) {
      a.I[b * q + c.tid] = sh.Isl[c.tid];
      a.J[b * q + c.tid] = sh.Jsl[c.tid];
    }
    if (c.tid == 0) {
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
  cluster_barrier(c);                // keep every CTA's shared memory alive until done
}

static size_t ca_smem_bytes(int rpc, int qp, int q, int Q, bool cplx) {
  const size_t esz = cplx ? 16 : 8;
  size_t off = (size_t)rpc * qp * esz;
  off = (off + 15) & ~(size_t)15;
  off += cplx ? (size_t)q * (q - 1) / 2 * 16 : (size_t)q * 3 * Q * 8;
  off += (size_t)rpc * 8 + (size_t)rpc;
  return (off + 15) & ~(size_t)15;
}

template <typename K>
static cudaError_t launch_cluster(K kern, const CAArgs &a, int64_t nb, int nt, size_t smem, cudaStream_t st) {
  cudaError_t e = cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
  if (e != cudaSuccess) return e;
  if (a.cs > 8) {
    e = cudaFuncSetAttribute(kern, cudaFuncAttributeNonPortableClusterSizeAllowed, 1);
    if (e != cudaSuccess) return e;
  }
  cudaLaunchConfig_t cfg = {};
  cfg.gridDim = dim3((unsigned)(nb * a.cs));
  cfg.blockDim = dim3(nt);
  cfg.dynamicSmemBytes = smem;
  cfg.stream = st;
  cudaLaunchAttribute attr[1];
  attr[0].id = cudaLaunchAttributeClusterDimension;
  attr[0].val.clusterDim.x = a.cs;
  attr[0].val.clusterDim.y = 1;
  attr[0].val.clusterDim.z = 1;
  cfg.attrs = attr;
  cfg.numAttrs = 1;
  return cudaLaunchKernelEx(&cfg, kern, a);
}

static bool pick_cluster(int64_t maxN, int nt, int qp, int q, int Q, bool cplx, int &cs, int &rpc) {
  const size_t limit = 227 * 1024 - sizeof(CAShared) - 256;
  for (cs = 1; cs <= 16; cs *= 2) {
    rpc = (int)((maxN + cs - 1) / cs);
    if (rpc <= nt && ca_smem_bytes(rpc, qp, q, Q, cplx) <= limit) return true;
  }
  return false;
}

size_t ca_grid_scratch_bytes(int cs) {
  return (size_t)2 * cs * sizeof(Tri) + (size_t)2 * cs * LRA_QMAX * 8 + (size_t)LRA_QMAX * LRA_QMAX * 8 + 256;
}

static int num_sms() {
  static int n = 0;
  if (!n) {
    int dev = 0;
    cudaGetDevice(&dev);
    cudaDeviceGetAttribute(&n, cudaDevAttrMultiProcessorCount, dev);
  }
  return n;
}

template <int Q, int TPR, int NT>
static cudaError_t launch_ca_t(CAArgs a, int64_t nb, int64_t maxN, cudaStream_t st, int *cs_out, Prof *pf) {
  cudaError_t e;
  if (a.y_complex) {                         // stage 2 on the complex sketch: own launch
    CAArgs y = a;
    if (!pick_cluster(a.op.m, 512, a.qp, a.q, LRA_QMAX, true, y.cs, y.rpc)) return cudaErrorInvalidConfiguration;
    pf->begin("k_ca_ycplx", st);
    e = launch_cluster(k_ca_ycplx<512>, y, nb, 512, ca_smem_bytes(y.rpc, y.qp, y.q, LRA_QMAX, true), st);
    pf->end(st);
    if (e != cudaSuccess) return e;
    a.I0 = a.I;
    a.i0_stride = a.q;
  }
  int cs, rpc;
  CAArgs r = a;
  r.y_complex = 0;
  if (a.y_complex) r.Y = nullptr;
  // small tier (ca_small.cu: one 128-thread CTA per problem, q <= 20, <= 512 rows), then the
  // cluster tier (ca_cluster.cu, q <= 48); k_ca's cluster form below covers 48 < q <= 64
  e = launch_ca_small(r, nb, maxN, st, cs_out, pf);
  if (e != cudaErrorInvalidConfiguration) return e;
  cudaGetLastError();
  e = launch_ca_cluster(r, nb, maxN, st, cs_out, pf);
  if (e != cudaErrorInvalidConfiguration) return e;
  cudaGetLastError();
  if (pick_cluster(maxN, NT / TPR, a.qp, a.q, Q, false, cs, rpc)) {   // cluster tier
    r.cs = cs;
    r.rpc = rpc;
    r.grid = 0;
    if (cs_out) *cs_out = cs;
    const size_t smem = ca_smem_bytes(rpc, a.qp, a.q, Q, false);
    pf->begin("k_ca", st);
    if (a.op.kind == LRA_OP_FACTORED_CSR) e = launch_cluster(k_ca<Q, TPR, NT, 2>, r, nb, NT, smem, st);
    else if (a.op.dtype == LRA_F64) e = launch_cluster(k_ca<Q, TPR, NT, 1>, r, nb, NT, smem, st);
    else e = launch_cluster(k_ca<Q, TPR, NT, 0>, r, nb, NT, smem, st);
    pf->end(st);
    return e;
  }
  // grid tier: one problem over ceil(maxN / rows-per-CTA) co-resident CTAs (cooperative)
  rpc = NT / TPR;
  cs = (int)((maxN + rpc - 1) / rpc);
  const size_t smem = ca_smem_bytes(rpc, a.qp, a.q, Q, false);
  if (cs > num_sms() || smem > 227 * 1024 - sizeof(CAShared) - 256 || !a.gscratch || a.y_complex)
    return cudaErrorInvalidConfiguration;
  r.cs = cs;
  r.rpc = rpc;
  r.grid = 1;
  if (cs_out) *cs_out = cs;
  void (*kern)(CAArgs) = a.op.kind == LRA_OP_FACTORED_CSR ? k_ca<Q, TPR, NT, 2>
                         : (a.op.dtype == LRA_F64 ? k_ca<Q, TPR, NT, 1> : k_ca<Q, TPR, NT, 0>);
  e = cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
  if (e != cudaSuccess) return e;
  const size_t esz = 8;
  for (int64_t b = 0; b < nb; ++b) {
    CAArgs rb = r;
    if (rb.op.kind == LRA_OP_DENSE)
      rb.op.w = (const char *)rb.op.w + b * rb.w_stride * (rb.op.dtype == LRA_F32 ? 4 : 8);
    if (rb.Y) rb.Y = (const char *)rb.Y + b * rb.y_stride * esz;
    if (rb.I0) rb.I0 += b * rb.i0_stride;
    rb.I += b * a.q;
    rb.J += b * a.q;
    if (rb.stats) rb.stats += b;
    rb.status += b;
    if (rb.yinfo) rb.yinfo += 4 * b;
    cudaLaunchConfig_t cfg = {};
    cfg.gridDim = dim3((unsigned)cs);
    cfg.blockDim = dim3(NT);
    cfg.dynamicSmemBytes = smem;
    cfg.stream = st;
    cudaLaunchAttribute attr[1];
    attr[0].id = cudaLaunchAttributeCooperative;
    attr[0].val.cooperative = 1;
    cfg.attrs = attr;
    cfg.numAttrs = 1;
    pf->begin("k_ca_grid", st);
    e = cudaLaunchKernelEx(&cfg, kern, rb);
    pf->end(st);
    if (e != cudaSuccess) return e;
  }
  return cudaSuccess;
}

// old-kernel counters + cluster-tier counters (ca_cluster.cu), elementwise (one of them is
// zero for any given run)
cudaError_t read_ca_counters(unsigned long long *out, bool reset) {
  cudaError_t e = cudaMemcpyFromSymbol(out, g_ca_cyc, sizeof(g_ca_cyc));
  if (e == cudaSuccess && reset) {
    unsigned long long z[16] = {0};
    e = cudaMemcpyToSymbol(g_ca_cyc, z, sizeof(z));
  }
  unsigned long long c2[16];
  if (e == cudaSuccess) e = read_cc_counters(c2, reset);
  if (e == cudaSuccess)
    for (int i = 0; i < 16; ++i) out[i] += c2[i];
  unsigned long long gx = 0;
  if (e == cudaSuccess) e = read_gm_exact(&gx, reset);
  if (e == cudaSuccess) out[8] += gx;          // exact second rounds of the global-memory tier
  unsigned long long nc[2];
  if (e == cudaSuccess) e = read_nuc_counters(nc, reset);
  if (e == cudaSuccess) { out[14] = nc[0]; out[15] = nc[1]; }
  return e;
}

bool ca_needs_global(int64_t maxN, int q) {
  static const bool force = getenv("LRA_CA_FORCE_GLOBAL") != nullptr;   // diagnostics / tests
  if (force || q > LRA_QMAX) return true;
  // cluster tier (ca_cluster.cu): 16 CTAs x 512/TPR rows (TPR = 1 for q <= 24, else 2)
  const int64_t rpc_cl = q <= 24 ? 512 : 256;
  if (q <= 48 && maxN <= 16 * rpc_cl) return false;
  // grid tier (ca.cu): one CTA per SM, NT/TPR = 256 rows each (TPR = 2 for q > 24)
  const int64_t rpc_g = q <= 24 ? 512 : 256;
  if (maxN <= (int64_t)num_sms() * rpc_g &&
      ca_smem_bytes((int)rpc_g, q | 1, q, q <= 8 ? 8 : (q <= 16 ? 16 : (q <= 24 ? 24 : (q <= 32 ? 32 : (q <= 48 ? 48 : 64)))),
                    false) <= 227 * 1024 - sizeof(CAShared) - 256)
    return false;
  return true;
}

cudaError_t launch_ca(CAArgs a, int64_t nb, int64_t maxN, cudaStream_t st, int *cs_out, Prof *pf) {
  // (Q, threads per row, CTA threads): W = Q/TPR doubles of the row per lane
  if (a.q <= 8) return launch_ca_t<8, 1, 512>(a, nb, maxN, st, cs_out, pf);
  if (a.q <= 16) return launch_ca_t<16, 1, 512>(a, nb, maxN, st, cs_out, pf);
  if (a.q <= 24) return launch_ca_t<24, 1, 512>(a, nb, maxN, st, cs_out, pf);
  if (a.q <= 32) return launch_ca_t<32, 2, 512>(a, nb, maxN, st, cs_out, pf);
  if (a.q <= 48) return launch_ca_t<48, 2, 512>(a, nb, maxN, st, cs_out, pf);
  return launch_ca_t<64, 2, 512>(a, nb, maxN, st, cs_out, pf);
}

}  // namespace lra
