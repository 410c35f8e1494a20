// ca.cu — stages 2-3 of Alg 10.2 with C-A iterations (Remark rerfnhmt),
// each C-A step a maxvol on a tall-skinny block: Alg D.2 stage 1 (LUP cold start,
// P:6550-6556) and the Alg D.1 swap loop with the rank-1 update.
//
// One thread-block CLUSTER per problem.  The N x q C-matrix of the current step lives in
// the cluster's distributed shared memory: CTA `rank` owns rows [rank*rpc, rank*rpc+rpc),
// one row per thread, fp64 (complex128 for the ARFT sketch).  Every pivot decision is a
// two-phase cluster reduction (global max, then the smallest row-major index with
// |c| >= (1-tau) max, reading C11) through DSMEM exchange slots; the pivot row is fetched
// from its owner's shared memory (ld.shared::cluster).  Rows in the selected set S are
// kept implicit (they are identity rows of C = (I_q | C'), reading C12b), so no CTA ever
// writes a row another CTA may be reading.  Blocks are gathered straight from W in HBM
// (vertical W[:,J]: coalesced columns; horizontal W[I,:]^T: one sector per element).
// The whole C-A (all sweeps, early exit) runs in one launch: no host round trips.
#include <cooperative_groups.h>
#include <climits>

#include "kernels.cuh"

namespace cg = cooperative_groups;

namespace lra {


struct CAShared {
  long long Isl[LRA_QMAX], Jsl[LRA_QMAX];
  double xd[2];
  long long xi[2];
  double red_d[LRA_NT / 32];
  long long red_i[LRA_NT / 32];
  double bd;
  long long bi;
  int piv[LRA_QMAX];
  int sing;
};

struct Ctx {
  CAShared *sh;
  unsigned char *smem_dyn;     // [Cs | Ls | prow | rmax | inS]
  void *Cs;                    // rpc x qp of T
  double *Ls;                  // L_S packed (cold) or G^T LU (warm, real)
  void *prow;                  // q of T
  double *rmax;                // rpc
  unsigned char *inS;          // rpc
  int rank, cs, rpc, qp, q, tid, lane, warp;
  int par;                     // exchange slot parity (identical in every CTA)
  double tau, tol;
};

// ------------------------------------------------------------------ reductions
__device__ double cta_max(Ctx &c, double v) {
  v = warp_max(v);
  if (c.lane == 0) c.sh->red_d[c.warp] = v;
  __syncthreads();
  if (c.warp == 0) {
    double x = c.lane < LRA_NT / 32 ? c.sh->red_d[c.lane] : -INFINITY;
    x = warp_max(x);
    if (c.lane == 0) c.sh->bd = x;
  }
  __syncthreads();
  return c.sh->bd;
}
__device__ long long cta_min(Ctx &c, long long v) {
  v = warp_min_ll(v);
  if (c.lane == 0) c.sh->red_i[c.warp] = v;
  __syncthreads();
  if (c.warp == 0) {
    long long x = c.lane < LRA_NT / 32 ? c.sh->red_i[c.lane] : LLONG_MAX;
    x = warp_min_ll(x);
    if (c.lane == 0) c.sh->bi = x;
  }
  __syncthreads();
  return c.sh->bi;
}
// Cluster-wide max: every CTA reduces the same CS partials in the same order, so all
// CTAs take the same decision.  Slots alternate parity; a slot is rewritten only after
// the next cluster barrier, by which time every reader of its previous value is done.
__device__ double cluster_max(Ctx &c, double v) {
  v = cta_max(c, v);
  if (c.cs == 1) return v;
  cg::cluster_group cl = cg::this_cluster();
  const int p = c.par;
  c.par ^= 1;
  if (c.tid == 0) c.sh->xd[p] = v;
  cl.sync();
  if (c.warp == 0) {
    double x = c.lane < c.cs ? *cl.map_shared_rank(&c.sh->xd[p], c.lane) : -INFINITY;
    x = warp_max(x);
    if (c.lane == 0) c.sh->bd = x;
  }
  __syncthreads();
  return c.sh->bd;
}
__device__ long long cluster_min(Ctx &c, long long v) {
  v = cta_min(c, v);
  if (c.cs == 1) return v;
  cg::cluster_group cl = cg::this_cluster();
  const int p = c.par;
  c.par ^= 1;
  if (c.tid == 0) c.sh->xi[p] = v;
  cl.sync();
  if (c.warp == 0) {
    long long x = c.lane < c.cs ? *cl.map_shared_rank(&c.sh->xi[p], c.lane) : LLONG_MAX;
    x = warp_min_ll(x);
    if (c.lane == 0) c.sh->bi = x;
  }
  __syncthreads();
  return c.sh->bi;
}
__device__ __forceinline__ void cluster_barrier(const Ctx &c) {
  if (c.cs > 1) cg::this_cluster().sync();
  else __syncthreads();
}
// pointer to element (row, col) of the C-matrix held by CTA `owner`
template <typename T>
__device__ __forceinline__ const T *remote_row(const Ctx &c, int owner, int row_loc) {
  T *base = reinterpret_cast<T *>(c.Cs) + (size_t)row_loc * c.qp;
  if (c.cs == 1) return base;
  return cg::this_cluster().map_shared_rank(base, owner);
}

// ------------------------------------------------------------------ block loads
template <typename T>
__device__ void load_Y(Ctx &c, const void *Yb, int64_t ldy, int64_t N) {
  const int64_t r0 = (int64_t)c.rank * c.rpc;
  const int nloc = (int)max((int64_t)0, min((int64_t)c.rpc, N - r0));
  T *Cs = reinterpret_cast<T *>(c.Cs);
  const T *Y = reinterpret_cast<const T *>(Yb);
  for (int e = c.tid; e < nloc * c.q; e += LRA_NT) {
    int j = e / nloc, i = e % nloc;
    Cs[(size_t)i * c.qp + j] = Y[(int64_t)j * ldy + r0 + i];
  }
}
// vertical block W[:, J] (N = m rows)
__device__ void load_cols(Ctx &c, const OpView &op, const long long *J, int64_t N) {
  const int64_t r0 = (int64_t)c.rank * c.rpc;
  const int nloc = (int)max((int64_t)0, min((int64_t)c.rpc, N - r0));
  double *Cs = reinterpret_cast<double *>(c.Cs);
  for (int e = c.tid; e < nloc * c.q; e += LRA_NT) {
    int j = e / nloc, i = e % nloc;
    Cs[(size_t)i * c.qp + j] = op.at(r0 + i, J[j]);
  }
}
// horizontal block W[I, :]^T (N = n rows; block row = column of W)
__device__ void load_rowsT(Ctx &c, const OpView &op, const long long *I, int64_t N) {
  const int64_t r0 = (int64_t)c.rank * c.rpc;
  const int nloc = (int)max((int64_t)0, min((int64_t)c.rpc, N - r0));
  double *Cs = reinterpret_cast<double *>(c.Cs);
  for (int e = c.tid; e < nloc * c.q; e += LRA_NT) {
    int s = e / nloc, i = e % nloc;
    Cs[(size_t)i * c.qp + s] = op.at(I[s], r0 + i);
  }
}

// ------------------------------------------------------------------ maxvol pieces
struct MVOut {
  int swaps, lu_steps;
  bool cap_hit;
  double cert;
};

// Alg D.2 stage 1: LU with partial pivoting (slack rule), pivots -> S; then C = L L_S^{-1}
// for the non-pivot rows (C = B B_S^{-1}, Alg D.2 stage 2).  Returns false if singular.
template <typename T>
__device__ bool lup_cold(Ctx &c, int64_t N, long long *S) {
  using K = Sc<T>;
  T *Cs = reinterpret_cast<T *>(c.Cs);
  T *prow = reinterpret_cast<T *>(c.prow);
  T *Ls = reinterpret_cast<T *>(c.Ls);
  const int64_t r0 = (int64_t)c.rank * c.rpc;
  const int nloc = (int)max((int64_t)0, min((int64_t)c.rpc, N - r0));
  const int q = c.q;
  for (int i = c.tid; i < c.rpc; i += LRA_NT) c.inS[i] = 0;
  __syncthreads();
  for (int t = 0; t < q; ++t) {
    double lm = -1.0;
    for (int i = c.tid; i < nloc; i += LRA_NT)
      if (!c.inS[i]) lm = fmax(lm, K::abs(Cs[(size_t)i * c.qp + t]));
    const double M = cluster_max(c, lm);
    if (!(M > 0.0) || !isfinite(M)) return false;
    const double thr = (1.0 - c.tau) * M;
    long long li = LLONG_MAX;
    for (int i = c.tid; i < nloc; i += LRA_NT)
      if (!c.inS[i] && K::abs(Cs[(size_t)i * c.qp + t]) >= thr) { li = r0 + i; break; }
    const long long p = cluster_min(c, li);
    const int owner = (int)(p / c.rpc), ploc = (int)(p % c.rpc);
    if (c.tid < q) prow[c.tid] = remote_row<T>(c, owner, ploc)[c.tid];
    if (c.tid == 0) {
      S[t] = p;
      if (owner == c.rank) c.inS[ploc] = 1;
    }
    __syncthreads();
    if (c.tid < t) Ls[t * (t - 1) / 2 + c.tid] = prow[c.tid];   // L_S[t, 0..t-1]
    const T piv = prow[t];
    for (int i = c.tid; i < nloc; i += LRA_NT) {
      if (c.inS[i]) continue;
      T *row = Cs + (size_t)i * c.qp;
      const T f = K::div(row[t], piv);
      row[t] = f;                                               // multiplier L[i, t]
      for (int j = t + 1; j < q; ++j) row[j] = K::sub_mul(row[j], f, prow[j]);
    }
    __syncthreads();
  }
  // C_i = l_i L_S^{-1}:  c_j = l_j - sum_{t>j} c_t L_S[t, j],  j = q-1 .. 0
  for (int i = c.tid; i < nloc; i += LRA_NT) {
    if (c.inS[i]) continue;
    T *row = Cs + (size_t)i * c.qp;
    double mx = 0.0;
    for (int j = q - 1; j >= 0; --j) {
      T acc = row[j];
      for (int t = j + 1; t < q; ++t) acc = K::fsub_mul(acc, row[t], Ls[t * (t - 1) / 2 + j]);
      row[j] = acc;
      mx = fmax(mx, K::abs(acc));
    }
    c.rmax[i] = mx;
  }
  __syncthreads();
  return true;
}

// Warm start (real): C = B * G^{-1}, G = B[S,:], by LU of G^T with partial pivoting in
// every CTA (redundantly, identical results) and one forward/back substitution per row.
__device__ bool warm_start(Ctx &c, int64_t N, const long long *S) {
  double *Cs = reinterpret_cast<double *>(c.Cs);
  double *G = c.Ls;                 // q x q, G[a*q + b] = G^T[a][b] = B[S[b]][a]
  const int64_t r0 = (int64_t)c.rank * c.rpc;
  const int nloc = (int)max((int64_t)0, min((int64_t)c.rpc, N - r0));
  const int q = c.q;
  for (int i = c.tid; i < c.rpc; i += LRA_NT) c.inS[i] = 0;
  __syncthreads();
  if (c.tid < q) {
    long long s = S[c.tid];
    if (s / c.rpc == c.rank) c.inS[s % c.rpc] = 1;
  }
  cluster_barrier(c);               // every CTA's block rows are loaded
  for (int e = c.tid; e < q * q; e += LRA_NT) {
    int a = e / q, b = e % q;
    long long s = S[b];
    G[a * q + b] = remote_row<double>(c, (int)(s / c.rpc), (int)(s % c.rpc))[a];
  }
  __syncthreads();
  // LU of G^T (in G) with partial pivoting (first max on ties)
  for (int t = 0; t < q; ++t) {
    if (c.warp == 0) {
      double best = -1.0;
      int bi = t;
      for (int a = t + c.lane; a < q; a += 32) {
        double v = fabs(G[a * q + t]);
        if (v > best) { best = v; bi = a; }
      }
      for (int o = 16; o > 0; o >>= 1) {
        double ov = __shfl_xor_sync(0xffffffffu, best, o);
        int oi = __shfl_xor_sync(0xffffffffu, bi, o);
        if (ov > best || (ov == best && oi < bi)) { best = ov; bi = oi; }
      }
      if (c.lane == 0) {
        c.sh->piv[t] = bi;
        c.sh->sing = !(best > 0.0) || !isfinite(best);
      }
      __syncwarp();
      if (bi != t)
        for (int b = c.lane; b < q; b += 32) {
          double x = G[t * q + b];
          G[t * q + b] = G[bi * q + b];
          G[bi * q + b] = x;
        }
    }
    __syncthreads();
    if (c.sh->sing) return false;
    const double d = G[t * q + t];
    for (int a = t + 1 + c.tid; a < q; a += LRA_NT) G[a * q + t] /= d;
    __syncthreads();
    const int w = q - t - 1;
    for (int e = c.tid; e < w * w; e += LRA_NT) {
      int a = t + 1 + e / w, b = t + 1 + e % w;
      G[a * q + b] = fma(-G[a * q + t], G[t * q + b], G[a * q + b]);
    }
    __syncthreads();
  }
  // rows: solve G^T x = b  (x = C row)
  for (int i = c.tid; i < nloc; i += LRA_NT) {
    if (c.inS[i]) continue;
    double *row = Cs + (size_t)i * c.qp;
    for (int t = 0; t < q; ++t) {
      int p = c.sh->piv[t];
      if (p != t) { double x = row[t]; row[t] = row[p]; row[p] = x; }
    }
    for (int a = 1; a < q; ++a) {
      double acc = row[a];
      for (int t = 0; t < a; ++t) acc = fma(-G[a * q + t], row[t], acc);
      row[a] = acc;
    }
    double mx = 0.0;
    for (int a = q - 1; a >= 0; --a) {
      double acc = row[a];
      for (int t = a + 1; t < q; ++t) acc = fma(-G[a * q + t], row[t], acc);
      acc /= G[a * q + a];
      row[a] = acc;
      mx = fmax(mx, fabs(acc));
    }
    c.rmax[i] = mx;
  }
  __syncthreads();
  return true;
}

// Alg D.1 swap loop with the rank-1 update C <- C - C[:,j*] (C[i*,:] - e_j*^T) / c_{i*j*}.
template <typename T>
__device__ MVOut swap_loop(Ctx &c, int64_t N, long long *S, int cap) {
  using K = Sc<T>;
  T *Cs = reinterpret_cast<T *>(c.Cs);
  T *prow = reinterpret_cast<T *>(c.prow);
  const int64_t r0 = (int64_t)c.rank * c.rpc;
  const int nloc = (int)max((int64_t)0, min((int64_t)c.rpc, N - r0));
  const int q = c.q;
  MVOut o{0, 0, false, 0.0};
  for (;;) {
    double lm = 0.0;
    for (int i = c.tid; i < nloc; i += LRA_NT)
      if (!c.inS[i]) lm = fmax(lm, c.rmax[i]);
    const double M = cluster_max(c, lm);
    if (M <= 1.0 + c.tol || o.swaps >= cap) {
      o.cert = M;
      o.cap_hit = M > 1.0 + c.tol;
      return o;
    }
    const double thr = (1.0 - c.tau) * M;
    long long li = LLONG_MAX;
    for (int i = c.tid; i < nloc && li == LLONG_MAX; i += LRA_NT) {
      if (c.inS[i] || c.rmax[i] < thr) continue;
      const T *row = Cs + (size_t)i * c.qp;
      for (int j = 0; j < q; ++j)
        if (K::abs(row[j]) >= thr) { li = (r0 + i) * (long long)q + j; break; }
    }
    const long long L = cluster_min(c, li);
    const long long istar = L / q;
    const int jstar = (int)(L % q);
    const int owner = (int)(istar / c.rpc);
    if (c.tid < q) prow[c.tid] = remote_row<T>(c, owner, (int)(istar % c.rpc))[c.tid];
    const long long sold = S[jstar];
    __syncthreads();                 // S[jstar] read by all before it changes
    if (c.tid == 0) {
      S[jstar] = istar;
      if (owner == c.rank) c.inS[istar % c.rpc] = 1;
      if (sold / c.rpc == c.rank) {  // the leaving row becomes an explicit row e_{j*}
        int sl = (int)(sold % c.rpc);
        c.inS[sl] = 0;
        T *row = Cs + (size_t)sl * c.qp;
        for (int j = 0; j < q; ++j) row[j] = (j == jstar) ? K::one() : K::zero();
      }
    }
    __syncthreads();
    const T piv = prow[jstar];
    for (int i = c.tid; i < nloc; i += LRA_NT) {
      if (c.inS[i]) continue;
      T *row = Cs + (size_t)i * c.qp;
      const T g = K::div(row[jstar], piv);
      double mx = 0.0;
      for (int j = 0; j < q; ++j) {
        T v = (j == jstar) ? g : K::fsub_mul(row[j], g, prow[j]);
        row[j] = v;
        mx = fmax(mx, K::abs(v));
      }
      c.rmax[i] = mx;
    }
    __syncthreads();
    ++o.swaps;
  }
}

template <typename T>
__device__ bool maxvol_cold(Ctx &c, int64_t N, long long *S, int cap, MVOut &o) {
  if (!lup_cold<T>(c, N, S)) return false;
  o = swap_loop<T>(c, N, S, cap);
  o.lu_steps = c.q;
  return true;
}
__device__ bool maxvol_warm(Ctx &c, int64_t N, long long *S, int cap, MVOut &o) {
  if (!warm_start(c, N, S)) return false;
  o = swap_loop<double>(c, N, S, cap);
  o.lu_steps = 0;
  return true;
}

// ------------------------------------------------------------------ the C-A kernel
__global__ void __launch_bounds__(LRA_NT, 1) k_ca(CAArgs a) {
  extern __shared__ __align__(16) unsigned char dsm[];
  __shared__ CAShared sh;
  Ctx c;
  c.sh = &sh;
  c.cs = a.cs;
  c.rank = (a.cs > 1) ? (int)cg::this_cluster().block_rank() : 0;
  c.rpc = a.rpc;
  c.qp = a.qp;
  c.q = a.q;
  c.tid = threadIdx.x;
  c.lane = threadIdx.x & 31;
  c.warp = threadIdx.x >> 5;
  c.par = 0;
  c.tau = a.tau;
  c.tol = a.tol;
  const size_t esz = a.y_complex ? 16 : 8;
  size_t off = 0;
  c.Cs = dsm + off;
  off += (size_t)a.rpc * a.qp * esz;
  off = (off + 15) & ~(size_t)15;
  c.Ls = reinterpret_cast<double *>(dsm + off);
  size_t lsz = (size_t)a.q * a.q * 8;
  size_t lsz2 = (size_t)a.q * (a.q - 1) / 2 * esz;
  off += lsz > lsz2 ? lsz : lsz2;
  off = (off + 15) & ~(size_t)15;
  c.prow = dsm + off;
  off += (size_t)a.q * 16;
  c.rmax = reinterpret_cast<double *>(dsm + off);
  off += (size_t)a.rpc * 8;
  c.inS = dsm + off;

  const int64_t b = blockIdx.x / a.cs;
  OpView op = a.op;
  if (op.kind == LRA_OP_DENSE)
    op.w = (const char *)op.w + b * a.w_stride * (op.dtype == LRA_F32 ? 4 : 8);
  const int q = a.q;
  int32_t status = LRA_OK;
  int lu = 0, swaps = 0, caps = 0, sk_swaps = 0, loops = 0;
  double cert_r = 0.0, cert_c = 0.0;
  MVOut o;
  bool ok = true;

  // stage 2: I <- maxvol(Y), or the given I0
  if (a.Y) {
    const char *Yb = (const char *)a.Y + b * a.y_stride * esz;
    if (a.y_complex) {
      load_Y<cplx>(c, Yb, a.ldy, op.m);
      ok = maxvol_cold<cplx>(c, op.m, sh.Isl, a.cap, o);
    } else {
      load_Y<double>(c, Yb, a.ldy, op.m);
      ok = maxvol_cold<double>(c, op.m, sh.Isl, a.cap, o);
    }
    if (ok) { lu += o.lu_steps; swaps += o.swaps; caps += o.cap_hit; sk_swaps = o.swaps; }
  } else {
    if (c.tid < q) sh.Isl[c.tid] = a.I0[b * a.i0_stride + c.tid];
    __syncthreads();
  }
  // stage 3: C-A loops
  for (int loop = 0; ok && loop < a.sweeps; ++loop) {
    cluster_barrier(c);              // nobody still reads the previous block
    load_rowsT(c, op, sh.Isl, op.n);
    if (loop == 0) {
      __syncthreads();
      ok = maxvol_cold<double>(c, op.n, sh.Jsl, a.cap, o);
    } else {
      ok = maxvol_warm(c, op.n, sh.Jsl, a.cap, o);
    }
    if (!ok) break;
    const int sw_h = o.swaps;
    lu += o.lu_steps; swaps += o.swaps; caps += o.cap_hit; cert_c = o.cert;
    cluster_barrier(c);
    load_cols(c, op, sh.Jsl, op.m);
    ok = maxvol_warm(c, op.m, sh.Isl, a.cap, o);
    if (!ok) break;
    lu += o.lu_steps; swaps += o.swaps; caps += o.cap_hit; cert_r = o.cert;
    ++loops;
    if (loop > 0 && sw_h == 0 && o.swaps == 0) break;
  }
  if (!ok) status = LRA_ESINGULAR;
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
        a.stats[b] = s;
      }
    }
  }
  cluster_barrier(c);                // keep every CTA's shared memory alive until done
}

size_t ca_smem_bytes(int rpc, int qp, int q, bool cplx) {
  const size_t esz = cplx ? 16 : 8;
  size_t off = (size_t)rpc * qp * esz;
  off = (off + 15) & ~(size_t)15;
  size_t lsz = (size_t)q * q * 8, lsz2 = (size_t)q * (q - 1) / 2 * esz;
  off += lsz > lsz2 ? lsz : lsz2;
  off = (off + 15) & ~(size_t)15;
  off += (size_t)q * 16 + (size_t)rpc * 8 + (size_t)rpc;
  return (off + 15) & ~(size_t)15;
}

// Choose the smallest cluster size whose shared memory holds the block.
cudaError_t launch_ca(CAArgs a, int64_t nb, int64_t maxN, cudaStream_t st, int *cs_out, Prof *pf) {
  const bool cplx = a.y_complex != 0;
  const size_t limit = 227 * 1024 - sizeof(CAShared) - 256;
  int cs = 1;
  int rpc = 0;
  for (cs = 1; cs <= 16; cs *= 2) {
    rpc = (int)((maxN + cs - 1) / cs);
    if (ca_smem_bytes(rpc, a.qp, a.q, cplx) <= limit) break;
  }
  if (cs > 16) return cudaErrorInvalidConfiguration;
  a.cs = cs;
  a.rpc = rpc;
  if (cs_out) *cs_out = cs;
  const size_t smem = ca_smem_bytes(rpc, a.qp, a.q, cplx);
  cudaError_t e = cudaFuncSetAttribute(k_ca, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
  if (e != cudaSuccess) return e;
  if (cs > 8) {
    e = cudaFuncSetAttribute(k_ca, cudaFuncAttributeNonPortableClusterSizeAllowed, 1);
    if (e != cudaSuccess) return e;
  }
  cudaLaunchConfig_t cfg = {};
  cfg.gridDim = dim3((unsigned)(nb * cs));
  cfg.blockDim = dim3(LRA_NT);
  cfg.dynamicSmemBytes = smem;
  cfg.stream = st;
  cudaLaunchAttribute attr[1];
  attr[0].id = cudaLaunchAttributeClusterDimension;
  attr[0].val.clusterDim.x = cs;
  attr[0].val.clusterDim.y = 1;
  attr[0].val.clusterDim.z = 1;
  cfg.attrs = attr;
  cfg.numAttrs = 1;
  pf->begin("k_ca", st);
  e = cudaLaunchKernelEx(&cfg, k_ca, a);
  pf->end(st);
  return e;
}

}  // namespace lra
