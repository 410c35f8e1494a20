// nucleus.cu — canonical nucleus (Alg 3.1 "algcnnncl") and the rank-r
// factors of CUR = A*B.
//
// k_nucleus: one CTA per problem.  G = W[I,J] (k x l) is gathered to shared memory and
// its SVD G = S Sigma T^T computed by one-sided (Hestenes) Jacobi in fp64 with a parallel
// round-robin pair ordering (one warp per column pair).  Then
//   U  = T_r Sigma_r^{-1} S_r^T                (l x k)  -> caller
//   TS = T_r Sigma_r^{-1}  (l x r),  Sr = S_r  (k x r)  -> scratch for the factor kernels
// k_factor_A: A = W[:,J] * TS  (m x r),   k_factor_B: B = Sr^T * W[I,:]  (r x n).
#include "kernels.cuh"

#include <cstdlib>

namespace lra {

__device__ unsigned long long g_nuc_cnt[2];   // diagnostics: Jacobi sweeps, rotations (all problems)   // max threads; launched with 32 x (l/2) so each pair has a warp


__device__ __forceinline__ void rr_pair(int L, int round, int i, int &a, int &b) {
  // circle method on L (even) players: player 0 fixed, 1..L-1 rotate
  if (i == 0) {
    a = 0;
    b = 1 + round % (L - 1);
  } else {
    a = 1 + (round + i) % (L - 1);
    b = 1 + (round - i + (L - 1)) % (L - 1);
  }
}

// KU = ceil(k / 32) (k = the long side).  Each pair gets PL lanes; the loop reproduces the warp-wide dot product bit for bit: lane h holds the partials that
// lanes h, h+8, h+16, h+24 of a full warp held (same element order), adds them in the order of
// the xor-16 and xor-8 butterfly levels, then finishes with xor 4, 2, 1 — the same sums in the
// same association, so every rotation, and the whole SVD, is unchanged while a round issues a
// quarter of the warps (the round was fp64-issue-bound with one warp per pair).
template <int KU, int PL, int KC = 0>
__global__ void __launch_bounds__(512) k_nucleus(NucArgs a) {
  const int NT = blockDim.x, NW = NT >> 5;
  extern __shared__ __align__(16) double nsm[];
  const int64_t b = blockIdx.x;
  if (a.status[b] != LRA_OK) return;
  const int r = a.r;
  // A wide generator (k < l, NEXT-3 rectangular case) is handled through its transpose so
  // that Jacobi always orthogonalises the shorter dimension: H = G^T = S' Sigma V^T gives
  // G = V Sigma S'^T, i.e. S = V and T = S' (columns of the rotated H over sigma).
  const bool tr = KC ? false : a.k < a.l;
  // KC > 0: a square KC x KC generator known at compile time (constant-folded bounds)
  const int k = KC ? KC : (tr ? a.l : a.k), l = KC ? KC : (tr ? a.k : a.l);   // H is k x l, k >= l
  const int L = (l + 1) & ~1;          // even number of columns (zero pad)
  const int ldg = k;                   // H column stride
  double *G = nsm;                     // L columns of length k
  double *V = G + (size_t)L * ldg;     // L x L
  double *sig = V + (size_t)L * L;     // L
  int *ord = reinterpret_cast<int *>(sig + L);
  __shared__ int s_rot[2];   // rotation flag of sweep s in s_rot[s & 1] (double-buffered)
  OpView op = a.op;
  if (op.kind == LRA_OP_DENSE) op.w = (const char *)op.w + b * a.w_stride * (op.dtype == LRA_F32 ? 4 : 8);
  const int64_t *I = a.I + b * a.k, *J = a.J + b * a.l;
  const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
  for (int e = tid; e < L * k; e += NT) {
    int j = e / k, i = e % k;          // H[i, j] = tr ? G[j, i] : G[i, j]
    const int gi = tr ? j : i, gj = tr ? i : j;
    long long ii = 0, jj = 0;
    if (j < l && !a.Gd) {
      ii = I[gi];
      jj = J[gj];
      LRA_CHKIDX(1, b, ii, op.m);
      LRA_CHKIDX(2, b, jj, op.n);
    }
    G[e] = j < l ? (a.Gd ? a.Gd[(size_t)b * k * l + (size_t)gj * a.k + gi] : op.at(ii, jj)) : 0.0;
  }
  for (int e = tid; e < L * L; e += NT) V[e] = (e / L == e % L) ? 1.0 : 0.0;
  __syncthreads();
  // One-sided (Hestenes) Jacobi, Rutishauser's rotation.  Column norms are cached and
  // updated analytically (a_pp' = a_pp - t a_pq, a_qq' = a_qq + t a_pq), refreshed from
  // the data at every sweep, so a pair costs one dot product; the rotation uses
  // reciprocal / rsqrt instead of IEEE divisions and square roots.  Rotate while
  // cos(angle) between two columns exceeds 4·k·eps (the fp64 dot products of already
  // orthogonal columns carry relative errors ~k·eps, so a tighter test never stops).
  // Every fused multiply-add is written out (a*b - c*d = fma(a, b, -(c*d))), so the
  // rounding does not depend on the compiler's contraction choices in each instantiation.
  double *nrm = sig;                   // cached squared column norms (L)
  __shared__ unsigned char s_pair[127 * 64 * 2];  // round-robin schedule (L <= 128)
  for (int e = tid; e < (L - 1) * (L / 2); e += NT) {
    int p, qq;
    rr_pair(L, e / (L / 2), e % (L / 2), p, qq);
    s_pair[2 * e] = (unsigned char)p;
    s_pair[2 * e + 1] = (unsigned char)qq;
  }
  const double eps = 4.0 * (double)k * 2.220446049250313e-16;
  const double eps2 = eps * eps;
  if (tid == 0) s_rot[0] = s_rot[1] = 0;   // ordered before any use by the barrier after the norms
  for (int sweep = 0; sweep < 40; ++sweep) {
    for (int j = warp; j < L; j += NW) {
      double s2 = 0.0;
      for (int i = lane; i < k; i += 32) s2 = fma(G[(size_t)j * ldg + i], G[(size_t)j * ldg + i], s2);
      s2 = warp_sum(s2);
      if (lane == 0) nrm[j] = s2;
    }
    __syncthreads();
    int rot = 0;
    {
    constexpr int GPW = 32 / PL, C = 32 / PL;   // pairs per warp, full-warp lanes per lane
    constexpr int EV = (32 * KU) / PL;            // V elements per lane (L <= 32 KU)
    const int grp = lane / PL, hl = lane % PL;
    const unsigned gmask = 0xffffffffu;
    for (int round = 0; round < L - 1; ++round) {
      for (int base = warp * GPW; base < L / 2; base += NW * GPW) {   // warp-uniform trip count
        const int pi = base + grp;
        const bool act = pi < L / 2;
        int p = 0, qq = 1;
        if (act) {
          p = s_pair[2 * (round * (L / 2) + pi)];
          qq = s_pair[2 * (round * (L / 2) + pi) + 1];
        }
        double *gp = G + (size_t)p * ldg, *gq = G + (size_t)qq * ldg;
        double *vp = V + (size_t)p * L, *vq = V + (size_t)qq * L;
        double xs[C][KU], ys[C][KU], vx[EV], vy[EV], v[C];
#pragma unroll
        for (int c = 0; c < C; ++c) {            // full-warp lane l = hl + PL c
#pragma unroll
          for (int u = 0; u < KU; ++u) {
            const int i = hl + PL * c + 32 * u;
            xs[c][u] = i < k ? gp[i] : 0.0;
            ys[c][u] = i < k ? gq[i] : 0.0;
          }
        }
#pragma unroll
        for (int e = 0; e < EV; ++e) {           // independent of the rotation: load early
          const int i = hl + PL * e;
          vx[e] = i < L ? vp[i] : 0.0;
          vy[e] = i < L ? vq[i] : 0.0;
        }
        const double al = nrm[p], be = nrm[qq];
#pragma unroll
        for (int c = 0; c < C; ++c) {
          double acc = 0.0;
#pragma unroll
          for (int u = 0; u < KU; ++u) acc = fma(xs[c][u], ys[c][u], acc);
          v[c] = acc;
        }
#pragma unroll
        for (int o = 16; o >= PL; o >>= 1) {     // butterfly levels held inside the lane
          const int d = o / PL;
#pragma unroll
          for (int c = 0; c < C; ++c)
            if ((c & d) == 0 && c + d < C) v[c] = v[c] + v[c + d];
        }
        double ga = v[0];
#pragma unroll
        for (int o = PL / 2; o > 0; o >>= 1) ga += __shfl_xor_sync(gmask, ga, o);
        if (act && ga * ga > eps2 * al * be && ga != 0.0) {
          const double zeta = (be - al) * (0.5 * __drcp_rn(ga));
          const double z2 = fma(zeta, zeta, 1.0);
          // t = sign(zeta) / (|zeta| + sqrt(1 + zeta^2)), sqrt(1 + zeta^2) = z2 * rsqrt(z2) fused;
          // t -> 1 / (2 zeta) once zeta^2 overflows, t = 0 for a non-finite zeta (degenerate pairs:
          // a column at rounding level, ga below the reciprocal's range)
          const double t = z2 < INFINITY ? copysign(__drcp_rn(fma(z2, rsqrt(z2), fabs(zeta))), zeta)
                                         : (isfinite(zeta) ? 0.5 / zeta : 0.0);
          const double cs = rsqrt(fma(t, t, 1.0)), sn = cs * t;
#pragma unroll
          for (int c = 0; c < C; ++c) {
#pragma unroll
            for (int u = 0; u < KU; ++u) {
              const int i = hl + PL * c + 32 * u;
              if (i < k) {
                gp[i] = fma(cs, xs[c][u], -__dmul_rn(sn, ys[c][u]));
                gq[i] = fma(sn, xs[c][u], __dmul_rn(cs, ys[c][u]));
              }
            }
          }
#pragma unroll
          for (int e = 0; e < EV; ++e) {
            const int i = hl + PL * e;
            if (i < L) {
              vp[i] = fma(cs, vx[e], -__dmul_rn(sn, vy[e]));
              vq[i] = fma(sn, vx[e], __dmul_rn(cs, vy[e]));
            }
          }
          if (hl == 0) {
            nrm[p] = fma(-t, ga, al);
            nrm[qq] = fma(t, ga, be);
          }
          rot = 1;
        }
      }
      __syncthreads();
    }
    }
    if (rot && lane == 0) atomicOr(&s_rot[sweep & 1], 1);
    __syncthreads();
    // Every thread reads this sweep's flag; the NEXT sweep's flag is cleared here, after the
    // barrier that ends this sweep (all of its readers, in the previous sweep, are past it).
    // (Round 1 reset a single flag at the top of the sweep: a fast warp could clear it before a
    // slow warp had read it, the slow warp left the loop alone and the CTA desynchronised —
    // caught by cuda-gdb as an out-of-range shared-memory address in the TS write under
    // concurrent batch groups.)
    const int any = s_rot[sweep & 1];
    if (tid == 0) {
      s_rot[(sweep + 1) & 1] = 0;
      atomicAdd(&g_nuc_cnt[0], 1ull);
    }
    if (!any) break;
  }
  // singular values, descending order (ties: lower column first)
  for (int j = warp; j < L; j += NW) {
    double s = 0.0;
    for (int i = lane; i < k; i += 32) s = fma(G[(size_t)j * ldg + i], G[(size_t)j * ldg + i], s);
    s = warp_sum(s);
    if (lane == 0) sig[j] = sqrt(s);
  }
  __syncthreads();
  if (tid == 0) {
    for (int j = 0; j < L; ++j) ord[j] = j;
    for (int x = 1; x < L; ++x) {   // insertion sort, stable
      int v = ord[x];
      int y = x - 1;
      while (y >= 0 && sig[ord[y]] < sig[v]) { ord[y + 1] = ord[y]; --y; }
      ord[y + 1] = v;
    }
    if (!(sig[ord[r - 1]] > 0.0) || !isfinite(sig[ord[0]])) a.status[b] = LRA_ESINGULAR;
    if (a.stats && a.k == a.l) {   // log|det G| = sum of log sigma_i over the whole generator
      double lv = 0.0;
      for (int j = 0; j < l; ++j) lv += log(sig[j]);   // the l real columns (not the pad)
      a.stats[b].logvol_final = lv;
    }
  }
  __syncthreads();
  if (a.status[b] != LRA_OK) return;
  const int gk = a.k, gl = a.l;        // G's own shape
  double *TS = a.TS + b * (int64_t)gl * r, *Sr = a.Sr + b * (int64_t)gk * r;
  for (int e = tid; e < gl * r; e += NT) {     // TS[j, t] = T[j, ord t] / sigma
    int t = e / gl, j = e % gl;
    int c = ord[t];
    TS[(size_t)t * gl + j] = tr ? G[(size_t)c * ldg + j] / (sig[c] * sig[c]) : V[(size_t)c * L + j] / sig[c];
  }
  for (int e = tid; e < gk * r; e += NT) {     // Sr[i, t] = S[i, ord t]
    int t = e / gk, i = e % gk;
    int c = ord[t];
    Sr[(size_t)t * gk + i] = tr ? V[(size_t)c * L + i] : G[(size_t)c * ldg + i] / sig[c];
  }
  __syncthreads();
  if (a.U) {
    double *U = a.U + b * (int64_t)gl * gk;
    for (int e = tid; e < gl * gk; e += NT) {  // U (l x k, col-major) = TS * Sr^T
      int col = e / gl, row = e % gl;
      double s = 0.0;
      for (int t = 0; t < r; ++t) s = fma(TS[(size_t)t * gl + row], Sr[(size_t)t * gk + col], s);
      U[(size_t)col * gl + row] = s;
    }
  }
}

// the generator sizes whose H and V fit in shared memory next to the static pair schedule
bool nucleus_fits(int k, int l) { return nucleus_smem(k, l) + 127 * 64 * 2 + 64 <= 227 * 1024; }

size_t nucleus_smem(int k, int l) {
  if (k < l) { int t = k; k = l; l = t; }     // transposed wide case
  int L = (l + 1) & ~1;
  return ((size_t)L * k + (size_t)L * L + L) * 8 + (size_t)L * 4 + 16;
}

// ---------------------------------------------------------------------- factors

// A = W[:,J] * TS: one thread per row of A computes all r outputs (accumulated in ascending j,
// as before), the l gathered values W[i, J[j]] loaded 16 at a time (coalesced across rows).
// grid (ceil(m/128), nb), 128 threads.  r <= 64 (registers: r doubles per thread).
// The coefficient matrix (TS for A, Sr for B) sits in shared memory transposed, c[j][u]
// (RMAX columns, zero beyond r), so one 16-byte load feeds two outputs; each thread owns RR
// rows of A (columns of B) that share those loads.  Every output is the same fma chain over
// j (s) ascending as before, so A and B are bit-identical to the one-row version.
template <int RMAX, int RR>
__global__ void __launch_bounds__(128) k_factor_A(FacArgs a) {
  extern __shared__ __align__(16) double ts[];   // l x RMAX: ts[j * RMAX + u]
  const int64_t b = blockIdx.y;
  if (a.status[b] != LRA_OK) return;
  OpView op = a.op;
  if (op.kind == LRA_OP_DENSE) op.w = (const char *)op.w + b * a.w_stride * (op.dtype == LRA_F32 ? 4 : 8);
  const int l = a.l, r = a.r;
  const double *TS = a.TS + b * (int64_t)l * r;
  for (int e = threadIdx.x; e < l * RMAX; e += 128) {
    const int j = e / RMAX, u = e % RMAX;
    ts[e] = u < r ? TS[u * l + j] : 0.0;
  }
  __syncthreads();
  const int64_t i0 = (int64_t)blockIdx.x * (128 * RR) + threadIdx.x;
  if (i0 >= op.m) return;
  const int64_t *J = a.J + b * l;
  double acc[RR][RMAX];
#pragma unroll
  for (int x = 0; x < RR; ++x)
#pragma unroll
    for (int u = 0; u < RMAX; ++u) acc[x][u] = 0.0;
  constexpr int PF = 8;
  for (int j0 = 0; j0 < l; j0 += PF) {
    double w[RR][PF];
#pragma unroll
    for (int x = 0; x < RR; ++x)
#pragma unroll
      for (int y = 0; y < PF; ++y) {
        const int64_t i = i0 + 128 * x;
        long long jj = (j0 + y < l && i < op.m) ? J[j0 + y] : 0;
        LRA_CHKIDX(3, b, jj, op.n);
        w[x][y] = (j0 + y < l && i < op.m) ? op.at(i, jj) : 0.0;
      }
#pragma unroll
    for (int y = 0; y < PF; ++y) {
      if (j0 + y < l) {
        const double2 *c2 = reinterpret_cast<const double2 *>(ts + (j0 + y) * RMAX);
#pragma unroll
        for (int u2 = 0; u2 < RMAX / 2; ++u2) {
          const double2 c = c2[u2];
#pragma unroll
          for (int x = 0; x < RR; ++x) {
            acc[x][2 * u2] = fma(w[x][y], c.x, acc[x][2 * u2]);
            acc[x][2 * u2 + 1] = fma(w[x][y], c.y, acc[x][2 * u2 + 1]);
          }
        }
      }
    }
  }
  double *A = a.A + b * a.a_stride;
#pragma unroll
  for (int x = 0; x < RR; ++x) {
    const int64_t i = i0 + 128 * x;
    if (i < op.m)
#pragma unroll
      for (int u = 0; u < RMAX; ++u)
        if (u < r) A[(int64_t)u * op.m + i] = acc[x][u];
  }
}

// B = Sr^T * W[I,:]: thread = RR columns of B (all r outputs, ascending s).
template <int RMAX, int RR>
__global__ void __launch_bounds__(128) k_factor_B(FacArgs a) {
  extern __shared__ __align__(16) double sr[];   // k x RMAX: sr[s * RMAX + u]
  const int64_t b = blockIdx.y;
  if (a.status[b] != LRA_OK) return;
  OpView op = a.op;
  if (op.kind == LRA_OP_DENSE) op.w = (const char *)op.w + b * a.w_stride * (op.dtype == LRA_F32 ? 4 : 8);
  const int k = a.k, r = a.r;
  const double *Sr = a.Sr + b * (int64_t)k * r;
  for (int e = threadIdx.x; e < k * RMAX; e += 128) {
    const int s = e / RMAX, u = e % RMAX;
    sr[e] = u < r ? Sr[u * k + s] : 0.0;
  }
  __syncthreads();
  const int64_t j0c = (int64_t)blockIdx.x * (128 * RR) + threadIdx.x;
  if (j0c >= op.n) return;
  const int64_t *I = a.I + b * k;
  double acc[RR][RMAX];
#pragma unroll
  for (int x = 0; x < RR; ++x)
#pragma unroll
    for (int u = 0; u < RMAX; ++u) acc[x][u] = 0.0;
  constexpr int PF = 8;
  for (int s0 = 0; s0 < k; s0 += PF) {
    double w[RR][PF];
#pragma unroll
    for (int x = 0; x < RR; ++x)
#pragma unroll
      for (int y = 0; y < PF; ++y) {
        const int s = s0 + y;
        const int64_t j = j0c + 128 * x;
        long long ii = (s < k && j < op.n && !a.Rt) ? I[s] : 0;
        LRA_CHKIDX(4, b, ii, op.m);
        w[x][y] = (s < k && j < op.n) ? (a.Rt ? a.Rt[(int64_t)s * op.n + j] : op.at(ii, j)) : 0.0;
      }
#pragma unroll
    for (int y = 0; y < PF; ++y) {
      if (s0 + y < k) {
        const double2 *c2 = reinterpret_cast<const double2 *>(sr + (s0 + y) * RMAX);
#pragma unroll
        for (int u2 = 0; u2 < RMAX / 2; ++u2) {
          const double2 c = c2[u2];
#pragma unroll
          for (int x = 0; x < RR; ++x) {
            acc[x][2 * u2] = fma(c.x, w[x][y], acc[x][2 * u2]);
            acc[x][2 * u2 + 1] = fma(c.y, w[x][y], acc[x][2 * u2 + 1]);
          }
        }
      }
    }
  }
  double *B = a.B + b * a.b_stride;
#pragma unroll
  for (int x = 0; x < RR; ++x) {
    const int64_t j = j0c + 128 * x;
    if (j < op.n)
#pragma unroll
      for (int u = 0; u < RMAX; ++u)
        if (u < r) B[j * r + u] = acc[x][u];
  }
}

cudaError_t launch_nucleus(const NucArgs &na, const FacArgs &fa, int64_t nb, cudaStream_t st, int *nlaunch, Prof *pf) {
  const size_t smem = nucleus_smem(na.k, na.l);
  static const int pl_env = getenv("LRA_NUC_PL") ? atoi(getenv("LRA_NUC_PL")) : 0;
  const int kl = na.k > na.l ? na.k : na.l, ku = (kl + 31) / 32;
  // lanes per pair (measured on B200: 16 fastest for k <= 64 and k > 96, 32 for 64 < k <= 96)
  const int PLs = pl_env == 8 || pl_env == 16 || pl_env == 32 ? pl_env : (ku == 3 ? 32 : 16);
  using KF = void (*)(NucArgs);
  static const KF tab[3][4] = {
      {k_nucleus<1, 8>, k_nucleus<2, 8>, k_nucleus<3, 8>, k_nucleus<4, 8>},
      {k_nucleus<1, 16>, k_nucleus<2, 16>, k_nucleus<3, 16>, k_nucleus<4, 16>},
      {k_nucleus<1, 32>, k_nucleus<2, 32>, k_nucleus<3, 32>, k_nucleus<4, 32>}};
  const int row = PLs == 8 ? 0 : PLs == 16 ? 1 : 2;
  KF kern = tab[row][ku - 1];
  int PLk = PLs;
  if (pl_env == 0 && na.k == na.l) {   // square shapes of the BASELINE configs (bounds fold)
    if (na.k == 48) {
      kern = k_nucleus<2, 16, 48>;
    } else if (na.k == 20) {
      kern = k_nucleus<1, 16, 20>;
    } else if (na.k == 8) {
      kern = k_nucleus<1, 16, 8>;
    } else if (na.k == 96) {
      kern = k_nucleus<3, 32, 96>;
      PLk = 32;
    }
  }
  cudaError_t e = cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
  if (e != cudaSuccess) return e;
  pf->begin("k_nucleus", st);
  const int L = ((na.k < na.l ? na.k : na.l) + 1) & ~1;
  const int gpw = 32 / PLk;                 // pairs per warp
  int nt = ((L / 2 + gpw - 1) / gpw) * 32;
  if (nt < 256) nt = 256;
  if (nt > 512) nt = 512;                   // the pair loop strides over the rest
  kern<<<(unsigned)nb, nt, smem, st>>>(na);
  pf->end(st);
  if ((e = cudaGetLastError()) != cudaSuccess) return e;
  if (!fa.A && !fa.B) {           // nucleus only (TS, Sr for the caller)
    *nlaunch += 1;
    return cudaSuccess;
  }
  static const int rr_env = getenv("LRA_FAC_RR") ? atoi(getenv("LRA_FAC_RR")) : 1;   // diagnostics
  const int RM = fa.r <= 16 ? 16 : (fa.r <= 32 ? 32 : 64), RRf = (RM <= 32 && rr_env == 2) ? 2 : 1;
  dim3 gA((unsigned)((fa.op.m + 128 * RRf - 1) / (128 * RRf)), (unsigned)nb);
  const size_t sA = (size_t)fa.l * RM * 8, sB = (size_t)fa.k * RM * 8;
  void (*kA)(FacArgs) = RM == 16 ? (RRf == 2 ? k_factor_A<16, 2> : k_factor_A<16, 1>)
                        : (RM == 32 ? (RRf == 2 ? k_factor_A<32, 2> : k_factor_A<32, 1>) : k_factor_A<64, 1>);
  void (*kB)(FacArgs) = RM == 16 ? (RRf == 2 ? k_factor_B<16, 2> : k_factor_B<16, 1>)
                        : (RM == 32 ? (RRf == 2 ? k_factor_B<32, 2> : k_factor_B<32, 1>) : k_factor_B<64, 1>);
  if ((e = cudaFuncSetAttribute(kA, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)sA)) != cudaSuccess) return e;
  if ((e = cudaFuncSetAttribute(kB, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)sB)) != cudaSuccess) return e;
  pf->begin("k_factor_A", st);
  kA<<<gA, 128, sA, st>>>(fa);
  pf->end(st);
  if ((e = cudaGetLastError()) != cudaSuccess) return e;
  dim3 gB((unsigned)((fa.op.n + 128 * RRf - 1) / (128 * RRf)), (unsigned)nb);
  pf->begin("k_factor_B", st);
  kB<<<gB, 128, sB, st>>>(fa);
  pf->end(st);
  *nlaunch += 3;
  return cudaGetLastError();
}

cudaError_t read_idx_err_nuc(long long *out, bool reset) {
  cudaError_t e = cudaMemcpyFromSymbol(out, g_idx_err, sizeof(g_idx_err));
  if (e == cudaSuccess && reset) {
    long long z[4] = {0, 0, 0, 0};
    e = cudaMemcpyToSymbol(g_idx_err, z, sizeof(z));
  }
  return e;
}

cudaError_t read_nuc_counters(unsigned long long *out, bool reset) {
  cudaError_t e = cudaMemcpyFromSymbol(out, g_nuc_cnt, sizeof(g_nuc_cnt));
  if (e == cudaSuccess && reset) {
    unsigned long long z[2] = {0, 0};
    e = cudaMemcpyToSymbol(g_nuc_cnt, z, sizeof(z));
  }
  return e;
}

}  // namespace lra
