// sketch_tc.cu — the dense Gaussian (and quasi-Gaussian) sketch Y = W * Omega of Alg 10.2
// stage 1 ("Compute m x lbar matrix W H-bar") on the tcgen05 tensor cores, as an
// int8 digit-slice (Ozaki-style) contraction, reading C36.
//
// Scaling.  Row i of W gets the exponent e_i with max_j |W_ij| < 2^e_i * 127/128 (a prologue
// pass over W: k_stc_rowmax), column t of Omega the exponent f_t likewise.  The integers
//   X_ij = rn(W_ij 2^(55 - e_i)),   Z_jt = rn(Omega_jt 2^(55 - f_t))      (|X|, |Z| < 2^55 127/128)
// are written in balanced base 256 with seven digits, most significant first:
//   X = sum_s D_s 256^(6-s),  Z = sum_u E_u 256^(6-u),  D_s, E_u in [-128, 127]
// (the bytes of X + 0x80..80 minus 128 each: one 64-bit add gives all seven digits).  Then
//   Y_it = 2^(e_i + f_t - 110) sum_{s,u} 256^(12-s-u) sum_j D_s E_u
// and the levels L = s + u <= 6 are kept (28 of the 49 digit products; the dropped levels weigh
// <= 2^-48 of max|W_i| max|Omega_t| per term and are zero-mean).  The per-level sums P_L are
// exact int32 tensor-core accumulations (|P_L| <= 7 * 255 * 128 * K < 2^31 for K <= 8192 per
// accumulation; longer ranges are drained in chunks of 256 K-steps), combined exactly in int64:
//   hi = sum_{L<=3} P_L 2^(8(3-L)),  lo = sum_{L>=4} P_L 2^(8(6-L)),
//   Y_it = 2^(e_i + f_t - 62) ((double)hi 2^24 + (double)lo).
//
// The digits of 4 values come out of one 64-bit add each, a 4x7 byte transpose (15 PRMT) and
// an XOR 0x80 per byte (the bytes of X + 0x80..80 are D_s + 128).
//
// k_sketch_tc (persistent, one CTA per SM, stream-K over (problem, 128-row tile, 48-column
// tile) x 32-wide K-steps; every CTA gets a contiguous range of K-steps):
//   1 producer warp: lane 0 streams the W tiles (TMA boxes of 128 rows x 32 columns into a ring
//     of shared-memory stages; the Q parts of one K range run side by side over all row tiles, so
//     a column's 128-row pieces are fetched together), lane 1 Omega's pre-digitized slices;
//   8 digitizer warps (warp w: TMEM lane quadrant w % 4, K-step half w / 4): each thread owns one
//     row and converts 16 values per K-step to digits (2 FMUL + F2I + one 64-bit add + a byte
//     transpose by PRMT) written into a TMEM A region (tcgen05.st, 3 regions in flight);
//   3 MMA warps (one elected lane each; levels split 9/9/10 MMAs per K-step so that no two
//     warps write one accumulator): tcgen05.mma kind::i8 TS (A from TMEM, Omega's slice from
//     shared memory), M = 128, N = NP (16/32/48), K = 32, into 7 level accumulators in TMEM;
//   the digitizer warps also drain the accumulators at the end of each range segment (TMEM ->
//     int64 recombination -> Y), and tiles split between CTAs are finished by the last CTA to
//     arrive (exact int64 sums of the partials: deterministic).
#include "kernels.cuh"
#include "tc.cuh"

#include <cuda.h>
#include <cudaTypedefs.h>

#include <algorithm>
#include <cstring>
#include <mutex>

namespace lra {
// phase counters (STC_PROF builds, tools/stc_prof.cu): clock64 cycles summed over CTAs
//  0 dig wait W, 1 dig wait A-empty, 2 dig compute+store, 3 MMA wait A, 4 MMA wait B, 5 MMA issue,
//  6 prod wait W-empty, 7 prod wait B-empty, 8 epi wait acc, 9 epi work, 10 K-steps (count)
__device__ unsigned long long g_stc_cyc[16];
__device__ unsigned long long g_stc_t[1024][4];   // STC_PROF: per CTA globaltimer at entry / ready / loops done / exit
#ifndef STC_PROF
#define STC_PROF 0
#endif
#define STC_CLK() (STC_PROF ? clock64() : 0ll)
#ifndef STC_NWS32
#define STC_NWS32 8      // W stages for fp32 W
#endif
#ifndef STC_NBS
#define STC_NBS 4        // Omega stages
#endif
#ifndef STC_SPIN
#define STC_SPIN 1       // handshake waits without a suspend hint
#endif
#ifndef STC_NO_DIG
#define STC_NO_DIG 0     // diagnostics (tools/stc_prof.cu): skip the digit conversion
#endif
#ifndef STC_NO_MMA
#define STC_NO_MMA 0     // diagnostics: skip the MMAs (commits only)
#endif
#define STC_ADD(k, v)                                            \
  do {                                                          \
    if (STC_PROF) atomicAdd(&g_stc_cyc[k], (unsigned long long)(v)); \
  } while (0)
namespace stc {

#define WAIT(a, p) (STC_SPIN ? tc::mbar_wait_spin(a, p) : tc::mbar_wait(a, p))

constexpr int BM = 128;           // rows per tile (MMA M)
constexpr int BK = 32;            // K per MMA / per K-step
constexpr int S = 7;              // digit slices per operand
constexpr int NLEV = 7;           // kept levels L = s + u <= 6
constexpr int NDW = 8;            // digitizer / epilogue warps
constexpr int NMW = 3;            // MMA warps (12 warps in all: 168 registers per thread)
constexpr int NTHR = 32 * (NDW + NMW + 1);
constexpr int NBS = STC_NBS;        // Omega stages
template <typename TW> constexpr int nws() { return sizeof(TW) == 4 ? STC_NWS32 : 4; }   // W stages (TMA boxes 128 x 32)
constexpr int SLOT = 2 * 48 * BM;  // int64 entries of one (hi, lo) tile buffer
constexpr int KCHUNK = 256;       // max K-steps per accumulation (int32 safety)

struct Args {
  const void *w;
  int64_t ldw, w_stride;
  int64_t m, n, lbar, nb;
  double *y;
  int64_t ldy, y_stride;
  const unsigned long long *rowmax;   // per (problem, row): max |W_ij| bits (fp32 bits zero-extended / fp64 bits)
  const signed char *od;              // Omega digits [NTN][KS][S][NP * 32] (canonical K-major tiles)
  const int *fexp;                    // [NTN * NP] column exponents
  long long *tacc;                    // [P][2][48][128] split-tile accumulators (zero between launches)
  int *cnt;                           // [P] arrivals per split tile (zero between launches)
  long long *own;                     // [P][2][48][128] a CTA's running sum over the chunks of one segment
  int64_t KS, MT, NTN, T;
  int Q;                              // K parts per tile (grid = T Q CTAs, one per SM)
};

// work unit of CTA c: tile c % T, K-steps [q KS / Q, (q + 1) KS / Q) with q = c / T (the Q parts of
// one K range run side by side over all tiles, so the row tiles of a column are read together)
__device__ __forceinline__ int64_t unit_lo(const Args &a, int c) {
  const int64_t tile = c % a.T, q = c / a.T;
  return tile * a.KS + q * a.KS / a.Q;
}
__device__ __forceinline__ int64_t unit_hi(const Args &a, int c) {
  const int64_t tile = c % a.T, q = c / a.T;
  return tile * a.KS + (q + 1) * a.KS / a.Q;
}

// levels of MMA warp mw: {6, 1}, {5, 2}, {4, 3, 0}: 9 / 9 / 10 MMAs per K-step (one issuing
// thread needs ~54 cycles per MMA, so three issue 28 MMAs within the ~672-cycle math time).
// Every offset is a compile-time constant (the issue loop is the MMA warps' critical path).
template <int NP, int L>
__device__ __forceinline__ void issue_level(uint32_t tmem, uint32_t at, uint64_t bd, uint32_t first) {
  constexpr uint32_t IDESC = tc::idesc_i8(BM, NP, true, true);
#pragma unroll
  for (int s = 0; s <= L; ++s)
    tc::mma_i8_ts(tmem + (uint32_t)(L * NP), at + (uint32_t)(s * 8), bd + (uint64_t)(((L - s) * NP * BK) >> 4), IDESC,
                  (s == 0 && first) ? 0u : 1u);
}
template <int NP, int MW>
__device__ __forceinline__ void issue_kstep(uint32_t tmem, uint32_t at, uint64_t bd, uint32_t first) {
  issue_level<NP, 6 - MW>(tmem, at, bd, first);
  issue_level<NP, 1 + MW>(tmem, at, bd, first);
  if (MW == 2) issue_level<NP, 0>(tmem, at, bd, first);
}

template <typename TW>
__device__ __forceinline__ int row_exp(unsigned long long bits) {
  double mx;
  if (sizeof(TW) == 4) mx = (double)__uint_as_float((unsigned)bits);
  else mx = __longlong_as_double((long long)bits);
  if (!(mx > 0.0)) return 0;
  int e = ilogb(mx) + 1;                                // 2^(e-1) <= mx < 2^e
  if (mx >= ldexp(127.0 / 128.0, e)) ++e;
  return e;
}

// 7 balanced digits of 4 values -> 7 words of signed bytes (slice s: byte 6 - s of X + 0x80..80,
// minus 128, i.e. XOR 0x80)
__device__ __forceinline__ void pack4(const long long (&X)[4], uint32_t (&w)[S]) {
  uint32_t lo[4], hi[4];
#pragma unroll
  for (int e = 0; e < 4; ++e) {
    const unsigned long long B = (unsigned long long)X[e] + 0x0080808080808080ull;
    lo[e] = (uint32_t)B;
    hi[e] = (uint32_t)(B >> 32);
  }
  const uint32_t p01 = __byte_perm(lo[0], lo[1], 0x5140), p01h = __byte_perm(lo[0], lo[1], 0x7362);
  const uint32_t p23 = __byte_perm(lo[2], lo[3], 0x5140), p23h = __byte_perm(lo[2], lo[3], 0x7362);
  w[6] = __byte_perm(p01, p23, 0x5410);
  w[5] = __byte_perm(p01, p23, 0x7632);
  w[4] = __byte_perm(p01h, p23h, 0x5410);
  w[3] = __byte_perm(p01h, p23h, 0x7632);
  const uint32_t q01 = __byte_perm(hi[0], hi[1], 0x5140), q01h = __byte_perm(hi[0], hi[1], 0x7362);
  const uint32_t q23 = __byte_perm(hi[2], hi[3], 0x5140), q23h = __byte_perm(hi[2], hi[3], 0x7362);
  w[2] = __byte_perm(q01, q23, 0x5410);
  w[1] = __byte_perm(q01, q23, 0x7632);
  w[0] = __byte_perm(q01h, q23h, 0x5410);
#pragma unroll
  for (int k = 0; k < S; ++k) w[k] ^= 0x80808080u;
}

// X = rn(w 2^sh): fp32 by two exact power-of-two FMULs (2^sh = s1 s2, each a normal fp32) and
// F2I.S64; fp64 by one DMUL and F2I.S64.F64
__device__ __forceinline__ long long to_fixed(float w, float s1, float s2, double) { return __float2ll_rn((w * s1) * s2); }
__device__ __forceinline__ long long to_fixed(double w, float, float, double sd) { return __double2ll_rn(w * sd); }

// ---------------------------------------------------------------- prologue: row maxima of |W|
// Thread = 4 consecutive rows (one 16-byte load per column when ldw and W are 16-byte aligned),
// CTA = 1024 rows x a range of columns (4 KB contiguous per column: the HBM-friendly pattern),
// 16 columns in flight; the maxima are order-free (integer max of the |w| bit patterns).
template <typename TW>
__device__ __forceinline__ unsigned long long absbits(TW v) {
  if (sizeof(TW) == 4) return __float_as_uint(fabsf((float)v));
  return (unsigned long long)__double_as_longlong(fabs((double)v));
}
template <typename TW>
__device__ __forceinline__ void stc_rowmax(const TW *W, int64_t ldw, int64_t w_stride, int64_t m, int64_t n,
                                           int64_t cols_per, unsigned long long *rowmax, int64_t bx, int64_t by,
                                           int64_t b) {
  const int64_t i0 = (bx * 256 + threadIdx.x) * 4;
  if (i0 >= m) return;
  const TW *p = W + b * w_stride + i0;
  const int64_t j0 = by * cols_per, j1 = min(n, j0 + cols_per);
  unsigned long long mx[4] = {0, 0, 0, 0};
  const bool vec = i0 + 4 <= m && (ldw & 3) == 0 && (reinterpret_cast<uintptr_t>(W + b * w_stride) & 15) == 0;
  if (vec) {
    int64_t j = j0;
    constexpr int U = sizeof(TW) == 4 ? 16 : 8;           // 256 B per thread in flight
    for (; j + U <= j1; j += U) {
      TW v[U][4];
#pragma unroll
      for (int u = 0; u < U; ++u) {
        const TW *q = p + (j + u) * ldw;
        if (sizeof(TW) == 4) {
          const float4 f = __ldcg(reinterpret_cast<const float4 *>(q));
          v[u][0] = f.x; v[u][1] = f.y; v[u][2] = f.z; v[u][3] = f.w;
        } else {
          const double2 d0 = __ldcg(reinterpret_cast<const double2 *>(q));
          const double2 d1 = __ldcg(reinterpret_cast<const double2 *>(q) + 1);
          v[u][0] = d0.x; v[u][1] = d0.y; v[u][2] = d1.x; v[u][3] = d1.y;
        }
      }
#pragma unroll
      for (int u = 0; u < U; ++u)
#pragma unroll
        for (int r = 0; r < 4; ++r) {
          const unsigned long long x = absbits<TW>(v[u][r]);
          mx[r] = x > mx[r] ? x : mx[r];
        }
    }
    for (; j < j1; ++j)
#pragma unroll
      for (int r = 0; r < 4; ++r) {
        const unsigned long long x = absbits<TW>(__ldcg(p + j * ldw + r));
        mx[r] = x > mx[r] ? x : mx[r];
      }
  } else {
    for (int64_t j = j0; j < j1; ++j)
      for (int r = 0; r < 4 && i0 + r < m; ++r) {
        const unsigned long long x = absbits<TW>(__ldcg(p + j * ldw + r));
        mx[r] = x > mx[r] ? x : mx[r];
      }
  }
#pragma unroll
  for (int r = 0; r < 4; ++r)
    if (mx[r] && i0 + r < m) atomicMax(rowmax + b * m + i0 + r, mx[r]);
}

// ---------------------------------------------------------------- prologue: Omega's digits
// CTA = (padded column (nt, t), 8 K-steps): the column exponent f_t (the column max, read by
// every CTA of the column from L2), then the 7 balanced digits of its 256 entries into the
// canonical B tiles [nt][ks][slice][t, k] (zero beyond n and lbar).
template <int NP>
__device__ __forceinline__ void stc_omega(const double *omega, int64_t ldo, int64_t n, int64_t lbar, int64_t KS,
                                          signed char *od, int *fexp, int64_t bx, int64_t by) {
  const int nt = (int)(bx / NP), t = (int)(bx % NP);
  const int64_t c = (int64_t)nt * NP + t;                    // column of Omega (padding beyond lbar)
  const bool live = c < lbar;
  const double *col = omega + c * ldo;
  __shared__ double red[8];
  double mx = 0.0;
  if (live)
    for (int64_t j = threadIdx.x; j < n; j += 256) mx = fmax(mx, fabs(__ldg(col + j)));
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) mx = fmax(mx, __shfl_xor_sync(0xffffffffu, mx, o));
  if ((threadIdx.x & 31) == 0) red[threadIdx.x >> 5] = mx;
  __syncthreads();
  mx = 0.0;
  for (int w = 0; w < 8; ++w) mx = fmax(mx, red[w]);
  int f = 0;
  if (mx > 0.0) {
    f = ilogb(mx) + 1;
    if (mx >= ldexp(127.0 / 128.0, f)) ++f;
  }
  if (threadIdx.x == 0 && by == 0) fexp[c] = f;
  const double sc = ldexp(1.0, 55 - f);
  const int64_t j = by * 8 * BK + threadIdx.x;
  if (j >= KS * BK) return;
  const double v = (live && j < n) ? __ldg(col + j) : 0.0;
  const unsigned long long B = (unsigned long long)__double2ll_rn(v * sc) + 0x0080808080808080ull;
  signed char *tile = od + ((size_t)nt * KS + j / BK) * S * (NP * BK) + tc::canon_off(t, (int)(j % BK));
#pragma unroll
  for (int s = 0; s < S; ++s) tile[(size_t)s * (NP * BK)] = (signed char)((int)((B >> (8 * (6 - s))) & 0xffu) - 128);
}

// ---------------------------------------------------------------- the prologue in one launch
// blocks [0, R): row maxima (R = RB x CS x nb), blocks [R, R + O): Omega digits (O = NTN NP x KSB)
template <typename TW, int NP>
__global__ void __launch_bounds__(256) k_stc_prep(const TW *W, int64_t ldw, int64_t w_stride, int64_t m, int64_t n,
                                                  int64_t cols_per, int64_t RB, int64_t CS, int64_t nbr,
                                                  unsigned long long *rowmax, const double *omega, int64_t ldo,
                                                  int64_t lbar, int64_t KS, int64_t KSB, signed char *od, int *fexp) {
  const int64_t blk = blockIdx.x;
  if (blk < nbr) {
    const int64_t bx = blk % RB, by = (blk / RB) % CS, b = blk / (RB * CS);
    stc_rowmax<TW>(W, ldw, w_stride, m, n, cols_per, rowmax, bx, by, b);
  } else {
    const int64_t o = blk - nbr;
    stc_omega<NP>(omega, ldo, n, lbar, KS, od, fexp, o / KSB, o % KSB);
  }
}

// ---------------------------------------------------------------- main kernel
template <typename TW, int NP>
__global__ void __launch_bounds__(NTHR, 1) k_sketch_tc(const __grid_constant__ Args a,
                                                        const __grid_constant__ CUtensorMap tmW) {
  constexpr int NA = (512 - NLEV * NP) / (S * 8) > 4 ? 4 : (512 - NLEV * NP) / (S * 8);   // TMEM A regions
  constexpr int BT = NP * BK;            // bytes of one slice tile of Omega
  constexpr int BST = S * BT;            // bytes of one Omega stage
  constexpr int ACOL = NLEV * NP;        // first TMEM column of the A regions
  constexpr int WST = BM * BK * (int)sizeof(TW);   // bytes of one W stage
  constexpr int NWS = nws<TW>();
  extern __shared__ __align__(1024) unsigned char bsm[];
  __shared__ __align__(8) unsigned long long bars[2 * NA + 2 * NBS + 2 * nws<TW>() + 2];
  __shared__ uint32_t tmem_sh;
  __shared__ int last_sh;
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const long long k_entry = STC_CLK();
  const uint32_t b0 = tc::smem_u32(bars);
  auto A_FULL = [&](int x) { return b0 + 8u * x; };
  auto A_EMPTY = [&](int x) { return b0 + 8u * (NA + x); };
  auto B_FULL = [&](int x) { return b0 + 8u * (2 * NA + x); };
  auto B_EMPTY = [&](int x) { return b0 + 8u * (2 * NA + NBS + x); };
  auto W_FULL = [&](int x) { return b0 + 8u * (2 * NA + 2 * NBS + x); };
  auto W_EMPTY = [&](int x) { return b0 + 8u * (2 * NA + 2 * NBS + NWS + x); };
  const uint32_t ACC_FULL = b0 + 8u * (2 * NA + 2 * NBS + 2 * NWS), ACC_EMPTY = ACC_FULL + 8u;
  unsigned char *wsm = bsm + (size_t)NBS * BST;        // W stages after the Omega stages
  if (warp == 0) {
    asm volatile("tcgen05.alloc.cta_group::1.sync.aligned.shared::cta.b32 [%0], 512;\n" ::"r"(tc::smem_u32(&tmem_sh)));
    asm volatile("tcgen05.relinquish_alloc_permit.cta_group::1.sync.aligned;\n");
  }
  if (threadIdx.x == 32) {
    for (int x = 0; x < NA; ++x) {
      tc::mbar_init(A_FULL(x), NDW);
      tc::mbar_init(A_EMPTY(x), NMW);
    }
    for (int x = 0; x < NBS; ++x) {
      tc::mbar_init(B_FULL(x), 1);
      tc::mbar_init(B_EMPTY(x), NMW);
    }
    for (int x = 0; x < NWS; ++x) {
      tc::mbar_init(W_FULL(x), 1);
      tc::mbar_init(W_EMPTY(x), NDW);
    }
    tc::mbar_init(ACC_FULL, NMW);
    tc::mbar_init(ACC_EMPTY, NDW);
    asm volatile("fence.mbarrier_init.release.cluster;\n" ::: "memory");
  }
  tc::fence_before();
  __syncthreads();
  tc::fence_after();
  const uint32_t tmem = tmem_sh;
  const int cta = blockIdx.x;
  const long long k_ready = STC_CLK();
  if (STC_PROF && threadIdx.x == 0) {
    STC_ADD(13, k_ready - k_entry);
    unsigned long long t;
    asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t));
    g_stc_t[blockIdx.x][0] = t;
  }
  const int64_t g0 = unit_lo(a, cta), g1 = unit_hi(a, cta);
  unsigned smid;
  asm volatile("mov.u32 %0, %%smid;" : "=r"(smid));

  if (warp < NDW) {
    // ------------------------------------------------ digitizers + epilogue
    const int grp = warp >> 2, q = warp & 3;
    const int iloc = 32 * q + lane;
    const uint32_t lane_base = (uint32_t)(32 * q) << 16;
    int i = 0;               // CTA-local K-step counter (all chunks)
    int ck = 0;              // chunk counter
    for (int64_t g = g0; g < g1; ++ck) {
      const int64_t tile = g / a.KS;
      const int64_t ks0 = g - tile * a.KS;
      const int64_t ksc = min(min(a.KS, ks0 + (g1 - g)), ks0 + (int64_t)KCHUNK);   // chunk [ks0, ksc)
      const int nks = (int)(ksc - ks0);
      // the CTA's segment of this tile: [sa, sb) in K-steps
      const int64_t sa = max(g0 - tile * a.KS, (int64_t)0), sb = min(g1 - tile * a.KS, a.KS);
      const bool first = ks0 == sa, last = ksc == sb, full = sa == 0 && sb == a.KS;
      const int64_t nt = tile % a.NTN, mt = (tile / a.NTN) % a.MT, b = tile / (a.NTN * a.MT);
      const int64_t grow = mt * BM + iloc;
      const bool rowok = grow < a.m;
      const int e = row_exp<TW>(rowok ? a.rowmax[b * a.m + grow] : 0ull);
      const int sh = 55 - e;                                 // |sh| <= 55 + 149 for fp32 rows
      const int sh1 = sh > 127 ? 127 : (sh < -126 ? -126 : sh), sh2 = sh - sh1;
      const float s1 = __int_as_float((sh1 + 127) << 23);
      const float s2 = __int_as_float(((sh2 > 127 ? 127 : sh2) + 127) << 23);
      const double sd = ldexp(1.0, sh);
      // every K-step of the chunk: warp half grp converts columns [16 grp, 16 grp + 16) of its 32 rows
      for (int x = 0; x < nks; ++x) {
        const int ii = i + x;
        const int ws = ii % NWS, ab = ii % NA;
        long long c0 = STC_CLK();
        WAIT(W_FULL(ws), (uint32_t)((ii / NWS) & 1));
        long long c1 = STC_CLK();
        const TW *wt = reinterpret_cast<const TW *>(wsm + (size_t)ws * WST) + iloc + (size_t)grp * 16 * BM;
        TW v[16];
#pragma unroll
        for (int c = 0; c < 16; ++c) v[c] = wt[c * BM];
        __syncwarp();
        if (lane == 0) tc::mbar_arrive(W_EMPTY(ws));
        WAIT(A_EMPTY(ab), (uint32_t)(((ii / NA) & 1) ^ 1));
        long long c2 = STC_CLK();
        tc::fence_after();
        const uint32_t abase = tmem + lane_base + (uint32_t)(ACOL + ab * S * 8 + grp * 4);
        uint32_t wd[4][S];
#pragma unroll
        for (int c4 = 0; c4 < 4; ++c4) {
          long long X[4];
#pragma unroll
          for (int u = 0; u < 4; ++u) X[u] = to_fixed(v[c4 * 4 + u], s1, s2, sd);
          if (STC_NO_DIG) {
#pragma unroll
            for (int k = 0; k < S; ++k) wd[c4][k] = (uint32_t)X[k & 3];
          } else {
            pack4(X, wd[c4]);
          }
        }
#pragma unroll
#pragma unroll
        for (int s3 = 0; s3 < S; ++s3) tc::tmem_st4(abase + s3 * 8, wd[0][s3], wd[1][s3], wd[2][s3], wd[3][s3]);
        tc::tmem_wait_st();
        tc::fence_before();
        __syncwarp();
        if (lane == 0) tc::mbar_arrive(A_FULL(ab));
        if (STC_PROF && lane == 0 && warp == 0) {
          const long long c3 = clock64();
          STC_ADD(0, c1 - c0);
          STC_ADD(1, c2 - c1);
          STC_ADD(2, c3 - c2);
          STC_ADD(10, 1);
        }
      }
      // ---- epilogue of the chunk: levels -> exact (hi, lo) -> Y, or the CTA's partial slot
      long long e0 = STC_CLK();
      WAIT(ACC_FULL, (uint32_t)(ck & 1));
      long long e1 = STC_CLK();
      tc::fence_after();
      // a split tile's Q parts meet in tacc[tile], counted in cnt[tile] (Q > 1 only when T Q <= the
      // SM count); the chunks of one unit meet in own[smid]
      const int cf = (int)tile, cl = cf + a.Q - 1;
      long long *ow = a.own + (size_t)smid * SLOT;     // one CTA per SM at a time
      unsigned long long *ta = reinterpret_cast<unsigned long long *>(a.tacc + (size_t)cf * SLOT);
      for (int ch = grp; ch < NP / 8; ch += 2) {
        uint32_t raw[NLEV][8];
#pragma unroll
        for (int L = 0; L < NLEV; ++L) tc::tmem_ld8(tmem + lane_base + (uint32_t)(L * NP + ch * 8), raw[L]);
        tc::tmem_wait_ld();
#pragma unroll
        for (int xx = 0; xx < 8; ++xx) {
          const int t = ch * 8 + xx;
          long long P[NLEV];
#pragma unroll
          for (int L = 0; L < NLEV; ++L) P[L] = (long long)(int)raw[L][xx];
          long long hi = ((P[0] * 256 + P[1]) * 256 + P[2]) * 256 + P[3];
          long long lo = (P[4] * 256 + P[5]) * 256 + P[6];
          const size_t o = (size_t)t * BM + iloc;
          if (!first) {                           // earlier chunks of this segment
            hi += ow[o];
            lo += ow[(size_t)48 * BM + o];
          }
          if (!last) {
            ow[o] = hi;
            ow[(size_t)48 * BM + o] = lo;
          } else if (full) {
            const int64_t gc = nt * NP + t;
            if (rowok && gc < a.lbar)
              a.y[b * a.y_stride + gc * a.ldy + grow] =
                  ldexp((double)hi * 16777216.0 + (double)lo, e + __ldg(a.fexp + gc) - 62);
          } else {                                // exact: int64 reductions commute
            atomicAdd(ta + o, (unsigned long long)hi);
            atomicAdd(ta + (size_t)48 * BM + o, (unsigned long long)lo);
          }
        }
      }
      tc::fence_before();
      __syncwarp();
      if (lane == 0) tc::mbar_arrive(ACC_EMPTY);
      if (STC_PROF && threadIdx.x == 0) {
        STC_ADD(8, e1 - e0);
        STC_ADD(9, clock64() - e1);
      }
      if (last && !full) {
        // the last part to arrive converts the tile's exact sum to Y and clears the accumulator
        __threadfence();
        asm volatile("bar.sync 1, %0;\n" ::"n"(NDW * 32) : "memory");
        if (threadIdx.x == 0) {
          const int old = atomicAdd(a.cnt + cf, 1);
          last_sh = old == cl - cf;
          if (old == cl - cf) a.cnt[cf] = 0;
        }
        asm volatile("bar.sync 1, %0;\n" ::"n"(NDW * 32) : "memory");
        const long long l0 = STC_CLK();
        if (last_sh) {
          __threadfence();
          for (int ch = grp; ch < NP / 8; ch += 2) {
            long long hv[8], lv[8];
#pragma unroll
            for (int xx = 0; xx < 8; ++xx) {
              const size_t o = (size_t)(ch * 8 + xx) * BM + iloc;
              hv[xx] = (long long)__ldcg(ta + o);
              lv[xx] = (long long)__ldcg(ta + (size_t)48 * BM + o);
            }
#pragma unroll
            for (int xx = 0; xx < 8; ++xx) {
              const size_t o = (size_t)(ch * 8 + xx) * BM + iloc;
              ta[o] = 0ull;
              ta[(size_t)48 * BM + o] = 0ull;
              const int64_t gc = nt * NP + ch * 8 + xx;
              if (rowok && gc < a.lbar)
                a.y[b * a.y_stride + gc * a.ldy + grow] =
                    ldexp((double)hv[xx] * 16777216.0 + (double)lv[xx], e + __ldg(a.fexp + gc) - 62);
            }
          }
        }
        if (STC_PROF && threadIdx.x == 0) STC_ADD(12, clock64() - l0);
      }
      i += nks;
      g += nks;
    }
  } else if (warp < NDW + NMW) {
    // ------------------------------------------------ MMA warps
    const int mw = warp - NDW;
    if (lane == 0) {
      int i = 0;
      int seg = 0;
      for (int64_t g = g0; g < g1; ++seg) {
        const int64_t tile = g / a.KS;
        const int64_t ks0 = g - tile * a.KS;
        const int64_t ksc = min(min(a.KS, ks0 + (g1 - g)), ks0 + (int64_t)KCHUNK);
        const int nks = (int)(ksc - ks0);
        if (seg > 0) {
          WAIT(ACC_EMPTY, (uint32_t)((seg - 1) & 1));
          tc::fence_after();
        }
        for (int x = 0; x < nks; ++x) {
          const int ii = i + x;
          const int ab = (int)(ii % NA), bs = (int)(ii % NBS);
          long long m0 = STC_CLK();
          WAIT(A_FULL(ab), (uint32_t)((ii / NA) & 1));
          long long m1 = STC_CLK();
          WAIT(B_FULL(bs), (uint32_t)((ii / NBS) & 1));
          long long m2 = STC_CLK();
          tc::fence_after();
          const uint32_t at = tmem + (uint32_t)(ACOL + ab * S * 8);
          const uint64_t bd = tc::smem_desc(tc::smem_u32(bsm + (size_t)bs * BST));
          const uint32_t first = x == 0 ? 1u : 0u;
          if (STC_NO_MMA) {
          } else if (mw == 0) issue_kstep<NP, 0>(tmem, at, bd, first);
          else if (mw == 1) issue_kstep<NP, 1>(tmem, at, bd, first);
          else issue_kstep<NP, 2>(tmem, at, bd, first);
          tc::mma_commit(A_EMPTY(ab));
          tc::mma_commit(B_EMPTY(bs));
          if (STC_PROF && mw == 0) {
            STC_ADD(3, m1 - m0);
            STC_ADD(4, m2 - m1);
            STC_ADD(5, clock64() - m2);
          }
        }
        tc::mma_commit(ACC_FULL);
        i += nks;
        g += nks;
      }
    }
    __syncwarp();
  } else {
    // ------------------------------------------------ producer (one thread): W tiles by TMA and Omega
    // slices by bulk copies, each issued as soon as its ring stage is free (non-blocking probes,
    // so a full Omega ring never holds back the W prefetch)
    if (lane == 0) {
      const int64_t tile = g0 / a.KS;
      const int64_t nt = tile % a.NTN, mt = (tile / a.NTN) % a.MT, b = tile / (a.NTN * a.MT);
      const int64_t k0 = g0 - tile * a.KS;
      const int n = (int)(g1 - g0);
      int wi = 0, bi = 0;
      while (wi < n || bi < n) {
        if (wi < n && tc::mbar_test(W_EMPTY(wi % NWS), (uint32_t)(((wi / NWS) & 1) ^ 1))) {
          const int ws = wi % NWS;
          tc::mbar_expect(W_FULL(ws), (uint32_t)WST);
          asm volatile(
              "cp.async.bulk.tensor.3d.shared::cluster.global.tile.mbarrier::complete_tx::bytes [%0], [%1, {%2, %3, %4}], [%5];\n" ::"r"(
                  tc::smem_u32(wsm + (size_t)ws * WST)),
              "l"(reinterpret_cast<uint64_t>(&tmW)), "r"((int)(mt * BM)), "r"((int)((k0 + wi) * BK)), "r"((int)b),
              "r"(W_FULL(ws))
              : "memory");
          ++wi;
        }
        if (bi < n && tc::mbar_test(B_EMPTY(bi % NBS), (uint32_t)(((bi / NBS) & 1) ^ 1))) {
          const int bs = bi % NBS;
          tc::mbar_expect(B_FULL(bs), (uint32_t)BST);
          tc::bulk_g2s(tc::smem_u32(bsm + (size_t)bs * BST), a.od + ((size_t)nt * a.KS + k0 + bi) * BST, (uint32_t)BST,
                       B_FULL(bs));
          ++bi;
        }
      }
    }
    __syncwarp();
  }
  if (STC_PROF && threadIdx.x == 0) {
    STC_ADD(11, clock64() - k_ready);
    unsigned long long t;
    asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t));
    g_stc_t[blockIdx.x][1] = t;
  }
  tc::fence_before();
  __syncthreads();
  if (warp == 0) {
    tc::fence_after();
    asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, 512;\n" ::"r"(tmem));
  }
  if (STC_PROF && threadIdx.x == 0) {
    unsigned long long t;
    asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t));
    g_stc_t[blockIdx.x][2] = t;
  }
}

// Scratch layout: the split-tile accumulators and counters first, at offsets that do not depend
// on the problem (they must be zero between launches: zeroed when the buffer is allocated —
// sketch_tc_zero_bytes — and cleared again by each tile's last CTA), then the per-launch data.
struct Plan {
  int NP;
  int64_t KS, MT, NTN, T;
  int Q;
  size_t off_tacc, off_cnt, off_own, off_rowmax, off_od, off_fexp, bytes;
};

static int sm_count() {
  static int n = 0;
  if (!n) {
    int dev = 0;
    cudaGetDevice(&dev);
    cudaDeviceGetAttribute(&n, cudaDevAttrMultiProcessorCount, dev);
    if (n <= 0) n = 148;
  }
  return n;
}

static Plan plan(int64_t m, int64_t n, int64_t lbar, int64_t nb) {
  Plan p{};
  p.NTN = (lbar + 47) / 48;
  const int64_t per = (lbar + p.NTN - 1) / p.NTN;
  p.NP = (int)((per + 15) / 16 * 16);
  p.KS = (n + BK - 1) / BK;
  p.MT = (m + BM - 1) / BM;
  p.T = nb * p.MT * p.NTN;
  p.Q = (int)std::max<int64_t>(1, std::min<int64_t>(sm_count() / p.T, p.KS / 4));
  auto al = [](size_t x) { return (x + 255) & ~(size_t)255; };
  const int pmax = sm_count();
  size_t o = 0;
  p.off_tacc = o;
  o = al(o + (size_t)pmax * SLOT * 8);
  p.off_cnt = o;
  o = al(o + (size_t)pmax * 4);
  p.off_own = o;
  o = al(o + (size_t)pmax * SLOT * 8);
  p.off_rowmax = o;
  o = al(o + (size_t)nb * m * 8);
  p.off_od = o;
  o = al(o + (size_t)p.NTN * p.KS * S * p.NP * BK);
  p.off_fexp = o;
  o = al(o + (size_t)p.NTN * p.NP * 4);
  p.bytes = o + 256;
  return p;
}

static PFN_cuTensorMapEncodeTiled_v12000 tmap_encode() {
  static PFN_cuTensorMapEncodeTiled_v12000 fn = nullptr;
  static std::once_flag once;
  std::call_once(once, [] {
    cudaDriverEntryPointQueryResult q;
    void *p = nullptr;
    if (cudaGetDriverEntryPoint("cuTensorMapEncodeTiled", &p, cudaEnableDefault, &q) == cudaSuccess &&
        q == cudaDriverEntryPointSuccess)
      fn = reinterpret_cast<PFN_cuTensorMapEncodeTiled_v12000>(p);
    cudaGetLastError();
  });
  return fn;
}

template <typename TW, int NP>
static cudaError_t launch_main(const Args &a, const CUtensorMap &tm, cudaStream_t st) {
  constexpr int BST = S * NP * BK;
  const size_t smem = (size_t)NBS * BST + (size_t)nws<TW>() * BM * BK * sizeof(TW);
  cudaError_t e = cudaFuncSetAttribute(k_sketch_tc<TW, NP>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
  if (e != cudaSuccess) return e;
  k_sketch_tc<TW, NP><<<(unsigned)(a.T * a.Q), NTHR, smem, st>>>(a, tm);
  return cudaGetLastError();
}

}  // namespace stc

size_t sketch_tc_scratch_bytes(int64_t m, int64_t n, int64_t lbar, int64_t nb) { return stc::plan(m, n, lbar, nb).bytes; }
size_t sketch_tc_zero_bytes() { return stc::plan(1, 1, 1, 1).off_rowmax; }

// Y = W * Omega (m x lbar, fp64) on the tensor cores for nb problems sharing Omega (dense fp32 /
// fp64 W, column-major, ldw, w_stride; Omega n x lbar column-major fp64, ldo).  scratch: at least
// sketch_tc_scratch_bytes(m, n, lbar, nb), 256-byte aligned.  Two launches plus one memset.
cudaError_t launch_sketch_tc(const SketchArgs &sa, int64_t nb, const double *omega, int64_t ldo, void *scratch,
                             size_t scratch_bytes, cudaStream_t st, Prof *pf) {
  using namespace stc;
  const Plan p = plan(sa.m, sa.n, sa.lbar, nb);
  if (!scratch || scratch_bytes < p.bytes || sa.lbar < 1 || sa.m < 1 || sa.n < 1) return cudaErrorInvalidValue;
  char *base = reinterpret_cast<char *>(scratch);
  Args a{};
  a.w = sa.w;
  a.ldw = sa.ldw;
  a.w_stride = sa.w_stride;
  a.m = sa.m;
  a.n = sa.n;
  a.lbar = sa.lbar;
  a.nb = nb;
  a.y = reinterpret_cast<double *>(sa.y);
  a.ldy = sa.ldy;
  a.y_stride = sa.y_stride;
  a.rowmax = reinterpret_cast<unsigned long long *>(base + p.off_rowmax);
  a.cnt = reinterpret_cast<int *>(base + p.off_cnt);
  a.tacc = reinterpret_cast<long long *>(base + p.off_tacc);
  a.own = reinterpret_cast<long long *>(base + p.off_own);
  a.od = reinterpret_cast<signed char *>(base + p.off_od);
  a.fexp = reinterpret_cast<int *>(base + p.off_fexp);
  a.KS = p.KS;
  a.MT = p.MT;
  a.NTN = p.NTN;
  a.T = p.T;
  a.Q = p.Q;
  // W by TMA: a 3-D tensor map over (m, n, nb), box 128 x 32 x 1 (zero fill beyond the edges)
  const size_t elt = sa.dtype == LRA_F32 ? 4 : 8;
  const int64_t wstr = nb > 1 ? sa.w_stride : sa.ldw * sa.n;
  if (!tmap_encode() || (sa.ldw * (int64_t)elt) % 16 != 0 || (wstr * (int64_t)elt) % 16 != 0 ||
      (reinterpret_cast<uintptr_t>(sa.w) & 15) != 0)
    return cudaErrorInvalidConfiguration;
  CUtensorMap tm;
  memset(&tm, 0, sizeof(tm));
  {
    cuuint64_t dims[3] = {(cuuint64_t)sa.m, (cuuint64_t)sa.n, (cuuint64_t)nb};
    cuuint64_t strides[2] = {(cuuint64_t)(sa.ldw * elt), (cuuint64_t)(wstr * elt)};
    cuuint32_t box[3] = {(cuuint32_t)BM, (cuuint32_t)BK, 1u};
    cuuint32_t estr[3] = {1u, 1u, 1u};
    if (tmap_encode()(&tm, elt == 4 ? CU_TENSOR_MAP_DATA_TYPE_FLOAT32 : CU_TENSOR_MAP_DATA_TYPE_FLOAT64, 3,
                      const_cast<void *>(sa.w), dims, strides, box, estr, CU_TENSOR_MAP_INTERLEAVE_NONE,
                      CU_TENSOR_MAP_SWIZZLE_NONE, CU_TENSOR_MAP_L2_PROMOTION_L2_256B,
                      CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE) != CUDA_SUCCESS)
      return cudaErrorInvalidConfiguration;
  }
  pf->begin("k_sketch_tc_prep", st);
  cudaError_t e = cudaMemsetAsync(base + p.off_rowmax, 0, (size_t)nb * sa.m * 8, st);   // row maxima
  if (e != cudaSuccess) return e;
  {
    const int64_t RB = (sa.m + 1023) / 1024;
    int64_t CS = (2 * sm_count() + RB * nb - 1) / (RB * nb);  // ~two CTAs per SM, 128 KB in flight
    CS = std::max<int64_t>(1, std::min<int64_t>(CS, (sa.n + 15) / 16));
    const int64_t cols_per = (sa.n + CS - 1) / CS;
    const int64_t CSr = (sa.n + cols_per - 1) / cols_per;
    const int64_t nbr = RB * CSr * nb, KSB = (p.KS + 7) / 8, nbo = p.NTN * p.NP * KSB;
    unsigned long long *rm = const_cast<unsigned long long *>(a.rowmax);
    signed char *od = const_cast<signed char *>(a.od);
    int *fx = const_cast<int *>(a.fexp);
    const unsigned grid = (unsigned)(nbr + nbo);
#define STC_PREP(TW, NPV)                                                                                       \
  k_stc_prep<TW, NPV><<<grid, 256, 0, st>>>(reinterpret_cast<const TW *>(sa.w), sa.ldw, sa.w_stride, sa.m, sa.n, \
                                            cols_per, RB, CSr, nbr, rm, omega, ldo, sa.lbar, p.KS, KSB, od, fx)
    if (sa.dtype == LRA_F32) {
      if (p.NP == 16) STC_PREP(float, 16);
      else if (p.NP == 32) STC_PREP(float, 32);
      else STC_PREP(float, 48);
    } else {
      if (p.NP == 16) STC_PREP(double, 16);
      else if (p.NP == 32) STC_PREP(double, 32);
      else STC_PREP(double, 48);
    }
#undef STC_PREP
    if ((e = cudaGetLastError()) != cudaSuccess) return e;
  }
  pf->end(st);
  pf->begin("k_sketch_tc", st);
  const bool f32 = sa.dtype == LRA_F32;
  switch (p.NP) {
    case 16: e = f32 ? launch_main<float, 16>(a, tm, st) : launch_main<double, 16>(a, tm, st); break;
    case 32: e = f32 ? launch_main<float, 32>(a, tm, st) : launch_main<double, 32>(a, tm, st); break;
    default: e = f32 ? launch_main<float, 48>(a, tm, st) : launch_main<double, 48>(a, tm, st); break;
  }
  pf->end(st);
  return e;
}

}  // namespace lra
