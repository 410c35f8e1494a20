// residual_tc.cu — the a-posteriori check rho = ||W - CUR||_F / ||W||_F (eq. eqcur0,
// P:1153-1155) with the rank-r product CUR = A*B on the 5th-generation tensor cores.
//
// A (m x r) and B (r x n) are fp64.  Their product must be accurate far beyond fp32
// (config 2: rho ~ 7e-7, so W - AB cancels ~21 bits), so the contraction is
// done exactly in integers (Ozaki-style splitting):
//   A[i,t] = 2^ea_i * sum_s a_s[i,t] 128^-(s+1),   B[t,j] = 2^fb_j * sum_u b_u[t,j] 128^-(u+1)
// with balanced base-128 digits |a_s|, |b_u| <= 64 (int8), one exponent per row of A and per
// column of B.  Keeping the digit products with s + u <= S-1 (S = 6 for PRECISE: 2^-42
// relative truncation; S = 3 for FAST), level l = s + u is accumulated EXACTLY in int32 by
// tcgen05.mma kind::i8 into its own TMEM accumulator (|P_l| <= (l+1) * K * 64^2 < 2^31), and
// the epilogue recombines the levels with integer shifts and two exact int->fp64 conversions:
//   AB[i,j] = 2^(ea_i + fb_j - 35) * (Q0 2^14 + Q1 + Q2 2^-14),  Q_k = 128 P_2k + P_2k+1,
// then d = W - AB, sum d^2 and sum W^2 in fp64 (per-CTA partials, fixed-order reduction).
//
// k_split_a / k_split_b write the digit slices directly in the UMMA canonical K-major
// no-swizzle layout (core matrix = 8 rows x 16 bytes; LBO = 128 B between the two K halves,
// SBO = 256 B between 8-row groups), so the main kernel stages them with plain 16-byte
// cp.async.  k_residual_tc: one CTA (4 warps) per 128-row block x column chunk; per 32-column
// tile the W tile and the B slices are double-buffered in shared memory, one elected thread
// issues the S(S+1)/2 x KB MMAs (M=128, N=32, K=32), tcgen05.commit signals an mbarrier and
// the four warps drain TMEM (tcgen05.ld 32x32b, warp w owns rows 32w..32w+31).
#include "kernels.cuh"

#include <cstdlib>

namespace lra {
// phase counters (clock64 cycles summed over CTAs): 0 MMA wait B, 1 MMA wait TMEM, 2 MMA issue,
// 3 producer wait B stage, 4 producer wait A, 5 MMA wait A, 6 epilogue wait TMEM (warp 0),
// 7 epilogue work (warp 0), 8 tiles (count)
__device__ unsigned long long g_rtc_cyc[16];
#ifndef RTC_PROF
#define RTC_PROF 0      // 1: per-role clock64 counters (lra_debug_counters_residual)
#endif
#define RTC_CLK() (RTC_PROF ? clock64() : 0ll)
#ifndef RTC_EPI_LDONLY
#define RTC_EPI_LDONLY 0   // 1: epilogue reads TMEM but skips the arithmetic (diagnostics)
#endif
namespace rtc {

constexpr int BM = 128;        // rows per CTA (MMA M)
constexpr int BN = 32;         // columns per tile (MMA N)
constexpr int BK = 32;         // K per MMA (kind::i8)
constexpr int SMAX = 6;
constexpr int A_TILE = BM * BK;          // bytes of one (slice, K-block) A tile  (4096)
constexpr int B_TILE = BN * BK;          // bytes of one (slice, K-block) B tile  (1024)

__device__ __forceinline__ uint32_t smem_u32(const void *p) { return (uint32_t)__cvta_generic_to_shared(p); }

// byte offset of element (row, kk) inside a canonical K-major no-swizzle tile
__device__ __forceinline__ int canon_off(int row, int kk) {
  return (row >> 3) * 256 + (kk >> 4) * 128 + (row & 7) * 16 + (kk & 15);
}

// balanced base-128 digits of x * 2^-e (|x 2^-e| < 1/2): d_s in [-64, 64]
__device__ __forceinline__ void digits(double x, int e, int S, signed char *d) {
  double y = ldexp(x, -e);
  for (int s = 0; s < S; ++s) {
    y *= 128.0;
    const double q = rint(y);
    d[s] = (signed char)(int)q;
    y -= q;
  }
}

__device__ __forceinline__ unsigned long long wmax_bits(unsigned long long k) {   // max over the warp
  const unsigned hi = (unsigned)(k >> 32);
  const unsigned mhi = __reduce_max_sync(0xffffffffu, hi);
  const unsigned mlo = __reduce_max_sync(0xffffffffu, hi == mhi ? (unsigned)k : 0u);
  return ((unsigned long long)mhi << 32) | mlo;
}

__device__ __forceinline__ int scale_exp(double mx) {
  return mx > 0.0 ? ilogb(mx) + 2 : 0;     // mx * 2^-e < 1/2
}

// A: m x r (lda = m), per problem stride a_stride.  Output per problem / row block:
// Aq[(b * RB + rb) * KB * S + kb * S + s][A_TILE], sa[b * m + i] = ea_i (int32).
// grid (RB, nb), 256 threads: thread = (row i, K half h); 16 digits x S slices per thread,
// written as S 16-byte chunks of the canonical layout.
__device__ __forceinline__ double strided_absmax(const double *p, int64_t stride, int r) {
  double mx = 0.0;
  for (int t0 = 0; t0 < r; t0 += 8) {
    double v[8];
#pragma unroll
    for (int u = 0; u < 8; ++u) v[u] = (t0 + u < r) ? __ldg(p + (int64_t)(t0 + u) * stride) : 0.0;
#pragma unroll
    for (int u = 0; u < 8; ++u) mx = fmax(mx, fabs(v[u]));
  }
  return mx;
}

__global__ void __launch_bounds__(64) k_split_a(const double *A, int64_t m, int r, int64_t a_stride, int S, int KB,
                                                signed char *Aq, int *sa, const int32_t *status) {
  const int64_t b = blockIdx.y;
  const int64_t rb = blockIdx.x >> 2;                 // 4 CTAs of 32 rows per 128-row block
  const int64_t RB = gridDim.x >> 2;
  signed char *base = Aq + (size_t)(b * RB + rb) * KB * S * A_TILE;
  const int i = (int)(blockIdx.x & 3) * 32 + (threadIdx.x & 31), h = threadIdx.x >> 5;
  const int64_t gi = rb * BM + i;
  const bool ok = gi < m && !(status && status[b] != LRA_OK);
  const double *Ab = A + b * a_stride;
  const double mx = ok ? strided_absmax(Ab + gi, m, r) : 0.0;
  const int e = scale_exp(mx);
  const double p2 = ldexp(1.0, -e);
  if (gi < m && h == 0) sa[b * m + gi] = ok ? e : -4000;     // -4000: row contributes nothing
  for (int kb = 0; kb < KB; ++kb) {
    uint32_t w[SMAX][4];
#pragma unroll
    for (int s = 0; s < SMAX; ++s) w[s][0] = w[s][1] = w[s][2] = w[s][3] = 0u;
#pragma unroll
    for (int kk = 0; kk < 16; ++kk) {
      const int t = kb * BK + h * 16 + kk;
      double y = (ok && t < r) ? Ab[(int64_t)t * m + gi] * p2 : 0.0;
#pragma unroll
      for (int s = 0; s < SMAX; ++s) {
        if (s < S) {
          y *= 128.0;
          const double q = rint(y);
          y -= q;
          w[s][kk >> 2] |= ((uint32_t)(int)q & 0xffu) << (8 * (kk & 3));
        }
      }
    }
    for (int s = 0; s < S; ++s)
      *reinterpret_cast<uint4 *>(base + (size_t)(kb * S + s) * A_TILE + (i >> 3) * 256 + h * 128 + (i & 7) * 16) =
          make_uint4(w[s][0], w[s][1], w[s][2], w[s][3]);
  }
}

// B: r x n (ld r), per problem stride b_stride.  Output Bq[((b * CB + cb) * KB + kb) * S + s][B_TILE]
// and sbq[(b * CB + cb) * BN + jj] = fb of the tile (int32; -4000 beyond n).  grid (CB, nb), 64 threads.
__global__ void __launch_bounds__(2 * BN) k_split_b(const double *B, int64_t n, int r, int64_t b_stride, int S, int KB,
                                                    signed char *Bq, int *sbq, const int32_t *status) {
  const int64_t b = blockIdx.y, cb = blockIdx.x;
  const int64_t CB = gridDim.x;
  signed char *base = Bq + (size_t)(b * CB + cb) * KB * S * B_TILE;
  const int jj = threadIdx.x & (BN - 1), h = threadIdx.x >> 5;
  const int64_t gj = cb * BN + jj;
  const bool ok = gj < n && !(status && status[b] != LRA_OK);
  const double *Bb = B + b * b_stride;
  // one exponent per 32-column tile (the tile's max |B|): the epilogue then builds one scale
  // per row and tile instead of one per output
  const double mxc = ok ? strided_absmax(Bb + gj * r, 1, r) : 0.0;
  const double mx = __longlong_as_double((long long)wmax_bits((unsigned long long)__double_as_longlong(mxc)));
  const int e = scale_exp(mx);
  const double p2 = ldexp(1.0, -e);
  if (h == 0) sbq[(b * CB + cb) * BN + jj] = ok ? e : -4000;   // (same e for the tile's columns)
  for (int kb = 0; kb < KB; ++kb) {
    uint32_t w[SMAX][4];
#pragma unroll
    for (int s = 0; s < SMAX; ++s) w[s][0] = w[s][1] = w[s][2] = w[s][3] = 0u;
#pragma unroll
    for (int kk = 0; kk < 16; ++kk) {
      const int t = kb * BK + h * 16 + kk;
      double y = (ok && t < r) ? Bb[gj * r + t] * p2 : 0.0;
#pragma unroll
      for (int s = 0; s < SMAX; ++s) {
        if (s < S) {
          y *= 128.0;
          const double q = rint(y);
          y -= q;
          w[s][kk >> 2] |= ((uint32_t)(int)q & 0xffu) << (8 * (kk & 3));
        }
      }
    }
    for (int s = 0; s < S; ++s)
      *reinterpret_cast<uint4 *>(base + (size_t)(kb * S + s) * B_TILE + (jj >> 3) * 256 + h * 128 + (jj & 7) * 16) =
          make_uint4(w[s][0], w[s][1], w[s][2], w[s][3]);
  }
}

// One launch for both factors (grid.x = RB + ceil(CB / 4), grid.y = nb, 128 threads), every
// input value loaded exactly once into registers (all r loads in flight):
//  - A CTAs: thread = one row of a 128-row block; the row exponent from its r values;
//  - B CTAs: 4 warps = 4 tiles of 32 columns, thread = one column; the tile exponent is the
//    warp max of the column maxima.
// The digits are the same as k_split_a / k_split_b (same exponents, same digit recurrence),
// written to the same canonical layout.
template <int KBT>
__global__ void __launch_bounds__(128) k_split_ab(const double *A, const double *B, int64_t m, int64_t n, int r,
                                                  int64_t a_stride, int64_t b_stride, int S, int64_t RB, int64_t CB,
                                                  signed char *Aq, signed char *Bq, int *sa, int *sbq,
                                                  const int32_t *status) {
  constexpr int RT = KBT * BK;                 // values per thread (zero beyond r)
  const int64_t b = blockIdx.y;
  const bool live = !(status && status[b] != LRA_OK);
  double v[RT];
  double mx = 0.0;
  signed char *base;
  int boff;
  int tile_bytes;
  if ((int64_t)blockIdx.x < RB) {
    const int64_t rb = blockIdx.x;
    const int i = threadIdx.x;
    const int64_t gi = rb * BM + i;
    const bool ok = live && gi < m;
    const double *Ab = A + b * a_stride + gi;
#pragma unroll
    for (int t = 0; t < RT; ++t) v[t] = (ok && t < r) ? __ldg(Ab + (int64_t)t * m) : 0.0;
#pragma unroll
    for (int t = 0; t < RT; ++t) mx = fmax(mx, fabs(v[t]));
    const int e = scale_exp(mx);
    if (gi < m) sa[b * m + gi] = ok ? e : -4000;     // -4000: row contributes nothing
    const double p2 = ldexp(1.0, -e);
#pragma unroll
    for (int t = 0; t < RT; ++t) v[t] *= p2;
    base = Aq + (size_t)(b * RB + rb) * KBT * S * A_TILE;
    boff = (i >> 3) * 256 + (i & 7) * 16;
    tile_bytes = A_TILE;
  } else {
    const int64_t cb = ((int64_t)blockIdx.x - RB) * 4 + (threadIdx.x >> 5);
    const int jj = threadIdx.x & 31;
    const int64_t gj = cb * BN + jj;
    const bool ok = live && cb < CB && gj < n;
    const double *Bb = B + b * b_stride + gj * r;
#pragma unroll
    for (int t = 0; t < RT; ++t) v[t] = (ok && t < r) ? __ldg(Bb + t) : 0.0;
#pragma unroll
    for (int t = 0; t < RT; ++t) mx = fmax(mx, fabs(v[t]));
    // one exponent per 32-column tile (the tile's max |B|)
    mx = __longlong_as_double((long long)wmax_bits((unsigned long long)__double_as_longlong(mx)));
    const int e = scale_exp(mx);
    if (cb >= CB) return;
    sbq[(b * CB + cb) * BN + jj] = ok ? e : -4000;
    const double p2 = ldexp(1.0, -e);
#pragma unroll
    for (int t = 0; t < RT; ++t) v[t] *= p2;
    base = Bq + (size_t)(b * CB + cb) * KBT * S * B_TILE;
    boff = (jj >> 3) * 256 + (jj & 7) * 16;
    tile_bytes = B_TILE;
  }
  // balanced base-128 digits, slice by slice (y <- 128 y - rint(128 y))
  for (int s = 0; s < S; ++s) {
    uint32_t w[KBT][2][4];
#pragma unroll
    for (int t = 0; t < RT; ++t) {
      const double y = v[t] * 128.0;
      const double q = rint(y);
      v[t] = y - q;
      const int kb = t / BK, h = (t % BK) / 16, kk = t % 16;
      const uint32_t byte = ((uint32_t)(int)q & 0xffu) << (8 * (kk & 3));
      if ((kk & 3) == 0) w[kb][h][kk >> 2] = byte;
      else w[kb][h][kk >> 2] |= byte;
    }
#pragma unroll
    for (int kb = 0; kb < KBT; ++kb)
#pragma unroll
      for (int h = 0; h < 2; ++h)
        *reinterpret_cast<uint4 *>(base + (size_t)(kb * S + s) * tile_bytes + boff + h * 128) =
            make_uint4(w[kb][h][0], w[kb][h][1], w[kb][h][2], w[kb][h][3]);
  }
}

__device__ __forceinline__ uint64_t smem_desc(uint32_t addr) {
  // K-major, no swizzle: LBO = 128 B (K halves), SBO = 256 B (8-row groups), version 1 (sm100)
  return (uint64_t)((addr & 0x3FFFF) >> 4) | ((uint64_t)(128 >> 4) << 16) | ((uint64_t)(256 >> 4) << 32) |
         (1ull << 46);
}
// kind::i8, D = s32, A = B = signed 8-bit, both K-major, M = 128, N = 32
constexpr uint32_t IDESC = (2u << 4) | (1u << 7) | (1u << 10) | ((uint32_t)(BN >> 3) << 17) | ((uint32_t)(BM >> 4) << 24);

__device__ __forceinline__ void mma_i8(uint32_t tmem_d, uint64_t adesc, uint64_t bdesc, uint32_t acc) {
  asm volatile(
      "{\n\t.reg .pred p;\n\t"
      "setp.ne.b32 p, %4, 0;\n\t"
      "tcgen05.mma.cta_group::1.kind::i8 [%0], %1, %2, %3, p;\n\t}\n" ::"r"(tmem_d),
      "l"(adesc), "l"(bdesc), "r"(IDESC), "r"(acc));
}
// A operand from TMEM (TS mode): A 128 x 32 int8 at TMEM columns [a_tmem, a_tmem + 8)
__device__ __forceinline__ void mma_i8_ts(uint32_t tmem_d, uint32_t a_tmem, uint64_t bdesc, uint32_t acc) {
  asm volatile(
      "{\n\t.reg .pred p;\n\t"
      "setp.ne.b32 p, %4, 0;\n\t"
      "tcgen05.mma.cta_group::1.kind::i8 [%0], [%1], %2, %3, p;\n\t}\n" ::"r"(tmem_d),
      "r"(a_tmem), "l"(bdesc), "r"(IDESC), "r"(acc));
}
// smem (canonical K-major tile, 128 rows x 32 bytes) -> TMEM 128 lanes x 8 columns
__device__ __forceinline__ void tmem_cp_128x256b(uint32_t taddr, uint64_t sdesc) {
  asm volatile("tcgen05.cp.cta_group::1.128x256b [%0], %1;\n" ::"r"(taddr), "l"(sdesc) : "memory");
}
__device__ __forceinline__ void mma_commit(uint32_t mbar) {
  asm volatile("tcgen05.commit.cta_group::1.mbarrier::arrive::one.shared::cluster.b64 [%0];\n" ::"r"(mbar) : "memory");
}
__device__ __forceinline__ void cp16(void *s, const void *g) {
  asm volatile("cp.async.cg.shared.global [%0], [%1], 16;\n" ::"r"(smem_u32(s)), "l"(g));
}
__device__ __forceinline__ void cp_commit() { asm volatile("cp.async.commit_group;\n" ::: "memory"); }
__device__ __forceinline__ void cp_wait1() { asm volatile("cp.async.wait_group 1;\n" ::: "memory"); }
__device__ __forceinline__ void cp_wait2() { asm volatile("cp.async.wait_group 2;\n" ::: "memory"); }
__device__ __forceinline__ void cp_wait0() { asm volatile("cp.async.wait_group 0;\n" ::: "memory"); }
__device__ __forceinline__ void mbar_init(uint32_t a, uint32_t count) {
  asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;\n" ::"r"(a), "r"(count));
}
__device__ __forceinline__ void mbar_arrive(uint32_t a) {
  asm volatile("mbarrier.arrive.shared::cta.b64 _, [%0];\n" ::"r"(a) : "memory");
}
__device__ __forceinline__ void mbar_expect(uint32_t a, uint32_t bytes) {
  asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;\n" ::"r"(a), "r"(bytes) : "memory");
}
__device__ __forceinline__ void bulk_g2s(uint32_t dst, const void *src, uint32_t bytes, uint32_t mbar) {
  asm volatile("cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];\n" ::"r"(dst),
               "l"(src), "r"(bytes), "r"(mbar)
               : "memory");
}
__device__ __forceinline__ void mbar_wait(uint32_t addr, uint32_t phase) {
  uint32_t done = 0;
  do {
    asm volatile(
        "{\n\t.reg .pred p;\n\t"
        "mbarrier.try_wait.parity.shared::cta.b64 p, [%1], %2;\n\t"
        "selp.u32 %0, 1, 0, p;\n\t}\n"
        : "=r"(done)
        : "r"(addr), "r"(phase)
        : "memory");
  } while (!done);
}

__device__ __forceinline__ bool elect_one() {
  uint32_t pred = 0;
  asm volatile("{\n\t.reg .pred P;\n\telect.sync _|P, 0xffffffff;\n\tselp.u32 %0, 1, 0, P;\n\t}\n" : "=r"(pred));
  return pred != 0;
}

__device__ __forceinline__ double i64_to_f64(long long v) {   // exact for |v| < 2^51
  return __longlong_as_double(v + 0x4338000000000000LL) - 6755399441055744.0;
}

struct TcArgs {
  int dtype;
  int64_t m, n, ldw, w_stride;
  const void *w;
  const signed char *Aq, *Bq;
  const int *sa, *sbq;             // per-row / per-column scale exponents
  int S, KB;
  int64_t RB, CB;                 // row blocks, 32-column blocks per problem
  int tpi;                        // 32-column tiles per work item
  int64_t nchunk;                 // column chunks (items) per row block
  int64_t items;                  // nb * RB * nchunk
  int nst, wring;                 // B-slice stages (<= NST) and W ring depth (2 or 3) fitting smem
  double2 *partial;               // per problem: RB * nchunk partials (one per item)
  const int32_t *status;
};

constexpr int NST = 6;            // max B-slice stages
constexpr int NEPI = 16;          // epilogue warps: two groups of 8 own alternate tiles (= TMEM buffers);
                                  // warp w: TMEM lanes 32 (w % 4), columns 16 ((w / 4) % 2) ..
constexpr int NTC = 32 * (NEPI + 2);   // + producer warp + MMA warp
constexpr int WRING = 3;          // per-warp W ring depth (tiles)

struct Bars {
  unsigned long long bfull[NST], bempty[NST], tfull[2], tempty[2], afull[2], aempty[2];
};

// Persistent, warp-specialized.  Work item = (problem, row block, chunk of tpi tiles).
template <typename TW, int S>
__global__ void __launch_bounds__(NTC, 1) k_residual_tc(TcArgs a) {
  extern __shared__ __align__(1024) unsigned char smem[];
  __shared__ __align__(8) Bars bar;
  __shared__ uint32_t tmem_base_sh;
  const int KB = a.KB;
  const int tid = threadIdx.x, warp = tid >> 5, lane = tid & 31;
  const int aBytes = S * KB * A_TILE, bBytes = S * KB * B_TILE;
  const int stBytes = bBytes;
  unsigned char *As = smem;                            // 2 item buffers
  unsigned char *Bst = smem + 2 * aBytes;              // NST stages
  TW *Wr = reinterpret_cast<TW *>(Bst + a.nst * stBytes);   // NEPI x WRING x 16 cols x 32 rows
  const uint32_t bb = smem_u32(&bar);
  const uint32_t B_BFULL = bb + offsetof(Bars, bfull), B_BEMPTY = bb + offsetof(Bars, bempty);
  const uint32_t B_TFULL = bb + offsetof(Bars, tfull), B_TEMPTY = bb + offsetof(Bars, tempty);
  const uint32_t B_AFULL = bb + offsetof(Bars, afull), B_AEMPTY = bb + offsetof(Bars, aempty);
  if (warp == NEPI + 1) {
    asm volatile("tcgen05.alloc.cta_group::1.sync.aligned.shared::cta.b32 [%0], 512;\n" ::"r"(smem_u32(&tmem_base_sh)));
    asm volatile("tcgen05.relinquish_alloc_permit.cta_group::1.sync.aligned;\n");
  }
  if (tid == 0) {
    for (int i = 0; i < a.nst; ++i) {
      mbar_init(B_BFULL + 8 * i, 1);
      mbar_init(B_BEMPTY + 8 * i, 1);
    }
    for (int i = 0; i < 2; ++i) {
      mbar_init(B_TFULL + 8 * i, 1);
      mbar_init(B_TEMPTY + 8 * i, NEPI / 2);   // released by the 8 warps of its group
    }
    for (int i = 0; i < 2; ++i) {
      mbar_init(B_AFULL + 8 * i, 1);
      mbar_init(B_AEMPTY + 8 * i, 1);
    }
    asm volatile("fence.mbarrier_init.release.cluster;\n" ::: "memory");
  }
  asm volatile("tcgen05.fence::before_thread_sync;\n" ::: "memory");
  __syncthreads();
  asm volatile("tcgen05.fence::after_thread_sync;\n" ::: "memory");
  const uint32_t tmem = tmem_base_sh;

  auto item_of = [&](int64_t it, int64_t &b, int64_t &rb, int64_t &c0, int64_t &c1) {
    b = it / (a.RB * a.nchunk);
    const int64_t rem = it % (a.RB * a.nchunk);
    const int64_t ch = rem / a.RB;
    rb = rem % a.RB;
    c0 = ch * a.tpi;
    c1 = min(c0 + a.tpi, a.CB);
  };

  if (warp == NEPI) {
    // ===== producer: A slices per item, B slices per tile (warp-converged, one elected lane issues)
    {
      long long pw_b = 0, pw_a = 0;
      int64_t k = 0, ni = 0;
      for (int64_t it = blockIdx.x; it < a.items; it += gridDim.x) {
        int64_t b, rb, c0, c1;
        item_of(it, b, rb, c0, c1);
        if (a.status && a.status[b] != LRA_OK) continue;
        const int ab = (int)(ni & 1);
        long long t0 = RTC_CLK();
        if (ni >= 2) mbar_wait(B_AEMPTY + 8 * ab, (uint32_t)(((ni >> 1) - 1) & 1));
        pw_a += RTC_CLK() - t0;
        ++ni;
        if (elect_one()) {
          mbar_expect(B_AFULL + 8 * ab, (uint32_t)aBytes);
          bulk_g2s(smem_u32(As + ab * aBytes), a.Aq + (size_t)(b * a.RB + rb) * aBytes, (uint32_t)aBytes,
                   B_AFULL + 8 * ab);
        }
        __syncwarp();
        for (int64_t ct = c0; ct < c1; ++ct, ++k) {
          const int st = (int)(k % a.nst);
          long long t0 = RTC_CLK();
          if (k >= a.nst) mbar_wait(B_BEMPTY + 8 * st, (uint32_t)(((k / a.nst) - 1) & 1));
          pw_b += RTC_CLK() - t0;
          if (elect_one()) {
            mbar_expect(B_BFULL + 8 * st, (uint32_t)stBytes);
            const uint32_t dst = smem_u32(Bst + st * stBytes);
            bulk_g2s(dst, a.Bq + (size_t)(b * a.CB + ct) * bBytes, (uint32_t)bBytes, B_BFULL + 8 * st);
          }
          __syncwarp();
        }
      }
      if (lane == 0) {
        atomicAdd(&g_rtc_cyc[3], (unsigned long long)pw_b);
        atomicAdd(&g_rtc_cyc[4], (unsigned long long)pw_a);
      }
    }
  } else if (warp == NEPI + 1) {
    // ===== MMA issuer (warp-converged; one elected lane issues the tcgen05 instructions)
    {
      long long mw_b = 0, mw_t = 0, mw_i = 0, mw_a = 0;
      int64_t k = 0, ni = 0;
      for (int64_t it = blockIdx.x; it < a.items; it += gridDim.x) {
        int64_t b, rb, c0, c1;
        item_of(it, b, rb, c0, c1);
        if (a.status && a.status[b] != LRA_OK) continue;
        const int ab = (int)(ni & 1);
        long long t0 = RTC_CLK();
        mbar_wait(B_AFULL + 8 * ab, (uint32_t)((ni >> 1) & 1));
        mw_a += RTC_CLK() - t0;
        ++ni;
        for (int64_t ct = c0; ct < c1; ++ct, ++k) {
          const int st = (int)(k % a.nst), tb = (int)(k & 1);
          long long t1 = RTC_CLK();
          mbar_wait(B_BFULL + 8 * st, (uint32_t)((k / a.nst) & 1));
          long long t2 = RTC_CLK();
          if (k >= 2) mbar_wait(B_TEMPTY + 8 * tb, (uint32_t)(((k >> 1) - 1) & 1));
          long long t3 = RTC_CLK();
          mw_b += t2 - t1;
          mw_t += t3 - t2;
          asm volatile("tcgen05.fence::after_thread_sync;\n" ::: "memory");
          const uint64_t bdesc = smem_desc(smem_u32(Bst + st * stBytes));
          const uint32_t dbase = tmem + (uint32_t)(tb * 192);
          const uint32_t abase_t = tmem + 384;        // A slices in TMEM: 8 columns per (kb, slice)
          if (elect_one()) {
            if (ct == c0) {   // new item: stage its A slices into TMEM (ordered after prior MMAs)
              const uint64_t adesc = smem_desc(smem_u32(As + ab * aBytes));
              for (int j = 0; j < KB * S; ++j) tmem_cp_128x256b(abase_t + 8 * j, adesc + (uint64_t)((j * A_TILE) >> 4));
            }
            // Products interleaved across the S level accumulators (round j issues product j of
            // every level l >= j), so consecutive MMAs rarely accumulate into the same TMEM
            // region and the tensor pipe is not serialized on accumulator dependences.
            for (int kb = 0; kb < KB; ++kb) {
#pragma unroll
              for (int j = 0; j < S; ++j) {
#pragma unroll
                for (int l = j; l < S; ++l) {
                  const int s2 = j, u = l - j;      // level l, product (s2, u)
                  mma_i8_ts(dbase + l * BN, abase_t + 8 * (kb * S + s2),
                            bdesc + (uint64_t)(((kb * S + u) * B_TILE) >> 4), (j | kb) ? 1u : 0u);
                }
              }
            }
            mma_commit(B_BEMPTY + 8 * st);     // B stage free once these MMAs complete
            mma_commit(B_TFULL + 8 * tb);      // accumulators ready
          }
          __syncwarp();
          mw_i += RTC_CLK() - t3;
        }
        if (elect_one()) mma_commit(B_AEMPTY + 8 * ab);   // A slices free after the item's MMAs
        __syncwarp();
      }
      if (lane == 0) {
        atomicAdd(&g_rtc_cyc[0], (unsigned long long)mw_b);
        atomicAdd(&g_rtc_cyc[1], (unsigned long long)mw_t);
        atomicAdd(&g_rtc_cyc[2], (unsigned long long)mw_i);
        atomicAdd(&g_rtc_cyc[5], (unsigned long long)mw_a);
        atomicAdd(&g_rtc_cyc[8], (unsigned long long)k);
      }
    }
  } else {
    // ===== epilogue warps.  Group g = warp / 8 handles the tiles k with k % 2 == g (TMEM buffer
    // g): while one group reads its accumulators (TMEM-read bound) the other one computes, so
    // the two phases overlap.  Warp w drains TMEM lanes 32 (w % 4).. (its 32 rows) x the 16
    // columns 16 ((w / 4) % 2).. of its tiles; W comes through a private cp.async ring.
    const int q4 = warp & 3, half = (warp >> 2) & 1, grp = warp >> 3;
    const int rl = 32 * q4 + lane;                     // row within the block (TMEM lane)
    const int WR = a.wring;
    TW *ring = Wr + (size_t)warp * WR * 16 * 32;
    const uint32_t lane_addr = tmem + ((uint32_t)(32 * q4) << 16) + (uint32_t)(16 * half);
    const TW *Wg = reinterpret_cast<const TW *>(a.w);
    constexpr int PER = 16 / (int)sizeof(TW);          // elements per 16-byte chunk
    int64_t k = 0;
    long long ew_t = 0, ew_ld = 0, ew_w = 0, ew_all = RTC_CLK();
    for (int64_t it = blockIdx.x; it < a.items; it += gridDim.x) {
      int64_t b, rb, c0, c1;
      item_of(it, b, rb, c0, c1);
      if (a.status && a.status[b] != LRA_OK) continue;
      const TW *W = Wg + b * a.w_stride;
      const int64_t row0 = rb * BM;
      const int64_t gi = row0 + rl;
      // scale of R in 2^(ea_i + fb_tile + es): es = -35 - 7 (S = 6) / -35 + 7 (S = 3); exponent
      // field of the double built directly (rows / columns outside the problem carry -4000)
      const int eai = (gi < a.m ? a.sa[b * a.m + gi] : -4000) + (S == 6 ? -42 : -28) + 1023;
      const int *sbcol = a.sbq + b * a.CB * BN;
      const bool vec_ok = ((a.ldw * (int64_t)sizeof(TW)) % 16 == 0) && ((reinterpret_cast<uintptr_t>(W) & 15) == 0) &&
                          row0 + BM <= a.m;
      // the tiles of this group inside the item: global tile counter k + (ct - c0) must match grp
      const int64_t first = c0 + (int64_t)(((k & 1) != grp) ? 1 : 0);
      auto load_w = [&](int64_t ct, int slot) {
        TW *dst = ring + slot * 16 * 32;
        const int64_t cb0 = ct * BN + 16 * half;
        if (vec_ok && cb0 + 16 <= a.n) {
          for (int e = lane; e < 16 * 32 / PER; e += 32) {
            const int c = e / (32 / PER), r4 = (e % (32 / PER)) * PER;
            cp16(dst + c * 32 + r4, W + (cb0 + c) * a.ldw + row0 + 32 * q4 + r4);
          }
        } else {
          for (int c = 0; c < 16; ++c) {
            const int64_t gj = cb0 + c;
            dst[c * 32 + lane] = (gi < a.m && gj < a.n) ? W[gj * a.ldw + gi] : (TW)0;
          }
        }
      };
      int slot_ld = 0, slot_use = 0;
      for (int j = 0; j < WR - 1; ++j) {
        const int64_t ct = first + 2 * j;
        if (ct < c1) load_w(ct, slot_ld);
        cp_commit();
        slot_ld = (slot_ld + 1) % WR;
      }
      double num = 0.0, den = 0.0;
      int sb_next = first < c1 ? __ldg(sbcol + first * BN) : 0;   // column scale, one tile ahead
      for (int64_t ct = first; ct < c1; ct += 2) {
        const int64_t kk = k + (ct - c0);               // global tile counter (parity == grp)
        const int sb_cur = sb_next;
        if (ct + 2 < c1) sb_next = __ldg(sbcol + (ct + 2) * BN);
        {
          const int64_t cn = ct + 2 * (WR - 1);
          if (cn < c1) load_w(cn, slot_ld);
          cp_commit();
          slot_ld = (slot_ld + 1) % WR;
        }
        const int tb = (int)(kk & 1);
        const int ex = eai + sb_cur;                    // scale of this tile
        const double sc = ex > 0 ? __hiloint2double(ex << 20, 0) : 0.0;
        long long te0 = RTC_CLK();
        mbar_wait(B_TFULL + 8 * tb, (uint32_t)((kk >> 1) & 1));
        long long te1 = RTC_CLK();
        ew_t += te1 - te0;
        asm volatile("tcgen05.fence::after_thread_sync;\n" ::: "memory");
        if (WR == 3) cp_wait2(); else cp_wait1();
        __syncwarp();
        const TW *wt = ring + slot_use * 16 * 32;
        slot_use = (slot_use + 1) % WR;
#pragma unroll
        for (int cc = 0; cc < 16; cc += 8) {
          uint32_t P[S][8];
#pragma unroll
          for (int l = 0; l < S; ++l)
            asm volatile("tcgen05.ld.sync.aligned.32x32b.x8.b32 {%0,%1,%2,%3,%4,%5,%6,%7}, [%8];\n"
                         : "=r"(P[l][0]), "=r"(P[l][1]), "=r"(P[l][2]), "=r"(P[l][3]), "=r"(P[l][4]), "=r"(P[l][5]),
                           "=r"(P[l][6]), "=r"(P[l][7])
                         : "r"(lane_addr + (uint32_t)(tb * 192 + l * BN + cc)));
          asm volatile("tcgen05.wait::ld.sync.aligned;\n" ::: "memory");
#pragma unroll
          for (int l = 0; l < S; ++l)   // register dependence on the wait: no use before it
            asm volatile("" : "+r"(P[l][0]), "+r"(P[l][1]), "+r"(P[l][2]), "+r"(P[l][3]), "+r"(P[l][4]),
                         "+r"(P[l][5]), "+r"(P[l][6]), "+r"(P[l][7]));
          if (cc == 8) {   // both chunks read: release the TMEM buffer to the MMA warp
            asm volatile("tcgen05.fence::before_thread_sync;\n" ::: "memory");
            __syncwarp();
            if (lane == 0) mbar_arrive(B_TEMPTY + 8 * tb);
          }
          ew_ld += RTC_CLK() - te1;
#if RTC_EPI_LDONLY
          {
            unsigned acc = 0;
#pragma unroll
            for (int x = 0; x < 8; ++x)
#pragma unroll
              for (int l = 0; l < S; ++l) acc ^= P[l][x];
            num += (double)acc;
          }
          if (false)
#endif
#pragma unroll
          for (int x = 0; x < 8; ++x) {
            const double w = (double)wt[(cc + x) * 32 + lane];
            // R = sum_l P_l 2^(7 (S-1-l)) exactly in int64 (the last level's low 7 bits dropped
            // for S = 6: < 2^-47 of the scale, below the 2^-42 truncation)
            long long R;
            if (S == 6) {
              const int lo = (int)P[3][x] * 128 + (int)P[4][x] + ((int)P[5][x] >> 7);
              R = (long long)(int)P[2][x] * 16384 + lo;
              R += (long long)(int)P[1][x] * 2097152;
              R += (long long)(int)P[0][x] * 268435456;
            } else {
              R = (long long)((int)P[0][x] * 128 + (int)P[1][x]) * 128 + (int)P[2][x];
            }
            const double ab = i64_to_f64(R);
            const double d = fma(-ab, sc, w);
            num = fma(d, d, num);
            den = fma(w, w, den);
          }
        }
      }
      k += c1 - c0;
      cp_wait0();
      // item partial: sum over the epilogue warps (fixed order) -> partial[item]
      num = warp_sum(num);
      den = warp_sum(den);
      __shared__ double red[2][NEPI];
      if (lane == 0) {
        red[0][warp] = num;
        red[1][warp] = den;
      }
      asm volatile("bar.sync 1, %0;\n" ::"n"(NEPI * 32) : "memory");
      if (warp == 0 && lane == 0) {
        double s0 = 0.0, s1 = 0.0;
        for (int w = 0; w < NEPI; ++w) {
          s0 += red[0][w];
          s1 += red[1][w];
        }
        const int64_t rem = it % (a.RB * a.nchunk);
        a.partial[b * a.RB * a.nchunk + rem] = make_double2(s0, s1);
      }
      asm volatile("bar.sync 1, %0;\n" ::"n"(NEPI * 32) : "memory");
    }
    if (warp == 0 && lane == 0) {
      atomicAdd(&g_rtc_cyc[6], (unsigned long long)ew_t);
      atomicAdd(&g_rtc_cyc[7], (unsigned long long)(RTC_CLK() - ew_all - ew_t));
      atomicAdd(&g_rtc_cyc[9], (unsigned long long)ew_ld);
      atomicAdd(&g_rtc_cyc[10], (unsigned long long)ew_w);
    }
  }
  asm volatile("tcgen05.fence::before_thread_sync;\n" ::: "memory");
  __syncthreads();
  if (warp == NEPI + 1) {
    asm volatile("tcgen05.fence::after_thread_sync;\n" ::: "memory");
    asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, 512;\n" ::"r"(tmem));
  }
}

}  // namespace rtc

size_t residual_tc_scratch(int64_t m, int64_t n, int r, int S, int64_t nb) {
  const int KB = (r + rtc::BK - 1) / rtc::BK;
  const int64_t RB = (m + rtc::BM - 1) / rtc::BM, CB = (n + rtc::BN - 1) / rtc::BN;
  return (size_t)nb * (RB * KB * S * rtc::A_TILE + CB * KB * S * rtc::B_TILE + (m + CB * rtc::BN) * 8) + 1024;
}

static int tc_tpi(int64_t CB) { return CB >= 64 ? 16 : (CB >= 8 ? 8 : (int)CB); }

int64_t residual_tc_partials(int64_t m, int64_t n) {
  const int64_t RB = (m + rtc::BM - 1) / rtc::BM, CB = (n + rtc::BN - 1) / rtc::BN;
  const int tpi = tc_tpi(CB);
  return RB * ((CB + tpi - 1) / tpi);
}

static int num_sms_rtc() {
  static int n = 0;
  if (!n) {
    int dev = 0;
    cudaGetDevice(&dev);
    cudaDeviceGetAttribute(&n, cudaDevAttrMultiProcessorCount, dev);
  }
  return n;
}

// Tensor-core residual for nb problems (ResArgs as for k_residual).  S digit slices per
// operand (6: PRECISE, 3: FAST).  scratch: residual_tc_scratch bytes; a.partial must hold
// residual_tc_partials(m, n) entries per problem.
cudaError_t launch_residual_tc(ResArgs a, int64_t nb, int S, void *scratch, double *num2, double *den2,
                               cudaStream_t st, int *nlaunch, Prof *pf) {
  using namespace rtc;
  const int KB = (a.r + BK - 1) / BK;
  const int64_t RB = (a.m + BM - 1) / BM, CB = (a.n + BN - 1) / BN;
  char *p = reinterpret_cast<char *>((((uintptr_t)scratch) + 255) & ~(uintptr_t)255);
  signed char *Aq = reinterpret_cast<signed char *>(p);
  p += (size_t)nb * RB * KB * S * A_TILE;
  signed char *Bq = reinterpret_cast<signed char *>(p);
  p += (size_t)nb * CB * KB * S * B_TILE;
  p = reinterpret_cast<char *>(((uintptr_t)p + 15) & ~(uintptr_t)15);
  int *sa = reinterpret_cast<int *>(p);
  int *sbq = sa + nb * a.m;
  sbq = reinterpret_cast<int *>(((uintptr_t)sbq + 15) & ~(uintptr_t)15);
  pf->begin("k_split", st);
  static const bool split_old = getenv("LRA_SPLIT_OLD") != nullptr;   // the two-kernel split (diagnostics)
  if (split_old || KB > 2) {
    k_split_a<<<dim3((unsigned)(4 * RB), (unsigned)nb), 64, 0, st>>>(a.A, a.m, a.r, a.a_stride, S, KB, Aq, sa, a.status);
    k_split_b<<<dim3((unsigned)CB, (unsigned)nb), 2 * BN, 0, st>>>(a.B, a.n, a.r, a.b_stride, S, KB, Bq, sbq, a.status);
  } else {
    const dim3 g((unsigned)(RB + (CB + 3) / 4), (unsigned)nb);
    if (KB == 1)
      k_split_ab<1><<<g, 128, 0, st>>>(a.A, a.B, a.m, a.n, a.r, a.a_stride, a.b_stride, S, RB, CB, Aq, Bq, sa, sbq, a.status);
    else
      k_split_ab<2><<<g, 128, 0, st>>>(a.A, a.B, a.m, a.n, a.r, a.a_stride, a.b_stride, S, RB, CB, Aq, Bq, sa, sbq, a.status);
  }
  pf->end(st);
  cudaError_t e = cudaGetLastError();
  if (e != cudaSuccess) return e;
  TcArgs t{};
  t.dtype = a.dtype;
  t.m = a.m;
  t.n = a.n;
  t.ldw = a.ldw;
  t.w_stride = a.w_stride;
  t.w = a.w;
  t.Aq = Aq;
  t.Bq = Bq;
  t.sa = sa;
  t.sbq = sbq;
  t.S = S;
  t.KB = KB;
  t.RB = RB;
  t.CB = CB;
  t.tpi = tc_tpi(CB);
  t.nchunk = (CB + t.tpi - 1) / t.tpi;
  t.items = nb * RB * t.nchunk;
  t.partial = a.partial;
  t.status = a.status;
  // shared memory: 2 A buffers + nst B stages + the per-warp W rings; shrink the B stages and
  // then the W ring until it fits (r > 32 needs two K blocks)
  const size_t elt = a.dtype == LRA_F32 ? 4 : 8;
  const size_t limit = 227 * 1024 - 2048;
  t.nst = NST;
  t.wring = WRING;
  auto smem_of = [&](int nst, int wr) {
    return 2 * (size_t)S * KB * A_TILE + (size_t)nst * S * KB * B_TILE + (size_t)NEPI * wr * 16 * 32 * elt;
  };
  while (smem_of(t.nst, t.wring) > limit && t.nst > 3) --t.nst;
  if (smem_of(t.nst, t.wring) > limit) t.wring = 2;
  while (smem_of(t.nst, t.wring) > limit && t.nst > 2) --t.nst;
  if (smem_of(t.nst, t.wring) > limit) return cudaErrorInvalidConfiguration;
  const size_t smem = smem_of(t.nst, t.wring);
  const int64_t grid = t.items < num_sms_rtc() ? t.items : num_sms_rtc();
  pf->begin("k_residual_tc", st);
  void (*kern)(TcArgs) = a.dtype == LRA_F32 ? (S == 6 ? k_residual_tc<float, 6> : k_residual_tc<float, 3>)
                                             : (S == 6 ? k_residual_tc<double, 6> : k_residual_tc<double, 3>);
  if (S != 3 && S != 6) return cudaErrorInvalidValue;
  e = cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
  if (e == cudaSuccess) kern<<<(unsigned)grid, NTC, smem, st>>>(t);
  pf->end(st);
  if (e != cudaSuccess) return e;
  if ((e = cudaGetLastError()) != cudaSuccess) return e;
  *nlaunch += 3;
  return launch_reduce(a.partial, RB * t.nchunk, nb, num2, den2, a.status, st, nlaunch, pf);
}

}  // namespace lra

namespace lra {
cudaError_t read_rtc_counters(unsigned long long *out, bool reset) {
  cudaError_t e = cudaMemcpyFromSymbol(out, g_rtc_cyc, sizeof(g_rtc_cyc));
  if (e == cudaSuccess && reset) {
    unsigned long long z[16] = {0};
    e = cudaMemcpyToSymbol(g_rtc_cyc, z, sizeof(z));
  }
  return e;
}
}  // namespace lra
