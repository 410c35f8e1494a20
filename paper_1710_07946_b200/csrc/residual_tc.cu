// residual_tc.cu — the a-posteriori check rho = ||W - CUR||_F / ||W||_F (eq. eqcur0,
// P:1153-1155) with the rank-r product CUR = A*B on the 5th-generation tensor cores.
//
// A (m x r) and B (r x n) are fp64.  Their product must be accurate far beyond fp32
// (config 2: rho ~ 7e-7, so W - AB cancels ~21 bits), so the contraction is
// done exactly in integers (Ozaki-style splitting) with balanced base-256 digits:
//   A[i,t] = 2^ea_i * sum_s a_s[i,t] 256^-(s+1),   B[t,j] = 2^fb_J * sum_u b_u[t,j] 256^-(u+1),
// a_s, b_u in [-128, 127] (int8), one exponent per row of A and one per BN-column tile J of B.
// The digits come from the integer X = rint(x 2^(8S)) of the normalised value |x| < 127/256
// (so the top digit stays in range), peeled from the bottom: d = ((X + 128) mod 256) - 128.
// The digit products with s + u <= S-1 (S = 6 PRECISE, S = 3 FAST; tools/digits_precision.py:
// S = 6 puts rho within ~1e-8 of the exact fp64 product on configs 2, 3 and the ragged test
// shapes, ~30x closer than the round-1 base-128 split) are accumulated per level l = s + u
// EXACTLY in int32 by tcgen05.mma kind::i8 (|P_l| <= (l+1) r 2^14 < 2^31 for r <= 128) into
// TMEM; the epilogue recombines the levels in fp64 (int32 -> fp64 by the 2^52 + 2^31 magic add)
//   PRECISE: R = 2^16 (256 P0 + P1) + (256 P2 + P3) + floor(P4 / 2^8) + floor(P5 / 2^16),
//            AB = R 2^(ea + fb - 40)   (the floors cost < 2^-43 of the largest |R|)
//   FAST:    R = 2^16 P0 + (256 P1 + P2),  AB = R 2^(ea + fb - 32)
// (R exact in int64, |R| < 2^51, converted by the 2^52 + 2^51 magic add) and accumulates
// (W - AB)^2 and W^2 in fp64.
//
// k_split_ab writes the digit slices in the UMMA canonical K-major no-swizzle layout (core
// matrix = 8 rows x 16 bytes; LBO = 128 B between the two K halves, SBO = 256 B between 8-row
// groups).  k_resid: persistent (one CTA per SM), warp-specialised:
//   producer warp  — bulk copies (cp.async.bulk + mbarrier transaction counts) of the A slices
//                    of each work item and the B slices of each tile; the W tile (128 rows x BN
//                    columns) by one TMA tensor copy (cp.async.bulk.tensor.3d over (m, n, batch),
//                    zero fill beyond the edges), into rings of stages;
//   MMA warp       — stages A into TMEM (tcgen05.cp, TS-mode MMAs; A stays in shared memory,
//                    SS mode, when r > 64 leaves too few TMEM columns), issues the S(S+1)/2 x KB
//                    MMAs of a tile into one of NBUF TMEM accumulator buffers, commits;
//   16 epilogue warps in 4 groups — group g drains the tiles k with k % 4 == g (tcgen05.ld
//                    32x32b.x8 per level), reads W from the shared-memory stage, accumulates.
// Work item = (problem, 128-row block, chunk of TPI tiles); one partial per item (the 16 warps'
// sums added in warp order), reduced in a fixed order by k_reduce (deterministic).
#include "kernels.cuh"

#include <cuda.h>
#include <cudaTypedefs.h>

#include <cstdlib>
#include <mutex>

namespace lra {
// phase counters (clock64 cycles summed over CTAs): 0 MMA wait B, 1 MMA wait TMEM, 2 MMA issue,
// 3 producer wait B stage, 4 producer wait A, 5 MMA wait A, 6 epilogue wait TMEM (warp 0),
// 7 epilogue work (warp 0), 8 tiles (count), 9 epilogue wait W (warp 0), 10 producer wait W
__device__ unsigned long long g_rtc_cyc[16];
#ifndef RTC_PROF
#define RTC_PROF 0      // 1: per-role clock64 counters (lra_debug_counters_residual)
#endif
#define RTC_CLK() (RTC_PROF ? clock64() : 0ll)
namespace rtc {

constexpr int BM = 128;        // rows per CTA (MMA M)
constexpr int BK = 32;         // K per MMA (kind::i8)
constexpr int A_TILE = BM * BK;          // bytes of one (slice, K-block) A tile  (4096)
constexpr int NE = 16;                   // epilogue warps (G groups of NE / G)
constexpr int NWS = 8;                   // max W stages (a.nws: as many as fit in shared memory)
constexpr int NBS = 8;                   // B-slice stages
constexpr int NBMAX = 4;                 // max TMEM accumulator buffers

template <int S> struct Tr;
// Per mode: tile width BN (= MMA N), tiles per work item, TMEM accumulator buffers (S x BN
// columns each), MMA-issuing warps and the warp that issues each digit level, epilogue groups G
// (group g drains the tiles k with k % G == g, so one group's TMEM loads overlap another
// group's arithmetic).  One thread issues
// a tcgen05.mma every ~54 cycles (tools/mma_issue_bench.cu: one issuer 54 cycles per MMA, four
// issuers reach the M=128 N=32 math floor of 16), so the S(S+1)/2 products of a tile are spread
// over several warps by level: PRECISE levels {0,1,2,3} {4,5} = 10, 11 products (20 warps in
// all, a multiple of 4, keep 96 registers per thread for the epilogue).
#ifndef RTC_PREC_EARLY
#define RTC_PREC_EARLY 1  // PRECISE: drain TMEM, release, then the fp64 work
#endif
#ifndef RTC_PREC_G
#define RTC_PREC_G 1      // epilogue groups, PRECISE (one buffer: all 16 warps drain each tile)
#endif
#ifndef RTC_PREC_BN
#define RTC_PREC_BN 64    // PRECISE tile width and accumulator buffers (6 levels x BN columns each):
                          // 64 columns with ONE buffer (384 TMEM columns) halves the MMAs per byte
                          // of W against 32 x 2 buffers; the early drain releases the buffer before
                          // the fp64 work (16384^2 334 -> 320 us, config-2 bench +1.4 %)
#endif
#ifndef RTC_PREC_SMEM_KB
#define RTC_PREC_SMEM_KB 140
#endif
#ifndef RTC_PREC_NBUF
#define RTC_PREC_NBUF 1
#endif
#ifndef RTC_FAST_G
#define RTC_FAST_G 2      // epilogue groups, FAST
#endif
template <> struct Tr<6> {
  static constexpr int BN = RTC_PREC_BN, TPI = 512 / RTC_PREC_BN, NBUF = RTC_PREC_NBUF, NMW = 2, G = RTC_PREC_G, XW = 8;
  static constexpr bool EARLY = RTC_PREC_EARLY;
  static constexpr int warp_of(int l) { return l <= 3 ? 0 : 1; }
  // shared-memory budget: PRECISE runs inside lra_batch next to the nucleus / factor CTAs of
  // other groups, and a 200 KB CTA keeps them off its SM (config-2 bench 9395 -> 8393)
  static constexpr size_t SMEM_CAP = (size_t)RTC_PREC_SMEM_KB * 1024;
};
#ifndef RTC_FAST_BN
#define RTC_FAST_BN 64    // FAST tile width (diagnostic builds: 32 with 4 accumulator buffers)
#endif
#ifndef RTC_FAST_EARLY
#define RTC_FAST_EARLY 0
#endif
#ifndef RTC_FAST_NBUF
#define RTC_FAST_NBUF 2
#endif
template <> struct Tr<3> {
  static constexpr int BN = RTC_FAST_BN, TPI = 512 / RTC_FAST_BN, NBUF = RTC_FAST_NBUF, NMW = 2, G = RTC_FAST_G, XW = 8;
  static constexpr bool EARLY = RTC_FAST_EARLY;
  static constexpr int warp_of(int l) { return l <= 1 ? 0 : 1; }
  static constexpr size_t SMEM_CAP = 227 * 1024 - 4096;
};
template <int S> constexpr int nthreads() { return 32 * (NE + 2 + Tr<S>::NMW); }

__device__ __forceinline__ uint32_t smem_u32(const void *p) { return (uint32_t)__cvta_generic_to_shared(p); }

__device__ __forceinline__ unsigned long long wmax_bits(unsigned long long k) {   // max over the warp
  const unsigned hi = (unsigned)(k >> 32);
  const unsigned mhi = __reduce_max_sync(0xffffffffu, hi);
  const unsigned mlo = __reduce_max_sync(0xffffffffu, hi == mhi ? (unsigned)k : 0u);
  return ((unsigned long long)mhi << 32) | mlo;
}

// exponent e with mx 2^-e < 127/256 (the top balanced base-256 digit then stays in [-128, 127])
__device__ __forceinline__ int scale_exp(double mx) {
  if (!(mx > 0.0)) return 0;
  int e = ilogb(mx) + 2;                     // mx 2^-e in [1/4, 1/2)
  if (ldexp(mx, -e) >= 127.0 / 256.0) ++e;
  return e;
}

// balanced base-256 digits (most significant first) of x with |x| < 127/256, S digits
template <int S>
__device__ __forceinline__ void digits256(double x, int (&d)[S]) {
  long long X = __double2ll_rn(ldexp(x, 8 * S));
#pragma unroll
  for (int s = S - 1; s >= 1; --s) {
    const long long q = ((X + 128) & 255) - 128;
    d[s] = (int)q;
    X = (X - q) >> 8;
  }
  d[0] = (int)X;
}

// One launch for both factors (grid.x = RB + ceil(CB / (128 / BN)), grid.y = nb, 128 threads),
// every input value loaded once into registers:
//  - A CTAs: thread = one row of a 128-row block; the row exponent from its r values;
//  - B CTAs: thread = one column, BN consecutive threads = one tile; the tile exponent is the max
//    over the tile's columns.
template <int KBT, int S, int BN>
__global__ void __launch_bounds__(128) k_split_ab(const double *A, const double *B, int64_t m, int64_t n, int r,
                                                  int64_t a_stride, int64_t b_stride, int64_t RB, int64_t CB,
                                                  signed char *Aq, signed char *Bq, int *sa, int *sbq,
                                                  const int32_t *status) {
  constexpr int RT = KBT * BK;                 // values per thread (zero beyond r)
  const int64_t b = blockIdx.y;
  const bool live = !(status && status[b] != LRA_OK);
  // r > 32: two passes over the thread's values — the maximum first, then the digits K block by
  // K block (re-read from L1/L2) — so only 32 values are held at a time and r = 64 / 128 keep the
  // occupancy of r = 32 (32768^2 r = 64: 53 -> 41 us).  r <= 32 keeps its values from the one pass.
  const double *src;
  int64_t step;                                // stride between consecutive values t
  bool ok;
  double mx = 0.0;
  double keep[KBT == 1 ? BK : 1];              // r <= 32: the one pass keeps its values
  signed char *base;
  int boff;
  int tile_bytes;
  if ((int64_t)blockIdx.x < RB) {
    const int64_t rb = blockIdx.x;
    const int i = threadIdx.x;
    const int64_t gi = rb * BM + i;
    ok = live && gi < m;
    src = A + b * a_stride + gi;
    step = m;
#pragma unroll 8
    for (int t = 0; t < RT; ++t) {
      const double x = (ok && t < r) ? __ldg(src + (int64_t)t * step) : 0.0;
      if constexpr (KBT == 1) keep[t] = x;
      mx = fmax(mx, fabs(x));
    }
    const int e = scale_exp(mx);
    if (gi < m) sa[b * m + gi] = ok ? e : -4000;     // -4000: row contributes nothing
    mx = (double)e;                                  // the exponent travels in mx below
    base = Aq + (size_t)(b * RB + rb) * KBT * S * A_TILE;
    boff = (i >> 3) * 256 + (i & 7) * 16;
    tile_bytes = A_TILE;
  } else {
    constexpr int TPC = 128 / BN;             // tiles per CTA
    const int64_t cb = ((int64_t)blockIdx.x - RB) * TPC + threadIdx.x / BN;
    const int jj = threadIdx.x % BN;
    const int64_t gj = cb * BN + jj;
    ok = live && cb < CB && gj < n;
    src = B + b * b_stride + gj * r;
    step = 1;
#pragma unroll 8
    for (int t = 0; t < RT; ++t) {
      const double x = (ok && t < r) ? __ldg(src + t) : 0.0;
      if constexpr (KBT == 1) keep[t] = x;
      mx = fmax(mx, fabs(x));
    }
    // tile max: within the warp for BN <= 32, through shared memory for BN = 64 (two warps)
#pragma unroll
    for (int o = (BN < 32 ? BN : 32) / 2; o > 0; o >>= 1) mx = fmax(mx, __shfl_xor_sync(0xffffffffu, mx, o));
    if (BN > 32) {
      __shared__ double wm[4];
      if ((threadIdx.x & 31) == 0) wm[threadIdx.x >> 5] = mx;
      __syncthreads();
      const int w0 = (threadIdx.x >> 5) & ~(BN / 32 - 1);
      for (int w = 0; w < BN / 32; ++w) mx = fmax(mx, wm[w0 + w]);
    }
    const int e = scale_exp(mx);
    if (cb >= CB) return;
    if (jj == 0) sbq[b * CB + cb] = ok ? e : -4000;
    mx = (double)e;
    base = Bq + (size_t)(b * CB + cb) * KBT * S * (BN * BK);
    boff = (jj >> 3) * 256 + (jj & 7) * 16;
    tile_bytes = BN * BK;
  }
  const int e = (int)mx;
  // digits of all values, packed 16 bytes per (kb, K half, slice)
#pragma unroll 1
  for (int kb = 0; kb < KBT; ++kb) {
    double v[BK];
#pragma unroll
    for (int t = 0; t < BK; ++t) {
      const int tt = kb * BK + t;
      if constexpr (KBT == 1) v[t] = ldexp(keep[t], -e);
      else v[t] = ldexp((ok && tt < r) ? __ldg(src + (int64_t)tt * step) : 0.0, -e);
    }
#pragma unroll
    for (int h = 0; h < 2; ++h) {
      uint32_t w[S][4];
#pragma unroll
      for (int kk = 0; kk < 16; ++kk) {
        int d[S];
        digits256<S>(v[h * 16 + kk], d);
#pragma unroll
        for (int s = 0; s < S; ++s) {
          const uint32_t byte = ((uint32_t)d[s] & 0xffu) << (8 * (kk & 3));
          if ((kk & 3) == 0) w[s][kk >> 2] = byte;
          else w[s][kk >> 2] |= byte;
        }
      }
#pragma unroll
      for (int s = 0; s < S; ++s)
        *reinterpret_cast<uint4 *>(base + (size_t)(kb * S + s) * tile_bytes + boff + h * 128) =
            make_uint4(w[s][0], w[s][1], w[s][2], w[s][3]);
    }
  }
}

__device__ __forceinline__ uint64_t smem_desc(uint32_t addr) {
  // K-major, no swizzle: LBO = 128 B (K halves), SBO = 256 B (8-row groups), version 1 (sm100)
  return (uint64_t)((addr & 0x3FFFF) >> 4) | ((uint64_t)(128 >> 4) << 16) | ((uint64_t)(256 >> 4) << 32) |
         (1ull << 46);
}
// kind::i8, D = s32, A = B = signed 8-bit, both K-major, M = 128, N = BN
template <int BN>
struct Idesc {
  static constexpr uint32_t v = (2u << 4) | (1u << 7) | (1u << 10) | ((uint32_t)(BN >> 3) << 17) | ((uint32_t)(BM >> 4) << 24);
};
// A operand from TMEM (TS mode): A 128 x 32 int8 at TMEM columns [a_tmem, a_tmem + 8)
__device__ __forceinline__ void mma_i8_ts(uint32_t tmem_d, uint32_t a_tmem, uint64_t bdesc, uint32_t idesc,
                                          uint32_t acc) {
  asm volatile(
      "{\n\t.reg .pred p;\n\t"
      "setp.ne.b32 p, %4, 0;\n\t"
      "tcgen05.mma.cta_group::1.kind::i8 [%0], [%1], %2, %3, p;\n\t}\n" ::"r"(tmem_d),
      "r"(a_tmem), "l"(bdesc), "r"(idesc), "r"(acc));
}
// both operands from shared memory (SS mode; r > 64)
__device__ __forceinline__ void mma_i8_ss(uint32_t tmem_d, uint64_t adesc, uint64_t bdesc, uint32_t idesc, uint32_t acc) {
  asm volatile(
      "{\n\t.reg .pred p;\n\t"
      "setp.ne.b32 p, %4, 0;\n\t"
      "tcgen05.mma.cta_group::1.kind::i8 [%0], %1, %2, %3, p;\n\t}\n" ::"r"(tmem_d),
      "l"(adesc), "l"(bdesc), "r"(idesc), "r"(acc));
}
// W tile (128 rows x BN columns of problem b) by TMA: box (128, BN, 1) of the (m, n, nb) tensor
__device__ __forceinline__ void tma_w(uint32_t dst, const CUtensorMap *tm, int row0, int col0, int b, uint32_t mbar) {
  asm volatile(
      "cp.async.bulk.tensor.3d.shared::cluster.global.tile.mbarrier::complete_tx::bytes [%0], [%1, {%2, %3, %4}], [%5];\n" ::"r"(dst),
      "l"(reinterpret_cast<uint64_t>(tm)), "r"(row0), "r"(col0), "r"(b), "r"(mbar)
      : "memory");
}
// int32 -> fp64 exactly by the 2^52 + 2^31 magic add (one LOP + one DADD instead of an I2F)
__device__ __forceinline__ double i2d(int x) {
  return __hiloint2double(0x43300000, x ^ (int)0x80000000) - 4503601774854144.0;
}
// smem (canonical K-major tile, 128 rows x 32 bytes) -> TMEM 128 lanes x 8 columns
__device__ __forceinline__ void tmem_cp_128x256b(uint32_t taddr, uint64_t sdesc) {
  asm volatile("tcgen05.cp.cta_group::1.128x256b [%0], %1;\n" ::"r"(taddr), "l"(sdesc) : "memory");
}
__device__ __forceinline__ void mma_commit(uint32_t mbar) {
  asm volatile("tcgen05.commit.cta_group::1.mbarrier::arrive::one.shared::cluster.b64 [%0];\n" ::"r"(mbar) : "memory");
}
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
// Wait for the phase with the given parity to complete.  The suspend-time hint lets the hardware
// park the waiting warp until the phase completes instead of re-issuing try_wait in a loop, so
// waiting warps do not take issue slots from the working ones (ncu: the spin loop was the top
// stall site of the epilogue).
__device__ __forceinline__ void mbar_wait(uint32_t addr, uint32_t phase) {
  uint32_t done = 0;
  do {
    asm volatile(
        "{\n\t.reg .pred p;\n\t"
        "mbarrier.try_wait.parity.shared::cta.b64 p, [%1], %2, %3;\n\t"
        "selp.u32 %0, 1, 0, p;\n\t}\n"
        : "=r"(done)
        : "r"(addr), "r"(phase), "r"(0x989680u)
        : "memory");
  } while (!done);
}

__device__ __forceinline__ bool elect_one() {
  uint32_t pred = 0;
  asm volatile("{\n\t.reg .pred P;\n\telect.sync _|P, 0xffffffff;\n\tselp.u32 %0, 1, 0, P;\n\t}\n" : "=r"(pred));
  return pred != 0;
}

struct TcArgs {
  int64_t m, n, ldw, w_stride;
  const void *w;
  const signed char *Aq, *Bq;
  const int *sa, *sbq;             // per-row / per-tile scale exponents
  int KB;
  int64_t RB, CB;                 // row blocks, BN-column tiles per problem
  int64_t nchunk;                 // column chunks (items) per row block
  int tpi;                        // tiles per item (a multiple of Tr<S>::TPI, see launch_residual_tc)
  int64_t items;                  // nb * RB * nchunk
  int nabuf;                      // TMEM A regions (2: double-buffered across items, 1: single)
  int nas;                        // shared-memory A buffers (TS mode: 1 — A leaves for TMEM at once; SS: 2)
  int nws;                        // W stages (<= NWS)
  int nbs;                        // B-slice stages (<= NBS)
  double2 *partial;               // per problem: RB * nchunk partials (one per work item)
  const int32_t *status;
};

struct Bars {
  unsigned long long wfull[NWS], wempty[NWS], bfull[NBS], bempty[NBS], tfull[NBMAX], tempty[NBMAX], afull[2],
      aempty[2], astaged[2], aread[2];
};

// levels 0 .. S-1 of XW (4 or 8) consecutive accumulator columns, 32 lanes (32x32b shape)
template <int S, int BN, int XW>
__device__ __forceinline__ void tmem_ld(uint32_t addr, uint32_t (&P)[S][XW]) {
#pragma unroll
  for (int l = 0; l < S; ++l) {
    if constexpr (XW == 8)
      asm volatile("tcgen05.ld.sync.aligned.32x32b.x8.b32 {%0,%1,%2,%3,%4,%5,%6,%7}, [%8];\n"
                   : "=r"(P[l][0]), "=r"(P[l][1]), "=r"(P[l][2]), "=r"(P[l][3]), "=r"(P[l][4]), "=r"(P[l][5]),
                     "=r"(P[l][6]), "=r"(P[l][7])
                   : "r"(addr + (uint32_t)(l * BN)));
    else
      asm volatile("tcgen05.ld.sync.aligned.32x32b.x4.b32 {%0,%1,%2,%3}, [%4];\n"
                   : "=r"(P[l][0]), "=r"(P[l][1]), "=r"(P[l][2]), "=r"(P[l][3])
                   : "r"(addr + (uint32_t)(l * BN)));
  }
}
// register dependence on a tcgen05.wait::ld: no use of P is scheduled before the wait
template <int S, int XW>
__device__ __forceinline__ void reg_dep(uint32_t (&P)[S][XW]) {
#pragma unroll
  for (int l = 0; l < S; ++l)
#pragma unroll
    for (int x = 0; x < XW; ++x) asm volatile("" : "+r"(P[l][x]));
}

// The MMAs of MMA warp MW for one tile: round j issues product j of every level l >= j that the
// warp owns (level l, product (j, l - j)); all offsets are compile-time, so each MMA costs one
// descriptor add (the issue latency of one thread, ~54 cycles per MMA, is the limit).
template <int S, int MW, bool TS, int KB>
__device__ __forceinline__ void issue_tile(uint32_t dbase, uint32_t at, uint64_t adesc, uint64_t bdesc) {
  constexpr int BN = Tr<S>::BN;
  constexpr uint32_t IDESC = Idesc<BN>::v;
  constexpr int B_TILE = BN * BK;
#pragma unroll
  for (int kb = 0; kb < KB; ++kb)
#pragma unroll
    for (int j = 0; j < S; ++j)
#pragma unroll
      for (int l = j; l < S; ++l) {
        if (Tr<S>::warp_of(l) != MW) continue;
        const int u = l - j;
        const uint64_t bd = bdesc + (uint64_t)(((kb * S + u) * B_TILE) >> 4);
        const uint32_t acc = (j | kb) ? 1u : 0u;
        if (TS) mma_i8_ts(dbase + l * BN, at + 8 * (kb * S + j), bd, IDESC, acc);
        else mma_i8_ss(dbase + l * BN, adesc + (uint64_t)(((kb * S + j) * A_TILE) >> 4), bd, IDESC, acc);
      }
}
template <int S, bool TS, int KB>
__device__ __forceinline__ void issue_tile_mw(int mw, uint32_t dbase, uint32_t at, uint64_t adesc, uint64_t bdesc) {
  if (mw == 0) issue_tile<S, 0, TS, KB>(dbase, at, adesc, bdesc);
  else issue_tile<S, 1, TS, KB>(dbase, at, adesc, bdesc);
}

// Persistent, warp-specialized.  Work item = (problem, row block, chunk of TPI tiles).
//   warps 0 .. NE-1   epilogue          warp NE      producer of A (per item) and B (per tile)
//   warp NE + 1       producer of W     warps NE + 2 .. NE + 1 + NMW   MMA issuers (by level)
template <typename TW, int S, bool TS>
__global__ void __launch_bounds__(nthreads<S>(), 1) k_resid(const __grid_constant__ TcArgs a,
                                                           const __grid_constant__ CUtensorMap tmW) {
  constexpr int BN = Tr<S>::BN, NBUF = Tr<S>::NBUF, NMW = Tr<S>::NMW, GG = Tr<S>::G;
  constexpr int B_TILE = BN * BK;
  extern __shared__ __align__(1024) unsigned char smem[];
  __shared__ __align__(8) Bars bar;
  __shared__ uint32_t tmem_base_sh;
  __shared__ double2 red[4][NE];
  __shared__ int red_cnt[4];
  const int KB = a.KB;
  const int tid = threadIdx.x, warp = tid >> 5, lane = tid & 31;
  const int aBytes = S * KB * A_TILE, bBytes = S * KB * B_TILE;
  unsigned char *As = smem;                              // 2 item buffers
  unsigned char *Bst = As + a.nas * aBytes;              // NBS stages
  TW *Wst = reinterpret_cast<TW *>(Bst + a.nbs * bBytes);  // nws stages of BN columns x 128 rows
  const uint32_t bb = smem_u32(&bar);
  const uint32_t B_WFULL = bb + offsetof(Bars, wfull), B_WEMPTY = bb + offsetof(Bars, wempty);
  const uint32_t B_BFULL = bb + offsetof(Bars, bfull), B_BEMPTY = bb + offsetof(Bars, bempty);
  const uint32_t B_TFULL = bb + offsetof(Bars, tfull), B_TEMPTY = bb + offsetof(Bars, tempty);
  const uint32_t B_AFULL = bb + offsetof(Bars, afull), B_AEMPTY = bb + offsetof(Bars, aempty);
  const uint32_t B_ASTG = bb + offsetof(Bars, astaged), B_AREAD = bb + offsetof(Bars, aread);
  const int MW0 = NE + 2;                                // first MMA warp (allocates TMEM)
  if (warp == MW0) {
    asm volatile("tcgen05.alloc.cta_group::1.sync.aligned.shared::cta.b32 [%0], 512;\n" ::"r"(smem_u32(&tmem_base_sh)));
    asm volatile("tcgen05.relinquish_alloc_permit.cta_group::1.sync.aligned;\n");
  }
  if (tid < 4) red_cnt[tid] = 0;
  if (tid == 0) {
    for (int i = 0; i < a.nws; ++i) {
      mbar_init(B_WFULL + 8 * i, 1);
      mbar_init(B_WEMPTY + 8 * i, NE / GG);      // the warps of the consuming group
    }
    for (int i = 0; i < a.nbs; ++i) {
      mbar_init(B_BFULL + 8 * i, 1);
      mbar_init(B_BEMPTY + 8 * i, NMW);
    }
    for (int i = 0; i < NBUF; ++i) {
      mbar_init(B_TFULL + 8 * i, NMW);
      mbar_init(B_TEMPTY + 8 * i, NE / GG);
    }
    for (int i = 0; i < 2; ++i) {
      mbar_init(B_AFULL + 8 * i, 1);
      mbar_init(B_AEMPTY + 8 * i, TS ? 1 : NMW);
      mbar_init(B_ASTG + 8 * i, 1);
      mbar_init(B_AREAD + 8 * i, NMW);
    }
    asm volatile("fence.mbarrier_init.release.cluster;\n" ::: "memory");
  }
  asm volatile("tcgen05.fence::before_thread_sync;\n" ::: "memory");
  __syncthreads();
  asm volatile("tcgen05.fence::after_thread_sync;\n" ::: "memory");
  const uint32_t tmem = tmem_base_sh;
  const uint32_t abase_t = tmem + (uint32_t)(NBUF * S * BN);   // A regions: 8 columns per (kb, slice)
  const uint32_t aregion = (uint32_t)(S * KB * 8);

  const bool small_items = a.items < (1ll << 31);   // 32-bit index arithmetic (64-bit division is ~70 instructions)
  auto item_of = [&](int64_t it, int64_t &b, int64_t &rb, int64_t &c0, int64_t &c1) {
    int64_t ch;
    if (small_items) {
      const uint32_t per = (uint32_t)(a.RB * a.nchunk), i32 = (uint32_t)it, rem = i32 % per;
      b = i32 / per;
      ch = rem / (uint32_t)a.RB;
      rb = rem % (uint32_t)a.RB;
    } else {
      b = it / (a.RB * a.nchunk);
      const int64_t rem = it % (a.RB * a.nchunk);
      ch = rem / a.RB;
      rb = rem % a.RB;
    }
    c0 = ch * a.tpi;
    c1 = min(c0 + (int64_t)a.tpi, a.CB);
  };

  if (warp == NE) {
    // ===== producer of the digit slices: A per item, B per tile (one elected lane issues)
    long long pw_b = 0, pw_a = 0;
    int64_t k = 0, ni = 0;
    for (int64_t it = blockIdx.x; it < a.items; it += gridDim.x) {
      int64_t b, rb, c0, c1;
      item_of(it, b, rb, c0, c1);
      if (a.status && a.status[b] != LRA_OK) continue;
      const int ab = a.nas == 2 ? (int)(ni & 1) : 0;
      long long t0 = RTC_CLK();
      if (ni >= a.nas) mbar_wait(B_AEMPTY + 8 * ab, (uint32_t)(((ni / a.nas) - 1) & 1));
      pw_a += RTC_CLK() - t0;
      ++ni;
      if (elect_one()) {
        mbar_expect(B_AFULL + 8 * ab, (uint32_t)aBytes);
        bulk_g2s(smem_u32(As + ab * aBytes), a.Aq + (size_t)(b * a.RB + rb) * aBytes, (uint32_t)aBytes, B_AFULL + 8 * ab);
      }
      __syncwarp();
      for (int64_t ct = c0; ct < c1; ++ct, ++k) {
        const int bs = (int)(k % a.nbs);
        long long t1 = RTC_CLK();
        if (k >= a.nbs) mbar_wait(B_BEMPTY + 8 * bs, (uint32_t)(((k / a.nbs) - 1) & 1));
        pw_b += RTC_CLK() - t1;
        if (elect_one()) {
          mbar_expect(B_BFULL + 8 * bs, (uint32_t)bBytes);
          bulk_g2s(smem_u32(Bst + bs * bBytes), a.Bq + (size_t)(b * a.CB + ct) * bBytes, (uint32_t)bBytes,
                   B_BFULL + 8 * bs);
        }
        __syncwarp();
      }
    }
    if (RTC_PROF && lane == 0) {
      atomicAdd(&g_rtc_cyc[3], (unsigned long long)pw_b);
      atomicAdd(&g_rtc_cyc[4], (unsigned long long)pw_a);
    }
  } else if (warp == NE + 1) {
    // ===== producer of W: one TMA tensor copy (128 rows x BN columns) per tile
    long long pw_w = 0;
    int64_t k = 0;
    for (int64_t it = blockIdx.x; it < a.items; it += gridDim.x) {
      int64_t b, rb, c0, c1;
      item_of(it, b, rb, c0, c1);
      if (a.status && a.status[b] != LRA_OK) continue;
      const int64_t row0 = rb * BM;
      for (int64_t ct = c0; ct < c1; ++ct, ++k) {
        const int wsg = (int)(k % a.nws);
        long long t1 = RTC_CLK();
        if (k >= a.nws) mbar_wait(B_WEMPTY + 8 * wsg, (uint32_t)(((k / a.nws) - 1) & 1));
        pw_w += RTC_CLK() - t1;
        if (elect_one()) {
          mbar_expect(B_WFULL + 8 * wsg, (uint32_t)(BM * BN * sizeof(TW)));
          tma_w(smem_u32(Wst + (size_t)wsg * BM * BN), &tmW, (int)row0, (int)(ct * BN), (int)b, B_WFULL + 8 * wsg);
        }
        __syncwarp();
      }
    }
    if (RTC_PROF && lane == 0) atomicAdd(&g_rtc_cyc[10], (unsigned long long)pw_w);
  } else if (warp >= MW0) {
    // ===== MMA issuers: warp mw issues the products of its digit levels for every tile (one
    // elected lane).  MMA warp 0 also stages each item's A slices into a TMEM region (TS mode):
    // after every warp's MMAs of the item that last used the region (aread), before any warp's
    // MMAs of the new item (astaged).
    const int mw = warp - MW0;
    long long mw_b = 0, mw_t = 0, mw_i = 0, mw_a = 0;
    int64_t k = 0, ni = 0;
    for (int64_t it = blockIdx.x; it < a.items; it += gridDim.x) {
      int64_t b, rb, c0, c1;
      item_of(it, b, rb, c0, c1);
      if (a.status && a.status[b] != LRA_OK) continue;
      const int ab = a.nas == 2 ? (int)(ni & 1) : 0;            // shared-memory A buffer
      const uint32_t aph = (uint32_t)((ni / a.nas) & 1);
      const int ar = a.nabuf == 2 ? (int)(ni & 1) : 0;          // TMEM A region of this item
      const int64_t use = a.nabuf == 2 ? (ni >> 1) : ni;        // use count of that region
      long long t0 = RTC_CLK();
      if (TS) {
        if (mw == 0) {
          if (use >= 1) mbar_wait(B_AREAD + 8 * ar, (uint32_t)((use - 1) & 1));
          mbar_wait(B_AFULL + 8 * ab, aph);
          asm volatile("tcgen05.fence::after_thread_sync;\n" ::: "memory");
          if (elect_one()) {
            const uint64_t adesc = smem_desc(smem_u32(As + ab * aBytes));
            for (int j = 0; j < KB * S; ++j)
              tmem_cp_128x256b(abase_t + ar * aregion + 8 * j, adesc + (uint64_t)((j * A_TILE) >> 4));
            mma_commit(B_AEMPTY + 8 * ab);          // shared-memory A free once copied
            mma_commit(B_ASTG + 8 * ar);            // the region holds this item's A
          }
          __syncwarp();
        } else {
          mbar_wait(B_ASTG + 8 * ar, (uint32_t)(use & 1));
        }
      } else {
        mbar_wait(B_AFULL + 8 * ab, aph);
      }
      mw_a += RTC_CLK() - t0;
      ++ni;
      const uint64_t adesc = smem_desc(smem_u32(As + ab * aBytes));
      const uint32_t at = abase_t + ar * aregion;
      for (int64_t ct = c0; ct < c1; ++ct, ++k) {
        const int bs = (int)(k % a.nbs), tb = (int)(k % NBUF);
        long long t1 = RTC_CLK();
        mbar_wait(B_BFULL + 8 * bs, (uint32_t)((k / a.nbs) & 1));
        long long t2 = RTC_CLK();
        if (k >= NBUF) mbar_wait(B_TEMPTY + 8 * tb, (uint32_t)(((k / NBUF) - 1) & 1));
        long long t3 = RTC_CLK();
        mw_b += t2 - t1;
        mw_t += t3 - t2;
        asm volatile("tcgen05.fence::after_thread_sync;\n" ::: "memory");
        const uint64_t bdesc = smem_desc(smem_u32(Bst + bs * bBytes));
        const uint32_t dbase = tmem + (uint32_t)(tb * S * BN);
        if (elect_one()) {
          switch (KB) {
            case 1: issue_tile_mw<S, TS, 1>(mw, dbase, at, adesc, bdesc); break;
            case 2: issue_tile_mw<S, TS, 2>(mw, dbase, at, adesc, bdesc); break;
            case 3: issue_tile_mw<S, TS, 3>(mw, dbase, at, adesc, bdesc); break;
            default: issue_tile_mw<S, TS, 4>(mw, dbase, at, adesc, bdesc); break;
          }
          mma_commit(B_BEMPTY + 8 * bs);     // B stage free once these MMAs complete
          mma_commit(B_TFULL + 8 * tb);      // this warp's levels are ready
        }
        __syncwarp();
        mw_i += RTC_CLK() - t3;
      }
      if (elect_one()) {
        if (TS) mma_commit(B_AREAD + 8 * ar);           // this warp no longer reads the A region
        else mma_commit(B_AEMPTY + 8 * ab);             // SS mode: shared-memory A free
      }
      __syncwarp();
    }
    if (RTC_PROF && lane == 0 && mw == 0) {
      atomicAdd(&g_rtc_cyc[0], (unsigned long long)mw_b);
      atomicAdd(&g_rtc_cyc[1], (unsigned long long)mw_t);
      atomicAdd(&g_rtc_cyc[2], (unsigned long long)mw_i);
      atomicAdd(&g_rtc_cyc[5], (unsigned long long)mw_a);
      atomicAdd(&g_rtc_cyc[8], (unsigned long long)k);
    }
  } else {
    // ===== epilogue: group grp = warp / (NE / GG) drains the tiles k with k % GG == grp; inside a
    // group, warp q4 = warp % 4 reads TMEM lanes 32 q4 .. (its 32 rows) and the column slice cs
    // (BN / NCS columns, chunks of 8) for all S levels.  Branch-free: rows and columns beyond the
    // problem hold zero W (TMA fill), zero digits (split) and a zero scale, so they add nothing.
    constexpr int WPG = NE / GG, NCS = WPG / 4, CW = BN / NCS, XW = Tr<S>::XW, NCH = CW / XW;
    const int grp = warp / WPG, q4 = warp & 3, cs = (warp % WPG) >> 2;
    const int rl = 32 * q4 + lane;
    const uint32_t lane_addr = tmem + ((uint32_t)(32 * q4) << 16) + (uint32_t)(CW * cs);
    const int wsh = __ffs(a.nws) - 1;                    // nws is a power of two
    int k = 0, nitem = 0;
    long long ew_t = 0, ew_w = 0, ew_all = RTC_CLK();
    for (int64_t it = blockIdx.x; it < a.items; it += gridDim.x) {
      int64_t b, rb, c0, c1;
      item_of(it, b, rb, c0, c1);
      if (a.status && a.status[b] != LRA_OK) continue;
      const int64_t gi = rb * BM + rl;
      // biased exponent of the row's scale: 2^(ea_i + fb_tile - 40) (S = 6: R = v / 2^16) or
      // 2^(ea_i + fb_tile - 32) (S = 3); rows outside the problem carry -4000 (scale 0)
      const int eai = (gi < a.m ? a.sa[b * a.m + gi] : -4000) + (S == 6 ? -40 : -32) + 1023;
      const int *sbt = a.sbq + b * a.CB;
      double nu[4] = {0.0, 0.0, 0.0, 0.0}, de[4] = {0.0, 0.0, 0.0, 0.0};   // 4 chains each
      const int ntile = (int)(c1 - c0);
      for (int tt = 0; tt < ntile; ++tt, ++k) {
        if ((k & (GG - 1)) != grp) continue;
        const int tb = k & (NBUF - 1), wsg = k & (a.nws - 1);
        const int ex = eai + __ldg(sbt + c0 + tt);
        const double sc = ex > 0 ? __hiloint2double(ex << 20, 0) : 0.0;
        long long te0 = RTC_CLK();
        mbar_wait(B_TFULL + 8 * tb, (uint32_t)((k / NBUF) & 1));
        asm volatile("tcgen05.fence::after_thread_sync;\n" ::: "memory");
        long long te1 = RTC_CLK();
        ew_t += te1 - te0;
        const TW *wt = Wst + (size_t)wsg * BM * BN + (size_t)(CW * cs) * BM + rl;
        const uint32_t tbase = lane_addr + (uint32_t)(tb * S * BN);
        // R: the recombined levels as an exact int64 (|R| < 2^51), converted to fp64 by the
        // 1.5 2^52 magic add (integer + fp64 pipes: no XU conversion; profiling showed the XU
        // pipe, 16 ops/clk/SM, bounding the I2F-based version).  R = 2^16 b1 + lo with
        //   PRECISE b1 = 256 P0 + P1, lo = (256 P2 + P3) + floor(P4 / 2^8) + floor(P5 / 2^16)
        //           (the floors: < 2 units = 2^-43 of |R|max)
        //   FAST    b1 = P0,          lo = 256 P1 + P2.
        // R + 0x4338000000000000 is one wide multiply-add: the magic only touches the high word,
        // so the addend is the pair (lo, sign(lo) + 0x43380000) — no 64-bit adds.
        auto combine = [&](const uint32_t (&Q)[S][XW], int x, int &b1, int &lo) {
          if (S == 6) {
            b1 = (int)Q[0][x] * 256 + (int)Q[1][x];
            lo = (int)Q[2][x] * 256 + (int)Q[3][x] + ((int)Q[4][x] >> 8) + ((int)Q[5][x] >> 16);
          } else {
            b1 = (int)Q[0][x];
            lo = (int)Q[1][x] * 256 + (int)Q[2][x];
          }
        };
        auto accumulate = [&](int b1, int lo, int col, int x) {
          const long long cm = (long long)(((unsigned long long)(unsigned)((lo >> 31) + 0x43380000) << 32) |
                                           (unsigned long long)(unsigned)lo);
          const double u = __longlong_as_double((long long)b1 * 65536ll + cm) - 6755399441055744.0;
          const double wd = (double)wt[col * BM];
          const double d = fma(-u, sc, wd);
          nu[x & 3] = fma(d, d, nu[x & 3]);
          de[x & 3] = fma(wd, wd, de[x & 3]);
        };
        if constexpr (Tr<S>::EARLY) {
          // PRECISE: drain the whole TMEM slice first (levels combined into (b1, lo) pairs as
          // they arrive), release the buffer, then the fp64 work — the MMAs of the next tile
          // into this buffer overlap the arithmetic instead of waiting for it (the MMA side,
          // 21 products per tile, is what the epilogue waited on: TFULL stalls)
          int B1[CW], LO[CW];
#pragma unroll
          for (int c = 0; c < NCH; ++c) {
            uint32_t Q[S][XW];
            tmem_ld<S, BN, XW>(tbase + (uint32_t)(XW * c), Q);
            asm volatile("tcgen05.wait::ld.sync.aligned;\n" ::: "memory");
            reg_dep<S, XW>(Q);
#pragma unroll
            for (int x = 0; x < XW; ++x) combine(Q, x, B1[XW * c + x], LO[XW * c + x]);
          }
          asm volatile("tcgen05.fence::before_thread_sync;\n" ::: "memory");
          __syncwarp();
          if (lane == 0) mbar_arrive(B_TEMPTY + 8 * tb);
          long long tw0 = RTC_CLK();
          mbar_wait(B_WFULL + 8 * wsg, (uint32_t)((k >> wsh) & 1));
          ew_w += RTC_CLK() - tw0;
#pragma unroll
          for (int x = 0; x < CW; ++x) accumulate(B1[x], LO[x], x, x);
        } else {
          // FAST: chunk by chunk (loading chunk c + 1 ahead of chunk c's arithmetic was measured:
          // no gain — the drain is not TMEM-latency bound — for the registers of a second chunk)
#pragma unroll
          for (int c = 0; c < NCH; ++c) {
            uint32_t Q[S][XW];
            tmem_ld<S, BN, XW>(tbase + (uint32_t)(XW * c), Q);
            asm volatile("tcgen05.wait::ld.sync.aligned;\n" ::: "memory");
            reg_dep<S, XW>(Q);
            if (c == NCH - 1) {           // every chunk read: release the TMEM buffer to the MMA warps
              asm volatile("tcgen05.fence::before_thread_sync;\n" ::: "memory");
              __syncwarp();
              if (lane == 0) mbar_arrive(B_TEMPTY + 8 * tb);
            }
            if (c == 0) {
              long long tw0 = RTC_CLK();
              mbar_wait(B_WFULL + 8 * wsg, (uint32_t)((k >> wsh) & 1));
              ew_w += RTC_CLK() - tw0;
            }
#pragma unroll
            for (int x = 0; x < XW; ++x) {
              int b1, lo;
              combine(Q, x, b1, lo);
              accumulate(b1, lo, XW * c + x, x);
            }
          }
        }
        __syncwarp();
        if (lane == 0) mbar_arrive(B_WEMPTY + 8 * wsg);
      }
      // item partial: each warp parks its sums in the item's slot set; the warp that completes
      // the set adds the NE slots in warp order (deterministic, no barrier)
      double num = warp_sum((nu[0] + nu[1]) + (nu[2] + nu[3]));
      double den = warp_sum((de[0] + de[1]) + (de[2] + de[3]));
      if (lane == 0) {
        const int set = (int)(nitem & 3);
        red[set][warp] = make_double2(num, den);
        __threadfence_block();
        const int prev = atomicAdd(&red_cnt[set], 1);
        if (prev == NE - 1) {
          __threadfence_block();
          double s0 = 0.0, s1 = 0.0;
#pragma unroll
          for (int w = 0; w < NE; ++w) {
            const volatile double *xx = reinterpret_cast<volatile double *>(&red[set][w]);
            s0 += xx[0];
            s1 += xx[1];
          }
          red_cnt[set] = 0;
          const int64_t rem = it % (a.RB * a.nchunk);
          a.partial[b * a.RB * a.nchunk + rem] = make_double2(s0, s1);
        }
      }
      ++nitem;
    }
    if (RTC_PROF && warp == 0 && lane == 0) {
      atomicAdd(&g_rtc_cyc[6], (unsigned long long)ew_t);
      atomicAdd(&g_rtc_cyc[7], (unsigned long long)(RTC_CLK() - ew_all - ew_t - ew_w));
      atomicAdd(&g_rtc_cyc[9], (unsigned long long)ew_w);
    }
  }
  asm volatile("tcgen05.fence::before_thread_sync;\n" ::: "memory");
  __syncthreads();
  if (warp == MW0) {
    asm volatile("tcgen05.fence::after_thread_sync;\n" ::: "memory");
    asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, 512;\n" ::"r"(tmem));
  }
}

static int bn_of(int S) { return S == 6 ? Tr<6>::BN : Tr<3>::BN; }
static int tpi_of(int S) { return S == 6 ? Tr<6>::TPI : Tr<3>::TPI; }

}  // namespace rtc

size_t residual_tc_scratch(int64_t m, int64_t n, int r, int S, int64_t nb) {
  const int BN = rtc::bn_of(S);
  const int KB = (r + rtc::BK - 1) / rtc::BK;
  const int64_t RB = (m + rtc::BM - 1) / rtc::BM, CB = (n + BN - 1) / BN;
  return (size_t)nb * (RB * KB * S * rtc::A_TILE + CB * KB * S * BN * rtc::BK + (m + CB) * 4 + 64) + 1024;
}

// per problem: one partial per work item; the maximum over both modes so the callers' partial
// buffers fit either
int64_t residual_tc_partials(int64_t m, int64_t n) {
  const int64_t RB = (m + rtc::BM - 1) / rtc::BM;
  int64_t best = 0;
  for (int S : {3, 6}) {
    const int BN = rtc::bn_of(S), tpi = rtc::tpi_of(S);
    const int64_t CB = (n + BN - 1) / BN;
    const int64_t p = RB * ((CB + tpi - 1) / tpi);
    best = p > best ? p : best;
  }
  return best;
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

template <int S>
static cudaError_t launch_split(const ResArgs &a, int64_t nb, int KB, int64_t RB, int64_t CB, signed char *Aq,
                                signed char *Bq, int *sa, int *sbq, cudaStream_t st) {
  constexpr int BN = rtc::Tr<S>::BN;
  const dim3 g((unsigned)(RB + (CB + (128 / BN) - 1) / (128 / BN)), (unsigned)nb);
  switch (KB) {
    case 1: rtc::k_split_ab<1, S, BN><<<g, 128, 0, st>>>(a.A, a.B, a.m, a.n, a.r, a.a_stride, a.b_stride, RB, CB, Aq, Bq, sa, sbq, a.status); break;
    case 2: rtc::k_split_ab<2, S, BN><<<g, 128, 0, st>>>(a.A, a.B, a.m, a.n, a.r, a.a_stride, a.b_stride, RB, CB, Aq, Bq, sa, sbq, a.status); break;
    case 3: rtc::k_split_ab<3, S, BN><<<g, 128, 0, st>>>(a.A, a.B, a.m, a.n, a.r, a.a_stride, a.b_stride, RB, CB, Aq, Bq, sa, sbq, a.status); break;
    default: rtc::k_split_ab<4, S, BN><<<g, 128, 0, st>>>(a.A, a.B, a.m, a.n, a.r, a.a_stride, a.b_stride, RB, CB, Aq, Bq, sa, sbq, a.status); break;
  }
  return cudaGetLastError();
}

// cuTensorMapEncodeTiled through the runtime's driver entry point (no link against libcuda)
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

// Tensor-core residual for nb problems (ResArgs as for k_residual).  S digit slices per
// operand (6: PRECISE, 3: FAST), r <= 128.  scratch: residual_tc_scratch bytes; a.partial must
// hold residual_tc_partials(m, n) entries per problem.
cudaError_t launch_residual_tc(ResArgs a, int64_t nb, int S, void *scratch, double *num2, double *den2,
                               cudaStream_t st, int *nlaunch, Prof *pf) {
  using namespace rtc;
  if (S != 3 && S != 6) return cudaErrorInvalidValue;
  if (a.r < 1 || a.r > 4 * BK) return cudaErrorInvalidValue;
  const int BN = bn_of(S), TPI = tpi_of(S);
  const int KB = (a.r + BK - 1) / BK;
  const int64_t RB = (a.m + BM - 1) / BM, CB = (a.n + BN - 1) / BN;
  char *p = reinterpret_cast<char *>((((uintptr_t)scratch) + 255) & ~(uintptr_t)255);
  signed char *Aq = reinterpret_cast<signed char *>(p);
  p += (size_t)nb * RB * KB * S * A_TILE;
  signed char *Bq = reinterpret_cast<signed char *>(p);
  p += (size_t)nb * CB * KB * S * BN * BK;
  p = reinterpret_cast<char *>(((uintptr_t)p + 15) & ~(uintptr_t)15);
  int *sa = reinterpret_cast<int *>(p);
  int *sbq = sa + nb * a.m;
  pf->begin("k_split", st);
  cudaError_t e = S == 6 ? launch_split<6>(a, nb, KB, RB, CB, Aq, Bq, sa, sbq, st)
                         : launch_split<3>(a, nb, KB, RB, CB, Aq, Bq, sa, sbq, st);
  pf->end(st);
  if (e != cudaSuccess) return e;
  TcArgs t{};
  t.m = a.m;
  t.n = a.n;
  t.ldw = a.ldw;
  t.w_stride = a.w_stride;
  t.w = a.w;
  t.Aq = Aq;
  t.Bq = Bq;
  t.sa = sa;
  t.sbq = sbq;
  t.KB = KB;
  t.RB = RB;
  t.CB = CB;
  // Tiles per item: the base TPI, doubled (up to 8x) while every SM still gets >= 8 items.
  // Longer items amortise the per-item work (the A slices' load and TMEM copy, the exponent
  // loads, the 16 warps' partial sums): 32768^2 r = 64 FAST 949 -> see DESIGN.md §6.2.
  static const int tpi_max = getenv("LRA_RTC_TPIX") ? atoi(getenv("LRA_RTC_TPIX")) : 8;   // diagnostics
  int tpi = TPI;
  while (tpi < tpi_max * TPI && nb * RB * ((CB + 2 * tpi - 1) / (2 * tpi)) >= 8 * (int64_t)num_sms_rtc()) tpi *= 2;
  t.tpi = tpi;
  t.nchunk = (CB + tpi - 1) / tpi;
  t.items = nb * RB * t.nchunk;
  const size_t elt = a.dtype == LRA_F32 ? 4 : 8;
  // W through a TMA tensor map over (m, n, nb) when the strides allow it (16-byte multiples)
  CUtensorMap tm;
  memset(&tm, 0, sizeof(tm));
  bool tma_ok = false;
  const int64_t wstr = nb > 1 ? a.w_stride : a.ldw * a.n;
  if (tmap_encode() && (a.ldw * (int64_t)elt) % 16 == 0 && (wstr * (int64_t)elt) % 16 == 0 &&
      (reinterpret_cast<uintptr_t>(a.w) & 15) == 0) {
    cuuint64_t dims[3] = {(cuuint64_t)a.m, (cuuint64_t)a.n, (cuuint64_t)nb};
    cuuint64_t strides[2] = {(cuuint64_t)(a.ldw * elt), (cuuint64_t)(wstr * elt)};
    cuuint32_t box[3] = {(cuuint32_t)BM, (cuuint32_t)BN, 1u};
    cuuint32_t estr[3] = {1u, 1u, 1u};
    CUresult cr = tmap_encode()(&tm, elt == 4 ? CU_TENSOR_MAP_DATA_TYPE_FLOAT32 : CU_TENSOR_MAP_DATA_TYPE_FLOAT64, 3,
                                const_cast<void *>(a.w), dims, strides, box, estr, CU_TENSOR_MAP_INTERLEAVE_NONE,
                                CU_TENSOR_MAP_SWIZZLE_NONE, CU_TENSOR_MAP_L2_PROMOTION_L2_256B,
                                CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
    tma_ok = cr == CUDA_SUCCESS;
  }
  if (!tma_ok) return cudaErrorInvalidConfiguration;    // caller falls back to the fp64 SIMT pass
  bool ts_mode = true;
  {
    const int nbuf = S == 6 ? Tr<6>::NBUF : Tr<3>::NBUF;
    const int acc_cols = nbuf * S * BN, a_cols = S * KB * 8;
    ts_mode = acc_cols + a_cols <= 512;
    t.nabuf = acc_cols + 2 * a_cols <= 512 ? 2 : 1;
  }
  t.partial = a.partial;
  t.status = a.status;
  t.nas = ts_mode ? 1 : 2;
  auto smem_of = [&](int nws, int nbs) {
    return (size_t)t.nas * S * KB * A_TILE + (size_t)nbs * S * KB * BN * BK + (size_t)nws * BM * BN * elt;
  };
  // W stages first (the HBM stream the kernel is bound by), then B stages (L2-resident slices):
  // the first (nws, nbs) in (4, 2) x (8, 4, 2) within the mode's budget.  r = 64 FAST gets 4 W stages instead
  // of 2.  More than 4 W stages does not pay: PRECISE r = 32 at 8 W stages (200 KB of shared
  // memory) is no faster alone and, in lra_batch, keeps the next group's nucleus and factor CTAs
  // off the SMs (config-2 bench 9395 -> 8393 matrices/s).
  const size_t lim = 227 * 1024 - 4096;
  const size_t cap = S == 6 ? Tr<6>::SMEM_CAP : Tr<3>::SMEM_CAP;
  t.nws = 2;
  t.nbs = 2;
  {
    bool found = false;
    static const int nws_max = getenv("LRA_RTC_NWS") ? atoi(getenv("LRA_RTC_NWS")) : 4;   // diagnostics
    for (int w = nws_max; w >= 2 && !found; w >>= 1)
      for (int b = NBS; b >= 2 && !found; b >>= 1)
        if (smem_of(w, b) <= cap) {
          t.nws = w;
          t.nbs = b;
          found = true;
        }
  }
  const size_t smem = smem_of(t.nws, t.nbs);
  if (smem > lim) return cudaErrorInvalidConfiguration;   // caller falls back to the fp64 SIMT pass
  static const int grid_cap = getenv("LRA_RTC_GRID") ? atoi(getenv("LRA_RTC_GRID")) : 0;   // diagnostics
  int64_t ncta = grid_cap > 0 && grid_cap < num_sms_rtc() ? grid_cap : num_sms_rtc();
  const int64_t grid = t.items < ncta ? t.items : ncta;
  void (*kern)(TcArgs, CUtensorMap);
  if (ts_mode)
    kern = a.dtype == LRA_F32 ? (S == 6 ? k_resid<float, 6, true> : k_resid<float, 3, true>)
                              : (S == 6 ? k_resid<double, 6, true> : k_resid<double, 3, true>);
  else
    kern = a.dtype == LRA_F32 ? (S == 6 ? k_resid<float, 6, false> : k_resid<float, 3, false>)
                              : (S == 6 ? k_resid<double, 6, false> : k_resid<double, 3, false>);
  e = cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
  if (e != cudaSuccess) return e;
  pf->begin("k_residual_tc", st);
  kern<<<(unsigned)grid, S == 6 ? nthreads<6>() : nthreads<3>(), smem, st>>>(t, tm);
  pf->end(st);
  if ((e = cudaGetLastError()) != cudaSuccess) return e;
  *nlaunch += 2;
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
