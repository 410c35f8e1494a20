// kernels.cuh — argument blocks and launchers shared by the kernel files and lra_api.cu.
#pragma once
#include <vector>

#include "common.cuh"

namespace lra {

// Per-handle kernel timing (lra_profile_*): a CUDA event pair recorded on the launch
// stream around every kernel while enabled; read back (and reset) by lra_profile_read.
struct Prof {
  int on = 0;
  std::vector<cudaEvent_t> ev;
  std::vector<const char *> name;
  size_t used = 0;
  void begin(const char *nm, cudaStream_t st) {
    if (!on) return;
    grow();
    name[used / 2] = nm;
    cudaEventRecord(ev[used++], st);
  }
  void end(cudaStream_t st) {
    if (!on) return;
    cudaEventRecord(ev[used++], st);
  }
  void grow() {
    if (used + 2 <= ev.size()) return;
    for (int i = 0; i < 64; ++i) {
      cudaEvent_t e;
      cudaEventCreate(&e);
      ev.push_back(e);
    }
    name.resize(ev.size() / 2);
  }
};

struct SketchArgs {
  int kind, dtype, depth, nnz;
  int64_t m, n, lbar, ldw, ldy;
  const void *w;
  int64_t w_stride;                 // batch stride of W (elements)
  const int8_t *dsign;
  const int64_t *col, *sp_row;
  const int8_t *sp_sign;
  int64_t m_stride;                 // batch stride of the multiplier arrays (entries)
  void *y;
  int64_t y_stride;                 // batch stride of Y (elements of double / double2)
};
cudaError_t launch_sketch(const SketchArgs &a, int64_t nb, const double *omega, int64_t ldo, cudaStream_t st, Prof *pf,
                          void *tc_scratch = nullptr, size_t tc_bytes = 0);
// the Gaussian sketch on the tensor cores (sketch_tc.cu, reading C36)
size_t sketch_tc_scratch_bytes(int64_t m, int64_t n, int64_t lbar, int64_t nb);
size_t sketch_tc_zero_bytes();   // leading bytes of a fresh scratch buffer that must be zeroed once
cudaError_t launch_sketch_tc(const SketchArgs &a, int64_t nb, const double *omega, int64_t ldo, void *scratch,
                             size_t scratch_bytes, cudaStream_t st, Prof *pf);
// NEXT-1: all n columns of W D H_{n,d} P (pinv: n ints of scratch)
cudaError_t launch_transform_full(const SketchArgs &a, int *pinv, void *out, int64_t ldo, cudaStream_t st, Prof *pf);

struct CAArgs {
  OpView op;
  int64_t w_stride;            // batch stride of dense W (elements)
  const void *Y;               // sketch (m x q, column-major, fp64 / complex128) or null
  int64_t ldy, y_stride;
  int y_complex;
  const int64_t *I0;           // used iff Y == null
  int64_t i0_stride;
  int q, sweeps, cap, cs, rpc, qp;
  double tol, tau;
  int64_t *I, *J;              // outputs, stride q per problem
  lra_ca_stats *stats;         // per problem, may be null
  int diag;                    // diagnostics (global tier only): min_pivot_margin
  int32_t *status;             // per problem
  int32_t *yinfo;              // per problem x4: complex stage-2 result (scratch), or null
  int grid;                    // 1: grid tier (one problem over a cooperative grid)
  int y_warm;                  // 1: the maxvol on Y starts from the slots I0 (no LUP)
  const int32_t *skip;         // row-sharded chain control (nullable): nothing is done when skip[0]
                               // (an earlier step failed) or skip[1] (the C-A converged) is set
  void *gscratch;              // grid tier exchange buffers (ca_grid_scratch_bytes)
};
size_t ca_grid_scratch_bytes(int cs);
// tier chosen for a problem of maxN rows and q columns: 0 none, 1 cluster, 2 grid; cs out
int ca_tier(int64_t maxN, int q, bool cplx, int *cs_out);
cudaError_t launch_ca(CAArgs a, int64_t nb, int64_t maxN, cudaStream_t st, int *cs_out, Prof *pf);
cudaError_t read_ca_counters(unsigned long long *out, bool reset);
// cluster tier of the real C-A (ca_cluster.cu); cudaErrorInvalidConfiguration if it does not fit
cudaError_t launch_ca_cluster(CAArgs a, int64_t nb, int64_t maxN, cudaStream_t st, int *cs_out, Prof *pf);
// small tier (ca_small.cu): one 128-thread CTA per problem, several problems per SM
bool ca_small_fits(int64_t maxN, int q, int y_complex, int y_warm);
int ca_small_max_active(int64_t maxN, int q);
cudaError_t launch_ca_small(CAArgs a, int64_t nb, int64_t maxN, cudaStream_t st, int *cs_out, Prof *pf);
size_t nucleus_smem(int k, int l);
bool nucleus_fits(int k, int l);
cudaError_t read_nuc_counters(unsigned long long *out, bool reset);
cudaError_t read_idx_err_nuc(long long *out, bool reset);   // diagnostics (LRA_CHECK_IDX builds)
cudaError_t read_idx_err_cc(long long *out, bool reset);
cudaError_t read_cc_counters(unsigned long long *out, bool reset);
cudaError_t read_gm_exact(unsigned long long *out, bool reset);
int ca_cluster_max_active(int64_t maxN, int q);
// global-memory tier (ca_global.cu): any N, q <= 128; scratch ca_global_scratch_bytes
size_t ca_global_scratch_bytes(int64_t maxN, int q);
cudaError_t launch_ca_global(CAArgs a, int64_t nb, int64_t maxN, void *scratch, cudaStream_t st, Prof *pf);
// true when neither the cluster tier nor the grid tier holds a maxN x q block on chip
bool ca_needs_global(int64_t maxN, int q);
cudaError_t read_rtc_counters(unsigned long long *out, bool reset);

struct NucArgs {
  OpView op;
  int64_t w_stride;
  const int64_t *I, *J;   // stride q per problem
  int k, l, r;
  double *U;              // l x k per problem (stride l*k), may be null
  double *TS, *Sr;        // scratch: l x r and k x r per problem
  int32_t *status;        // per problem: already LRA_ESINGULAR -> skip
  const double *Gd;       // optional dense G = W[I,J] (k x l col-major) instead of gathering
  lra_ca_stats *stats;    // optional, per problem: logvol_final (square generators)
};
struct FacArgs {
  OpView op;
  int64_t w_stride;
  const int64_t *I, *J;
  int k, l, r;
  const double *TS, *Sr;
  double *A, *B;            // A: m x r (lda = m) per problem; B: r x n (ld r) per problem
  int64_t a_stride, b_stride;
  const int32_t *status;
  const double *Rt;         // optional dense R^T = W[I,:]^T (n x k col-major, ld n) for B
};
// row-sharded operands (shard.cu): owner-scattered blocks, assembled by an NCCL sum
cudaError_t launch_scatter_rows(const double *src, int64_t ld, int64_t m_local, int q, int64_t row0,
                                int64_t m_global, double *dst, cudaStream_t st);
cudaError_t launch_scatter_wcols(const OpView &op, const int64_t *J, int q, int64_t row0, int64_t m_global,
                                 double *dst, cudaStream_t st);
cudaError_t launch_scatter_wrows(const OpView &op, const int64_t *I, int q, int64_t row0, double *dst,
                                 cudaStream_t st);
cudaError_t launch_scatter_g(const OpView &op, const int64_t *I, const int64_t *J, int k, int l, int64_t row0,
                             double *dst, cudaStream_t st);
// allgather assembly of the row-sharded blocks (shard.cu): local rows packed into a cm x q chunk
// (zero rows beyond m_local), gathered chunks unpacked into the m_global x q block
cudaError_t launch_pack_rows(const double *src, int64_t ld, int64_t m_local, int q, int64_t cm, double *chunk,
                             cudaStream_t st);
cudaError_t launch_pack_wcols(const OpView &op, const int64_t *J, int q, int64_t cm, double *chunk, cudaStream_t st);
cudaError_t launch_unpack_chunks(const double *gathered, int64_t cm, int q, int nranks, int64_t m_global, double *dst,
                                 cudaStream_t st);
// device-side control of the row-sharded C-A chain (no host synchronization)
cudaError_t launch_ctl_step(const lra_ca_stats *sts, int idx, int kind, int loop, int32_t *ctl, cudaStream_t st);
cudaError_t launch_ctl_combine(const lra_ca_stats *sts, const int32_t *ctl, int has_y, lra_ca_stats *out,
                               cudaStream_t st);
cudaError_t launch_nucleus(const NucArgs &na, const FacArgs &fa, int64_t nb, cudaStream_t st, int *nlaunch, Prof *pf);

struct ResArgs {
  int dtype;
  int64_t m, n, ldw, w_stride;
  const void *w;
  const double *A, *B;       // per problem: A + b*a_stride (lda = m), B + b*b_stride (ld r)
  int64_t a_stride, b_stride;
  int r;
  int64_t tiles_m, tiles_n;  // tiles per problem
  double2 *partial;          // per problem per tile: (num2, den2)
  const int32_t *status;
};
cudaError_t launch_residual(ResArgs a, int64_t nb, double *num2, double *den2, cudaStream_t st, int *nlaunch, Prof *pf);
cudaError_t launch_reduce(const double2 *partial, int64_t ntiles, int64_t nb, double *num2, double *den2,
                          const int32_t *status, cudaStream_t st, int *nlaunch, Prof *pf);
// tensor-core residual (residual_tc.cu): S digit slices (6 PRECISE, 3 FAST)
size_t residual_tc_scratch(int64_t m, int64_t n, int r, int S, int64_t nb);
int64_t residual_tc_partials(int64_t m, int64_t n);
cudaError_t launch_residual_tc(ResArgs a, int64_t nb, int S, void *scratch, double *num2, double *den2,
                               cudaStream_t st, int *nlaunch, Prof *pf);
cudaError_t launch_error_sample(const OpView &op, const double *A, const double *B, int r, const int64_t *rows,
                                int64_t q, const int64_t *cols, int64_t s, double *g, double *out3, cudaStream_t st,
                                int *nlaunch, Prof *pf);
// NEXT-3 greedy column expansion (expand.cu); scratch: (k n + k k + n) doubles
size_t qrp_scratch_bytes(int k, int64_t n);
cudaError_t launch_qrp(const OpView &op, const int64_t *I, int k, int q, double tau, int64_t *piv, double *R,
                       int64_t ldr, double *Rt, int32_t *status, void *scratch, cudaStream_t st, int *nlaunch,
                       Prof *pf);
cudaError_t launch_contract_columns(const OpView &op, const int64_t *I, int k, int64_t *J, int g0, int l, double tau,
                                    void *scratch, int *ok, cudaStream_t st, int *nlaunch, Prof *pf);
cudaError_t launch_refine_columns(const OpView &op, const int64_t *I, int k, int64_t *J, int l, int cycles,
                                  double tau, void *scratch, int *ok, int *stop, int *changed, cudaStream_t st,
                                  int *nlaunch, Prof *pf);
cudaError_t launch_qg_build(int64_t n, int q, int64_t lbar, const int8_t *sign, const int64_t *perm,
                            const int64_t *col, int *work, double *omega, cudaStream_t st, Prof *pf);
size_t leverage_scratch_bytes(int k, int r, int64_t N);
cudaError_t launch_leverage_scores(const OpView &op, const int64_t *I, int k, int side, int r, double *p,
                                   int32_t *status, void *scratch, cudaStream_t st, int *nlaunch, Prof *pf);
cudaError_t launch_sample_exactly(const double *p, int64_t N, int l, const double *u, double *P, int64_t *idx,
                                  double *dsc, const int32_t *status, cudaStream_t st, int *nlaunch, Prof *pf);
cudaError_t launch_sample_expected(const double *p, int64_t N, int l, const double *u, int64_t cap, int64_t *idx,
                                   double *dsc, int64_t *count, const int32_t *status, cudaStream_t st, int *nlaunch,
                                   Prof *pf);
cudaError_t launch_expand_columns(const OpView &op, const int64_t *I, int k, int64_t *J, int g0, int l, double tau,
                                  void *scratch, int *ok, cudaStream_t st, int *nlaunch, Prof *pf);
cudaError_t launch_cert_norms(const OpView &op, const int64_t *I, const int64_t *J, int k, int l, const double *U,
                              double *out3, cudaStream_t st);
cudaError_t launch_sampled(const OpView &op, const double *A, const double *B, int r, const int64_t *si,
                           const int64_t *sj, int64_t Q, double2 *partial, int nblk, double *num2,
                           double *den2, cudaStream_t st, int *nlaunch, Prof *pf);

}  // namespace lra
