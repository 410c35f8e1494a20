/*
 * lra.h — C-ABI of the B200-native superfast CUR hot path (arXiv 1710.07946).
 *
 * Citation keys: P:n = line n of the paper's LaTeX, with \label names.
 * The path is Alg 10.2 ("algrhtcur") with C-A iterations at stage 3
 * (Remark "rerfnhmt"), maxvol by Alg D.2 stage 1 + Alg D.1 ("alggos",
 * "algdomin"), the canonical nucleus (Alg 3.1 "algcnnncl")
 * and the a-posteriori check rho = ||W - CUR||_F / ||W||_F (eq. "eqcur0").
 * DESIGN.md §2 lists every reading of the paper these functions implement.
 *
 * Conventions (all entry points):
 *  - Pointers are DEVICE pointers unless marked (host).  Matrices are COLUMN-MAJOR with
 *    0-based int64 indices; index sets are int64 arrays in slot order.
 *  - Ownership: every buffer is caller-owned; the library never frees caller memory.
 *    Scratch belongs to the handle, grows on first use at a size, and is reused (no
 *    allocation on the hot path once warm).
 *  - Asynchrony: every call is stream-ordered on `stream` (a cudaStream_t, NULL = legacy
 *    default stream) and returns after enqueueing.  Argument errors are returned
 *    synchronously; numerical failures of the data-dependent loops (LRA_ESINGULAR, cap
 *    hits) are written to device memory (lra_ca_stats.status, per-block status).
 *  - On a non-OK status the outputs are unspecified.  lra_last_error() returns a
 *    thread-local message describing the last non-OK status.
 *  - There is no CPU fallback: without a CUDA device every call returns LRA_ECUDA.
 */
#ifndef LRA_H
#define LRA_H

#include <stddef.h>
#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

typedef enum {
  LRA_OK = 0,
  LRA_EINVAL = -1,       /* shape / pointer / parameter violation                      */
  LRA_ESINGULAR = -2,    /* zero or non-finite pivot, singular generator, sigma_r = 0  */
  LRA_ENOMEM = -3,       /* scratch allocation failed                                  */
  LRA_ECUDA = -4,        /* CUDA runtime error (incl. no device)                       */
  LRA_ENCCL = -5,        /* reserved for the multi-GPU exchange                         */
  LRA_EUNSUPPORTED = -6  /* valid input outside this build's tiers   */
} lra_status;

typedef enum { LRA_F32 = 0, LRA_F64 = 1 } lra_dtype;

/* "W or an entry oracle" (the paper's input). */
typedef enum { LRA_OP_DENSE = 0, LRA_OP_FACTORED_CSR = 1 } lra_op_kind;

typedef struct {
  int32_t kind;             /* lra_op_kind                                                    */
  int32_t dtype;            /* lra_dtype of W's values (DENSE)                                */
  int64_t m, n;             /* shape of W                                                     */
  const void *w;            /* DENSE: m x n column-major, leading dimension ldw >= m          */
  int64_t ldw;
  /* FACTORED_CSR (config 4): W = A*B + E, never formed.  A m x p (ld m), B p x n (ld p),
     fp64 values; E in CSR over rows: e_rowptr[m+1], e_col[nnz] (ascending per row), e_val. */
  const double *fa, *fb;
  int64_t p;
  const int64_t *e_rowptr, *e_col;
  const double *e_val;
  /* Row sharding (multi-GPU): this rank holds rows [row0, row0 + m) of an
     m_global x n matrix (DENSE only).  m_global = 0: not sharded.  Requires a handle created
     with an NCCL communicator; every rank calls the entry points in the same order. */
  int64_t row0, m_global;
} lra_operand;

/* Realized randomized multiplier M (n x lbar). */
typedef enum {
  LRA_MUL_NONE = 0,      /* no sketch: C-A starts from a given I0 (Tests 2)       */
  LRA_MUL_GAUSSIAN = 1,  /* omega: n x lbar fp64 column-major (ld_omega)                       */
  LRA_MUL_ARHT = 2,      /* (D H_{n,d} P)[:, col]: dsign[n] in {+1,-1}, col[lbar], 2^depth | n  */
  LRA_MUL_ARFT = 3,      /* (D Omega_{n,d} P)[:, col]; Y is complex128                         */
  LRA_MUL_SPARSE_PM1 = 4,/* column c: rows sp_row[c*nnz+t], signs sp_sign[c*nnz+t], t < nnz    */
  LRA_MUL_QGAUSS = 5     /* quasi-Gaussian (def11; reading C30): G = M_0...M_{q-1},
                            M_i = B_i P_i, q = depth (1..30); B_i: ones on the diagonal, qg_sign
                            [i*n + c] at (c+1 mod n, c); P_i[qg_perm[i*n + c], c] = 1; the sketch
                            uses the lbar columns col of G (built exactly on the device, then
                            applied like a Gaussian omega)                                   */
} lra_mul_kind;

typedef struct {
  int32_t kind;             /* lra_mul_kind                          */
  int32_t depth;            /* d >= 1 (ARHT / ARFT)                  */
  int64_t lbar;             /* number of sketch columns (== k == l)  */
  const int8_t *dsign;      /* n entries                             */
  const int64_t *col;       /* lbar sampled columns of T, in order   */
  const int64_t *sp_row;    /* lbar * nnz_per_col                    */
  const int8_t *sp_sign;    /* lbar * nnz_per_col                    */
  int32_t nnz_per_col;
  const double *omega;      /* GAUSSIAN                              */
  int64_t ld_omega;
  const int8_t *qg_sign;    /* QGAUSS: depth x n subdiagonal signs   */
  const int64_t *qg_perm;   /* QGAUSS: depth x n permutations        */
} lra_multiplier;

typedef struct lra_handle_s *lra_handle;

/* Per-matrix statistics of lra_cross_approx / lra_batch (device memory). */
typedef struct {
  int32_t status;           /* LRA_OK or LRA_ESINGULAR                                       */
  int32_t loops_done;       /* C-A loops executed (early exit on a fixed point, reading C13) */
  int32_t lu_steps;         /* cold-start LUP steps (Alg D.2 stage 1)                        */
  int32_t swaps;            /* Alg D.1 swaps over all maxvol calls                           */
  int32_t cap_hits;         /* maxvol calls that stopped at the swap cap (not an error)      */
  int32_t sketch_swaps;     /* swaps of the stage-2 maxvol on Y                              */
  double cert_rows;         /* max |C'| at exit of the last vertical step   (<= 1 + tol)     */
  double cert_cols;         /* max |C'| at exit of the last horizontal step (<= 1 + tol)     */
  double logvol_final;      /* log v2(W[I,J]) = log|det W[I,J]| of the final generator (eq.
                               eqvol; every swap multiplies it by |c*| > 1,
                               P:6511-6513): the sum of log sigma_i of the nucleus' Jacobi SVD
                               of the whole k x k generator; NaN if the nucleus did not run   */
  double min_pivot_margin;  /* min over every pivot decision (cold LUP steps and swaps of all
                               maxvol calls) of the top-2 margin (M - M2)/M, M2 the largest
                               candidate other than the chosen one (reading C35): 0 = a tie
                               broken by the index rule, tiny = a rounding-level reorder risk.
                               Measured only with diagnostics on (lra_set_diagnostics), else NaN */
} lra_ca_stats;

/* Precision of the reconstruction A*B inside the full a-posteriori pass.
   Both run the product on the tcgen05 tensor cores as an exact int8 digit-slice
   (Ozaki-style) contraction with int32 TMEM accumulators, recombined exactly in int64:
   balanced base-256 digits, one exponent per row of A and per 32/64-column tile of B.
   PRECISE keeps 6 slices per operand (levels s + u <= 5: truncation ~2^-45 of
   max|A_i| max|B_j|; rho within ~1e-8 of the exact product on configs 2 and 3), FAST 3
   slices (~2^-21, fp32-class).  fp64 W in PRECISE mode, or a configuration the tensor-core
   kernel cannot hold (r > 64 in PRECISE), uses an fp64 FMA kernel (fp64-exact to rounding). */
typedef enum {
  LRA_RECON_FAST = 0,
  LRA_RECON_PRECISE = 1
} lra_recon;

/* Create a handle bound to CUDA device `device`.  nccl_unique_id (host, 128 bytes from
   lra_nccl_unique_id on one rank, distributed by the caller) creates an NCCL communicator of
   nranks ranks (this one = rank) used by the row-sharded path; NULL (with nranks == 1) for
   single-GPU use.  NCCL is loaded at run time (libnccl.so.2); LRA_ENCCL if it cannot be. */
lra_status lra_handle_create(lra_handle *h /* host */, int device, const void *nccl_unique_id,
                             int nranks, int rank);
/* Write a fresh NCCL unique id (128 bytes) to out (host). */
lra_status lra_nccl_unique_id(void *out /* host, 128 bytes */);
void lra_handle_destroy(lra_handle h);

/* Scratch of one workload shape (SURVEY 8(b) "lra_workspace_query"; the handle owns every
   scratch buffer and grows it on first use).  nb == 0: the single-problem calls
   lra_preprocess / lra_cross_approx (sweeps) / lra_cur_residual (either lra_recon) on W with
   rank r and k = l; nb >= 1: lra_batch over nb blocks shaped like W.  *bytes (host) = the
   device bytes those calls need.  lra_workspace_reserve allocates them now, so the calls of
   that shape allocate nothing (and can be captured in a CUDA graph).  Errors: EINVAL for a
   bad operand/shape (the checks of lra_cross_approx), ENOMEM. */
lra_status lra_workspace_query(lra_handle h, const lra_operand *W, int64_t r, int64_t k, int32_t sweeps,
                               int64_t nb, size_t *bytes /* host */);
lra_status lra_workspace_reserve(lra_handle h, const lra_operand *W, int64_t r, int64_t k, int32_t sweeps,
                                 int64_t nb);

/* Stage 1 of Alg 10.2: Y = W * M, an m x lbar fp64 column-major matrix
   (ARFT: complex128, interleaved re/im), leading dimension ldy >= m.  Sums run in a fixed
   order (ascending t for ARHT/ARFT, draw order for SPARSE_PM1, ascending k for GAUSSIAN)
   with fp64 accumulation; the SRHT scale sqrt(n/lbar) is omitted (reading C8).
   Errors: EINVAL for null pointers, lbar < 1, 2^depth not dividing n, non-DENSE W. */
lra_status lra_preprocess(lra_handle h, const lra_operand *W /* host struct */,
                          const lra_multiplier *M /* host struct */, void *Y, int64_t ldy,
                          void *stream);

/* Alg 10.1 stage 1 with u = n (the Table tb_fh protocol, with the
   ARHT multiplier of P:6110-6124): Wout = W D H_{n,d} P, all n columns, m x n column-major in
   W's dtype (ldo >= m).  M: kind ARHT, lbar == n, col = the whole permutation P (column c of
   Wout = column col[c] of W D H_{n,d}), depth <= 5.  Each output is the fp64 signed sum over
   its 2^d nonzeros in ascending t, rounded once to W's precision (reading C25).  Reads W once
   and writes Wout once.  Then C-A and the nucleus run on Wout (I0 = a random start, Tests 2),
   C = Wout[:,J], U = Wout_{k,l,r}^+ and R = R_H H^+ = W[I,:] (the residual of CUR on W equals
   the one on Wout since M M^T = 2^d I).  Errors: EINVAL / EUNSUPPORTED synchronously. */
lra_status lra_preprocess_full(lra_handle h, const lra_operand *W /* host struct */,
                               const lra_multiplier *M /* host struct */, void *Wout, int64_t ldo, void *stream);

/* Row-sharded operands (W.m_global > 0): the sketch Y is this rank's m x lbar part; every C-A
   block (Y, W[I,:]^T, W[:,J], W[I,J]) is assembled on every rank by an exact NCCL sum of the
   owners' rows and the maxvol runs replicated, so I, J, U, B are identical on every rank and
   equal to the single-GPU result; A holds this rank's rows.  ARFT sketches are not sharded.
   Stages 2-3 of Alg 10.2 with C-A at stage 3 (Remark rerfnhmt), then Alg 3.1:
     I <- maxvol(Y) (cold)  or  I <- I0 (if Y == NULL);
     for loop < sweeps:  J <- maxvol(W[I,:]^T, warm from J after loop 1)
                         I <- maxvol(W[:,J],  warm from I);  stop when a later loop swaps nothing;
     U = W_{k,l,r}^+ via the SVD W[I,J] = S Sigma T^T  (l x k, column-major),
     A = W[:,J] T_r Sigma_r^{-1}  (m x r, ld m),   B = S_r^T W[I,:]  (r x n, ld r),
   so that CUR = A*B.  maxvol: pivot rule = smallest row-major index among |c| >= (1-tie_slack)*max
   (reading C11), stop when max |C'| <= 1 + swap_tol (C12), at most swap_cap swaps per call.
   Requires 0 < r <= k == l (reading C9), k <= min(m, n), k <= 112 (on-chip tiers for k <= 64,
   the global-memory tier beyond and for blocks too tall for the on-chip tiers).
   y_complex != 0 means Y is complex128 (ARFT).  stats (device) may be NULL.
   Errors: EINVAL / EUNSUPPORTED synchronously; ESINGULAR in stats->status. */
lra_status lra_cross_approx(lra_handle h, const lra_operand *W, const void *Y, int64_t ldy,
                            int y_complex, const int64_t *I0, int64_t r, int64_t k, int64_t l,
                            int32_t sweeps, double swap_tol, double tie_slack, int32_t swap_cap,
                            int64_t *I, int64_t *J, double *U, double *A, double *B,
                            lra_ca_stats *stats, void *stream);

/* A-posteriori check (eq. eqcur0): num2 = sum_ij (W_ij - (A B)_ij)^2 and
   den2 = sum_ij W_ij^2 in fp64 over the full matrix (nsamples == 0), or, when nsamples > 0,
   num2 = (m n / Q) sum_q d_q^2 over the Q given pairs (si[q], sj[q]) and den2
   = the exact ||W||_F^2 (dense: full pass; factored: tr((A^T A)(B B^T)) + 2 sum_E E.(AB) +
   sum E^2).  num2, den2: device scalars.  prec: lra_recon (full pass only; the sampled
   estimate is always fp64).  Row-sharded W: local rows with the local A, then an NCCL sum
   of num2 and den2 (the sampled estimate is not sharded). */
lra_status lra_cur_residual(lra_handle h, const lra_operand *W, const double *A, const double *B,
                            int64_t r, int32_t prec, int64_t nsamples, const int64_t *si,
                            const int64_t *sj, double *num2, double *den2, void *stream);

/* Rectangular generators (NEXT-3): greedy expansion of the column set J[0..g0) of the k x g0
   submatrix W[I, J] to l >= g0 columns (Alg D.4 "algrup"): each appended column j
   maximizes v2^2 growth 1 + b_j^T (C C^T)^{-1} b_j (eq. eqbun), ties -> smallest j among
   scores >= (1 - tie_slack) max (reading C11).  J (device, l entries) holds the g0 start
   columns on entry and all l on return.  Requires k <= g0 (C full row rank), k <= 128. */
lra_status lra_expand_columns(lra_handle h, const lra_operand *W, const int64_t *I, int64_t k, int64_t *J, int64_t g0,
                              int64_t l, double tie_slack, void *stream);
/* Greedy contraction (Def defgrdc; eq. eqbtr) of the column set of R = W[I,:]
   (k x n): J (device) holds g0 slots on entry and its first l on return (k <= l <= g0); each
   step removes the column of minimal leverage ||L^{-1} c_j||^2 (L L^T = C C^T), ties: the
   smallest slot within (1 + tie_slack) min; the other slots keep their order.  Dense or
   entry-oracle W, not row-sharded; k <= 128. */
lra_status lra_contract_columns(lra_handle h, const lra_operand *W, const int64_t *I, int64_t k, int64_t *J,
                                int64_t g0, int64_t l, double tie_slack, void *stream);
/* The expand-contract search of section scrsorth with p = 1: up to `cycles`
   times append the greedy expansion's column (Alg D.4) and remove the greedy contraction's
   column; stops on device at the fixed point (the contraction removes the appended column).
   J (device, l slots) is refined in place; changed (device int32) = the cycles that changed J.
   The volume of W[I,J] never decreases.  k <= l < n, k <= 128. */
lra_status lra_refine_columns(lra_handle h, const lra_operand *W, const int64_t *I, int64_t k, int64_t *J, int64_t l,
                              int32_t cycles, double tie_slack, int32_t *changed, void *stream);

/* SVD-based leverage scores (eq. eqlevsc with beta = 1, eq. eqlevsc1) of the N
   columns of the k x N block B: side 0 -> B = W[idx,:] (N = n, column scores), side 1 ->
   B = W[:,idx]^T (N = m, row scores).  p (device, N fp64): p_j = ||(V_r)_{j,:}||^2 / r with
   V_r the r top right singular vectors (computed from the eigenpairs of B B^T by the Jacobi
   nucleus kernel); sum p = 1 up to rounding.  status (device int32): LRA_OK or ESINGULAR
   (rank of B < r).  1 <= r <= k <= 112; dense or entry-oracle W, not row-sharded. */
lra_status lra_leverage_scores(lra_handle h, const lra_operand *W, const int64_t *idx, int64_t k, int32_t side,
                               int64_t r, double *p, int32_t *status, void *stream);
/* Exactly(l) sampling and rescaling (Alg C.1 "algsmplex"; reading C31): l picks
   with Probability(i_t = i) = p_i driven by the caller's uniforms u (device, l values in
   [0, 1)): i_t = the smallest i with u_t P_{N-1} < P_i, P the sequential prefix sums of p.
   p (device, N fp64) may be NULL: the uniform scores p_i = 1/N of the superfast variant of
   Alg 9.1 (section slrasmpav).
   idx (device, l int64) gets the picks (with replacement), dscale (device, l fp64, may be
   NULL) the rescaling 1 / sqrt(l p_{i_t}).  status (device, may be NULL): nothing is done
   when it is not LRA_OK (chained after lra_leverage_scores). */
lra_status lra_sample_exactly(lra_handle h, const double *p, int64_t N, int64_t l, const double *u, int64_t *idx,
                              double *dscale, const int32_t *status, void *stream);
/* Expected(l) sampling and rescaling (Alg C.2 "algsmplexp"; reading C33): every i
   in 0..N-1 is kept independently with probability pi_i = min{1, l p_i}, decided by the
   caller's uniform u_i (device, N values in [0, 1)): kept iff u_i < pi_i (fp64).  The kept i,
   in ascending order, go to idx (device, cap int64) and their rescaling 1 / min{1, sqrt(l p_i)}
   to dscale (device, cap fp64, may be NULL); count (device int64) gets the number kept (its
   expectation is sum_i pi_i <= l) — entries past cap are counted but not written.  p may be
   NULL (uniform p_i = 1/N).  status as for lra_sample_exactly.  One CTA; asynchronous. */
lra_status lra_sample_expected(lra_handle h, const double *p, int64_t N, int64_t l, const double *u, int64_t cap,
                               int64_t *idx, double *dscale, int64_t *count, const int32_t *status, void *stream);

/* maxvol of a dense fp64 block (Alg D.2 stage 1 + Alg D.1; readings C10-C12):
   B is N x q column-major (ld N, device, caller-owned, read only).  start == NULL: the LUP
   cold start with the slack pivot rule, then the swap loop; start (device, q slots): the swap
   loop from that set.  slots (device, q int64): the selected rows in slot order.  stats
   (device, may be NULL): certificate max|C| at exit, swaps, LU steps, status (ESINGULAR on a
   zero / non-finite pivot).  1 <= q <= min(N, 112); EINVAL otherwise.  Asynchronous. */
lra_status lra_maxvol(lra_handle h, const double *B, int64_t N, int64_t q, const int64_t *start, double swap_tol,
                      double tie_slack, int32_t swap_cap, int64_t *slots, lra_ca_stats *stats, void *stream);

/* Greedy column expansion from a vector to k x q by Householder QR with column pivoting
   (Alg D.3 "alg1tor"; reading C29), on R = W[I,:] (k x n; dense or entry-oracle
   W, not row-sharded; I device, k rows).  Step g takes the column of maximal trailing norm
   (ties: smallest column within the slack tie_slack, reading C11) and reflects the trailing
   rows with I - beta v v^T; sums in ascending row order, no fused operations (bit-identical
   to the oracle).  Outputs (device): piv (q pivots in order); optional R (q x n column-major,
   ld ldr >= q) and Rt (n x q column-major): the first q rows of H_{q-1}...H_0 R in the
   original column order — R' of Alg 7.1 when q = r.  status (device int32):
   LRA_OK or ESINGULAR (trailing norms all zero: rank < q).  1 <= q <= min(k, n), k <= 128. */
lra_status lra_qrp_columns(lra_handle h, const lra_operand *W, const int64_t *I, int64_t k, int64_t q,
                           double tie_slack, int64_t *piv, double *R, int64_t ldr, double *Rt, int32_t *status,
                           void *stream);

/* Canonical nucleus U = W_{k,l,r}^+ (Alg 3.1) of the generator W[I,J] (any k x l,
   k, l <= 128 whose Jacobi working set min(k,l)+1 columns of max(k,l) plus the rotation matrix
   fits in shared memory: square k = l <= 112; EUNSUPPORTED otherwise) and the factors A = W[:,J] T_r Sigma_r^{-1} (m x r), B = S_r^T W[I,:] (r x n),
   as lra_cross_approx computes them for k = l.  status (device int32): LRA_OK or ESINGULAR. */
lra_status lra_nucleus_factors(lra_handle h, const lra_operand *W, const int64_t *I, const int64_t *J, int64_t k,
                               int64_t l, int64_t r, double *U, double *A, double *B, int32_t *status, void *stream);

/* Superfast a-posteriori estimation (Section "spstr"; NEXT-2): the q x s
   submatrix E[rows, cols] of E = W - A B (rows[q], cols[s]: device int64) gives K = q s values
   g_i; stats3 (device, 4 doubles) = { mu_K = sum g_i / K, sigma_K^2 = sum (g_i - mu_K)^2 / K
   (reading C26), sum g_i^2, sum W_ij^2 over the same entries } — the last two extrapolate to
   ||E||_F^2 and ||W||_F^2 (times m n / K).  W: dense or the factored entry oracle.  O(K r)
   work: superfast for K = O((m+n) k l). */
lra_status lra_error_sample(lra_handle h, const lra_operand *W, const double *A, const double *B, int64_t r,
                            const int64_t *rows, int64_t q, const int64_t *cols, int64_t s, double *stats3,
                            void *stream);

/* Progressive-depth pre-processing ("typically at most three recursive steps";
   NEXT-2): for d = 1, 2, ... the sketch with Ms[d-1] (the caller's multipliers of increasing
   depth, realized host-side like any lra_multiplier; real kinds), the C-A (k = l, Y of m x k
   fp64 caller-owned, tol / tie slack 1e-12, swap cap 20 k) with its nucleus and factors into
   I, J, U, A, B, stats, then the superfast estimate est = sqrt(sum g^2 / sum W^2) over the
   rows x cols sample (lra_error_sample, its 4 values left in stats4).  Stops at the first d
   with est <= tol, or at d = nmult; *depth (host) = that d, *estimate (host) = its est, the
   outputs hold that depth's CUR.  Synchronizes the stream once per depth (the stop decision). */
lra_status lra_cur_progressive(lra_handle h, const lra_operand *W, const lra_multiplier *Ms, int32_t nmult, int64_t r,
                               int64_t k, int32_t sweeps, double tol, const int64_t *rows, int64_t q,
                               const int64_t *cols, int64_t s, void *Y, int64_t *I, int64_t *J, double *U, double *A,
                               double *B, lra_ca_stats *stats, double *stats4, int32_t *depth, double *estimate,
                               void *stream);

/* A-priori error certificate of Corollary cowc1 (ii), eq. (eqnrm11), Frobenius
   norm: |W - CUR| <= delta ((|R| + |C| + delta + eta |C||R||U|) xi |U| + 1), C = W[:,J],
   R = W[I,:], U (l x k, device), eta = 1 if r = min(k,l) else 2, (1 - theta) xi = sqrt(k l),
   theta = |U| eta delta with the spectral |U| bounded by |U|_F (reading C27); delta >= the
   Frobenius tail sigma~_{r+1} of W (eq. eqnsgmrfr) is the caller's bound.  out4 (host) =
   { bound (INFINITY when theta >= 1), |C|_F, |R|_F, |U|_F }.  Synchronizes the stream. */
lra_status lra_cur_certificate(lra_handle h, const lra_operand *W, const int64_t *I, const int64_t *J, const double *U,
                               int64_t k, int64_t l, int64_t r, double delta, double *out4 /* host */, void *stream);
/* The customary chi-square rule for the variance of a Gaussian variable: the
   one-sided (1 - alpha) upper confidence bound  K sigma_K^2 / chi2_{K-1}(alpha)  on sigma^2
   (chi-square quantile by Wilson-Hilferty; host scalars, 0 < alpha < 0.5, K >= 2). */
lra_status lra_variance_bound(double var_K, int64_t K, double alpha, double *bound /* host */);

/* A batch of nb independent dense problems (config 3, FMM-style blocks): block b
   is W0 with w = W0.w + b*w_stride elements (w_stride >= ldw*n).  SPARSE_PM1 multipliers may
   differ per block: sp_row / sp_sign of block b start at b*m_stride entries; ARHT / ARFT /
   GAUSSIAN blocks share one multiplier (m_stride must be 0).  Requires lbar == k.  Runs the
   whole path (lra_preprocess, lra_cross_approx, lra_cur_residual) per block; outputs are
   strided per block: I[b*k], J[b*l], U[b*l*k], num2[b], den2[b], stats[b] (may be NULL).
   A block whose generator is singular gets stats[b].status = LRA_ESINGULAR and NaN num2/den2;
   the other blocks are unaffected. */
lra_status lra_batch(lra_handle h, int64_t nb, const lra_operand *W0, int64_t w_stride,
                     const lra_multiplier *M0, int64_t m_stride, int64_t r, int64_t k, int64_t l,
                     int32_t sweeps, double swap_tol, double tie_slack, int32_t swap_cap,
                     int32_t prec, int64_t *I, int64_t *J, double *U, double *num2, double *den2,
                     lra_ca_stats *stats, void *stream);

/* Kernel timing for measurement (bench.py): while enabled, every kernel this handle launches is
   bracketed by a CUDA event pair recorded on its launch stream, and lra_batch runs its groups
   in order on one stream (no concurrent groups), so each interval is that kernel's own device
   time (an isolation pass; the overlapped schedule is timed with profiling disabled).  lra_profile_read synchronizes
   on the recorded events, aggregates per kernel name (name -> total ms, launch count; at most
   cap names, written to host arrays) and resets the record; returns the number of names or a
   negative lra_status.  Enabling resets the record. */
lra_status lra_profile_enable(lra_handle h, int enable);
int lra_profile_read(lra_handle h, int cap, const char **names /* host */, double *ms /* host */,
                     int64_t *counts /* host */);

/* Diagnostics: clock64 cycle counters of the C-A kernel's phases, summed over problems
   (CTA 0, thread 0): [0] block loads, [1] cold LUP, [2] warm-start gather, [3] Gauss-Jordan
   inverse, [4] C = B X^{-1} product, [5] swap loops, [6] whole kernel, [7] pivot steps,
   [8..14] sub-phases of a swap step and of the cluster exchange.
   out16: host array of 16.  Synchronizes the device.  reset != 0 zeroes the counters. */
lra_status lra_debug_counters(uint64_t *out16 /* host */, int reset);

/* Diagnostics: clock64 cycle counters of the tensor-core residual's warp roles, summed over
   CTAs: [0] MMA waits for B slices, [1] MMA waits for a free TMEM buffer, [2] MMA issue,
   [3] producer waits for a free B stage, [4] producer waits for a free A buffer, [5] MMA
   waits for A, [6] epilogue warp 0 waits for accumulators, [7] epilogue warp 0 work,
   [8] tiles.  out16: host array of 16.  Synchronizes the device. */
lra_status lra_debug_counters_residual(uint64_t *out16 /* host */, int reset);

/* Diagnostics level of the handle (default 0).  level >= 1: lra_cross_approx and lra_batch
   fill lra_ca_stats.min_pivot_margin; the C-A then runs on the global-memory tier (its pivots
   are bit-identical to the on-chip tiers') with one extra grid reduction per pivot decision, so
   it is a debugging mode, not a timed configuration.  ARFT (complex) sketches keep their tier
   and report NaN.  EINVAL for level < 0. */
lra_status lra_set_diagnostics(lra_handle h, int32_t level);

/* Diagnostics (builds with -DLRA_CHECK_IDX=1 only; zeros otherwise): the first out-of-range
   data-dependent row / column index seen by a kernel: out4 (host) = { kernel id (1-2 nucleus
   gather, 3-4 factor gathers, 5-6 C-A block gathers), problem, index, bound }; such an index is
   clamped to 0.  Synchronizes the device.  reset != 0 clears the record. */
lra_status lra_debug_index_errors(int64_t *out4 /* host */, int reset);

/* Thread-local message for the last non-OK status (never NULL). */
const char *lra_last_error(void);

/* Number of kernels this library has launched since the handle was created (host counter;
   used by bench.py to report gpu_launches). */
int64_t lra_launch_count(lra_handle h);

#ifdef __cplusplus
}
#endif
#endif /* LRA_H */
