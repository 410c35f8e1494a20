// lra_api.cu — the C-ABI of liblra.so (include/lra.h): handle, scratch, argument checks
// and the launch sequence of each entry point.  No compute happens on the host.
#include <cstdio>
#include <cstdlib>
#include <cstring>
#include <mutex>
#include <string>

#include <cstdarg>

#include <dlfcn.h>
#include <nccl.h>      // types only: the functions are resolved at run time (dlopen)

#include <vector>

#include "kernels.cuh"

using namespace lra;

// ---- NCCL, loaded on first use (no link-time dependency for single-GPU use)
struct NcclApi {
  bool ok = false;
  ncclResult_t (*GetUniqueId)(ncclUniqueId *);
  ncclResult_t (*CommInitRank)(ncclComm_t *, int, ncclUniqueId, int);
  ncclResult_t (*CommDestroy)(ncclComm_t);
  ncclResult_t (*AllReduce)(const void *, void *, size_t, ncclDataType_t, ncclRedOp_t, ncclComm_t, cudaStream_t);
  ncclResult_t (*AllGather)(const void *, void *, size_t, ncclDataType_t, ncclComm_t, cudaStream_t);
  const char *(*GetErrorString)(ncclResult_t);
};
static NcclApi &nccl() {
  static NcclApi api;
  static std::once_flag once;
  std::call_once(once, [] {
    void *lib = dlopen("libnccl.so.2", RTLD_NOW | RTLD_GLOBAL | RTLD_NOLOAD);   // torch's copy if loaded
    if (!lib) lib = dlopen("libnccl.so.2", RTLD_NOW | RTLD_GLOBAL);
    if (!lib) return;
    api.GetUniqueId = (decltype(api.GetUniqueId))dlsym(lib, "ncclGetUniqueId");
    api.CommInitRank = (decltype(api.CommInitRank))dlsym(lib, "ncclCommInitRank");
    api.CommDestroy = (decltype(api.CommDestroy))dlsym(lib, "ncclCommDestroy");
    api.AllReduce = (decltype(api.AllReduce))dlsym(lib, "ncclAllReduce");
    api.AllGather = (decltype(api.AllGather))dlsym(lib, "ncclAllGather");
    api.GetErrorString = (decltype(api.GetErrorString))dlsym(lib, "ncclGetErrorString");
    api.ok = api.GetUniqueId && api.CommInitRank && api.CommDestroy && api.AllReduce && api.AllGather &&
             api.GetErrorString;
  });
  return api;
}

static thread_local std::string g_err = "no error";

static lra_status fail(lra_status s, const char *fmt, ...) {
  char buf[512];
  va_list ap;
  va_start(ap, fmt);
  vsnprintf(buf, sizeof buf, fmt, ap);
  va_end(ap);
  g_err = buf;
  return s;
}

#define CK(call)                                                                              \
  do {                                                                                        \
    cudaError_t e_ = (call);                                                                  \
    if (e_ != cudaSuccess) return fail(LRA_ECUDA, "%s: %s", #call, cudaGetErrorString(e_));   \
  } while (0)

#define NK(call)                                                                              \
  do {                                                                                        \
    ncclResult_t r_ = (call);                                                                 \
    if (r_ != ncclSuccess) return fail(LRA_ENCCL, "%s: %s", #call, nccl().GetErrorString(r_));  \
  } while (0)

#define LRA_NSIDE 8
struct lra_handle_s {
  int device;
  int groups_env;                 // lra_batch groups from env LRA_BATCH_GROUPS (0: automatic)
  cudaStream_t side[LRA_NSIDE];
  cudaEvent_t fork, join[LRA_NSIDE];
  bool streams_ready;
  int nranks, rank;
  ncclComm_t comm;                // row-sharded path (nullptr: single GPU)
  int64_t launches;
  Prof prof;
  // scratch arena (grows; reused)
  void *ws;
  size_t ws_bytes;
  void *gs;                       // grid-tier exchange buffers
  size_t gs_bytes;
  void *gm;                       // global-memory C-A tier (block + C-matrix)
  size_t gm_bytes;
  void *sh;                       // row-sharded path: assembled blocks
  size_t sh_bytes;
  void *qg;                       // quasi-Gaussian multiplier: built omega + integer work
  size_t qg_bytes;
  int diag;                       // lra_set_diagnostics level
  void *sk;                       // tensor-core Gaussian sketch scratch (one slot per side stream)
  size_t sk_bytes;
};

static lra_status ensure_streams(lra_handle h) {
  if (h->streams_ready) return LRA_OK;
  for (int i = 0; i < LRA_NSIDE; ++i) {
    CK(cudaStreamCreateWithFlags(&h->side[i], cudaStreamNonBlocking));
    CK(cudaEventCreateWithFlags(&h->join[i], cudaEventDisableTiming));
  }
  CK(cudaEventCreateWithFlags(&h->fork, cudaEventDisableTiming));
  h->streams_ready = true;
  return LRA_OK;
}

static lra_status ws_reserve(lra_handle h, size_t bytes) {
  if (bytes <= h->ws_bytes) return LRA_OK;
  if (h->ws) cudaFree(h->ws);
  h->ws = nullptr;
  h->ws_bytes = 0;
  size_t want = bytes + bytes / 4;
  if (cudaMalloc(&h->ws, want) != cudaSuccess) {
    cudaGetLastError();
    return fail(LRA_ENOMEM, "cannot allocate %zu bytes of scratch", want);
  }
  h->ws_bytes = want;
  return LRA_OK;
}

// Exact-size reservation of one of the handle's secondary device buffers (grid-tier exchange,
// global-memory C-A tier, sharded blocks).
static lra_status buf_reserve(void **buf, size_t *have, size_t bytes, const char *what) {
  if (bytes <= *have) return LRA_OK;
  if (*buf) cudaFree(*buf);
  *buf = nullptr;
  *have = 0;
  if (cudaMalloc(buf, bytes) != cudaSuccess) {
    cudaGetLastError();
    return fail(LRA_ENOMEM, "cannot allocate %zu bytes for %s", bytes, what);
  }
  *have = bytes;
  return LRA_OK;
}

struct Carve {
  char *base;
  size_t off;
  template <typename T>
  T *take(size_t count) {
    off = (off + 255) & ~(size_t)255;
    T *p = reinterpret_cast<T *>(base + off);
    off += count * sizeof(T);
    return p;
  }
};

static OpView make_view(const lra_operand *W) {
  OpView v{};
  v.kind = W->kind;
  v.dtype = W->dtype;
  v.m = W->m;
  v.n = W->n;
  v.w = W->w;
  v.ldw = W->ldw;
  v.f.fa = W->fa;
  v.f.fb = W->fb;
  v.f.m = W->m;
  v.f.p = W->p;
  v.f.rowptr = W->e_rowptr;
  v.f.col = W->e_col;
  v.f.val = W->e_val;
  return v;
}

static lra_status check_operand(const lra_operand *W) {
  if (!W) return fail(LRA_EINVAL, "null operand");
  if (W->m < 1 || W->n < 1) return fail(LRA_EINVAL, "empty operand (m=%lld, n=%lld)", (long long)W->m, (long long)W->n);
  if (W->m_global < 0 || W->row0 < 0 || (W->m_global > 0 && W->row0 + W->m > W->m_global))
    return fail(LRA_EINVAL, "bad row shard (row0 = %lld, m = %lld, m_global = %lld)", (long long)W->row0,
                (long long)W->m, (long long)W->m_global);
  if (W->m_global > 0 && W->kind != LRA_OP_DENSE) return fail(LRA_EINVAL, "only dense operands are row-sharded");
  if (W->kind == LRA_OP_DENSE) {
    if (!W->w) return fail(LRA_EINVAL, "dense operand with null w");
    if (W->ldw < W->m) return fail(LRA_EINVAL, "ldw < m");
    if (W->dtype != LRA_F32 && W->dtype != LRA_F64) return fail(LRA_EINVAL, "bad dtype");
  } else if (W->kind == LRA_OP_FACTORED_CSR) {
    if (!W->fa || !W->fb || !W->e_rowptr || W->p < 1) return fail(LRA_EINVAL, "factored operand incomplete");
  } else {
    return fail(LRA_EINVAL, "bad operand kind");
  }
  return LRA_OK;
}

static lra_status check_device(lra_handle h) {
  if (!h) return fail(LRA_EINVAL, "null handle");
  int n = 0;
  if (cudaGetDeviceCount(&n) != cudaSuccess || n == 0) {
    cudaGetLastError();
    return fail(LRA_ECUDA, "no CUDA device (this library has no CPU fallback)");
  }
  CK(cudaSetDevice(h->device));
  return LRA_OK;
}

static lra_status check_mult(const lra_multiplier *M, int64_t n) {
  if (!M) return fail(LRA_EINVAL, "null multiplier");
  if (M->lbar < 1 || M->lbar > n) return fail(LRA_EINVAL, "lbar out of range");
  switch (M->kind) {
    case LRA_MUL_ARHT:
    case LRA_MUL_ARFT:
      if (M->depth < 1 || M->depth > 6 || (n % ((int64_t)1 << M->depth)) != 0)
        return fail(LRA_EINVAL, "need 1 <= depth <= 6 and 2^depth | n (reading C21)");
      if (!M->dsign || !M->col) return fail(LRA_EINVAL, "ARHT/ARFT needs dsign and col");
      return LRA_OK;
    case LRA_MUL_SPARSE_PM1:
      if (!M->sp_row || !M->sp_sign || M->nnz_per_col < 1 || M->nnz_per_col > 64)
        return fail(LRA_EINVAL, "sparse multiplier needs sp_row, sp_sign, 1 <= nnz <= 64");
      return LRA_OK;
    case LRA_MUL_GAUSSIAN:
      if (!M->omega || M->ld_omega < n) return fail(LRA_EINVAL, "gaussian multiplier needs omega, ld >= n");
      return LRA_OK;
    case LRA_MUL_QGAUSS:
      if (M->depth < 1 || M->depth > 30 || !M->qg_sign || !M->qg_perm || !M->col)
        return fail(LRA_EINVAL, "quasi-Gaussian multiplier needs 1 <= depth <= 30, qg_sign, qg_perm, col");
      return LRA_OK;
    default:
      return fail(LRA_EINVAL, "bad multiplier kind");
  }
}

static SketchArgs make_sketch(const lra_operand *W, const lra_multiplier *M, void *Y, int64_t ldy) {
  SketchArgs a{};
  a.kind = M->kind;
  a.dtype = W->dtype;
  a.depth = M->depth;
  a.nnz = M->nnz_per_col;
  a.m = W->m;
  a.n = W->n;
  a.lbar = M->lbar;
  a.ldw = W->ldw;
  a.ldy = ldy;
  a.w = W->w;
  a.dsign = M->dsign;
  a.col = M->col;
  a.sp_row = M->sp_row;
  a.sp_sign = M->sp_sign;
  a.y = Y;
  return a;
}

// A quasi-Gaussian multiplier is realized as its lbar sampled columns Omega = G_q[:, col]
// (exact integers, built on the device into the handle's qg buffer) and then applied exactly
// like a Gaussian omega; every other kind passes through unchanged.
static lra_status resolve_mult(lra_handle h, const lra_multiplier *M, int64_t n, cudaStream_t st,
                               lra_multiplier *out) {
  *out = *M;
  if (M->kind != LRA_MUL_QGAUSS) return LRA_OK;
  const size_t need = (size_t)n * M->lbar * (8 + 2 * 4) + 256;
  lra_status s;
  if ((s = buf_reserve(&h->qg, &h->qg_bytes, need, "the quasi-Gaussian multiplier")) != LRA_OK) return s;
  double *omega = (double *)h->qg;
  int *work = (int *)(omega + (size_t)n * M->lbar);
  CK(launch_qg_build(n, M->depth, M->lbar, M->qg_sign, M->qg_perm, M->col, work, omega, st, &h->prof));
  h->launches += 1;
  out->kind = LRA_MUL_GAUSSIAN;
  out->omega = omega;
  out->ld_omega = n;
  return LRA_OK;
}

// Tensor-core Gaussian sketch (sketch_tc.cu, reading C36): scratch for nslots concurrent calls
// of nb problems each; *per = 0 (SIMT kernel) for the other multiplier kinds or with
// LRA_SKETCH_SIMT=1 (diagnostics: the order-preserving DFMA kernel, bit-identical to the oracle).
static lra_status sketch_scratch(lra_handle h, const lra_multiplier *M, int64_t m, int64_t n, int64_t nb, int nslots,
                                 size_t *per) {
  static const bool simt = getenv("LRA_SKETCH_SIMT") != nullptr;
  *per = 0;
  if (M->kind != LRA_MUL_GAUSSIAN || simt) return LRA_OK;
  const size_t b = (sketch_tc_scratch_bytes(m, n, M->lbar, nb) + 255) & ~(size_t)255;
  lra_status s;
  void *before = h->sk;
  if ((s = buf_reserve(&h->sk, &h->sk_bytes, b * nslots, "the tensor-core sketch")) != LRA_OK) return s;
  if (h->sk != before)   // fresh buffer: the split-tile accumulators / counters start at zero
    for (int i = 0; i < nslots; ++i) CK(cudaMemset((char *)h->sk + i * b, 0, sketch_tc_zero_bytes()));
  *per = b;
  return LRA_OK;
}

// Reconstruction path of the full residual: fp32 W (or FAST) -> tensor-core
// Ozaki kernel with S = 6 (PRECISE) / 3 (FAST) balanced base-256 digit slices; fp64 W in
// PRECISE mode -> fp64 SIMT kernel.  LRA_RESID_SIMT=1 forces the SIMT kernel (diagnostics).
static int resid_slices(int dtype, int prec) {
  static const bool simt = getenv("LRA_RESID_SIMT") != nullptr;
  if (prec == LRA_RECON_FAST) return 3;
  if (dtype == LRA_F32 && !simt) return 6;
  return 0;
}
static size_t resid_scratch(int64_t m, int64_t n, int64_t r, int S, int64_t nb) {
  const int64_t simt_tiles = ((m + 127) / 128) * ((n + 127) / 128);
  const int64_t tc_parts = residual_tc_partials(m, n);
  size_t bytes = (size_t)nb * (simt_tiles > tc_parts ? simt_tiles : tc_parts) * sizeof(double2) + 256;
  if (S) bytes += residual_tc_scratch(m, n, (int)r, S, nb) + 256;
  return bytes;
}
static int64_t resid_partials(int64_t m, int64_t n) {
  const int64_t simt_tiles = ((m + 127) / 128) * ((n + 127) / 128);
  const int64_t tc_parts = residual_tc_partials(m, n);
  return simt_tiles > tc_parts ? simt_tiles : tc_parts;
}

extern "C" {

const char *lra_last_error(void) { return g_err.c_str(); }

lra_status lra_handle_create(lra_handle *h, int device, const void *nccl_unique_id, int nranks, int rank) {
  if (!h) return fail(LRA_EINVAL, "null handle pointer");
  *h = nullptr;
  if (nranks < 1 || rank < 0 || rank >= nranks) return fail(LRA_EINVAL, "bad nranks / rank");
  if (nranks > 1 && !nccl_unique_id) return fail(LRA_EINVAL, "nranks > 1 needs an NCCL unique id");
  int n = 0;
  if (cudaGetDeviceCount(&n) != cudaSuccess || n == 0) {
    cudaGetLastError();
    return fail(LRA_ECUDA, "no CUDA device (this library has no CPU fallback)");
  }
  if (device < 0 || device >= n) return fail(LRA_EINVAL, "bad device %d", device);
  CK(cudaSetDevice(device));
  lra_handle_s *p = new lra_handle_s();
  p->device = device;
  const char *g = getenv("LRA_BATCH_GROUPS");
  p->groups_env = g ? atoi(g) : 0;
  if (p->groups_env < 0) p->groups_env = 0;
  p->nranks = nranks;
  p->rank = rank;
  p->comm = nullptr;
  if (nccl_unique_id) {
    if (!nccl().ok) {
      delete p;
      return fail(LRA_ENCCL, "libnccl.so.2 could not be loaded");
    }
    ncclUniqueId id;
    memcpy(&id, nccl_unique_id, sizeof(id));
    ncclResult_t r = nccl().CommInitRank(&p->comm, nranks, id, rank);
    if (r != ncclSuccess) {
      delete p;
      return fail(LRA_ENCCL, "ncclCommInitRank: %s", nccl().GetErrorString(r));
    }
  }
  *h = p;
  return LRA_OK;
}

lra_status lra_nccl_unique_id(void *out) {
  if (!out) return fail(LRA_EINVAL, "null output");
  if (!nccl().ok) return fail(LRA_ENCCL, "libnccl.so.2 could not be loaded");
  ncclUniqueId id;
  NK(nccl().GetUniqueId(&id));
  memcpy(out, &id, sizeof(id));
  return LRA_OK;
}

void lra_handle_destroy(lra_handle h) {
  if (!h) return;
  if (h->ws) cudaFree(h->ws);
  if (h->gs) cudaFree(h->gs);
  if (h->gm) cudaFree(h->gm);
  if (h->sh) cudaFree(h->sh);
  if (h->qg) cudaFree(h->qg);
  if (h->comm) nccl().CommDestroy(h->comm);
  for (cudaEvent_t e : h->prof.ev) cudaEventDestroy(e);
  if (h->streams_ready) {
    for (int i = 0; i < LRA_NSIDE; ++i) {
      cudaStreamDestroy(h->side[i]);
      cudaEventDestroy(h->join[i]);
    }
    cudaEventDestroy(h->fork);
  }
  delete h;
}

lra_status lra_profile_enable(lra_handle h, int enable) {
  if (!h) return fail(LRA_EINVAL, "null handle");
  h->prof.on = enable ? 1 : 0;
  h->prof.used = 0;
  return LRA_OK;
}

int lra_profile_read(lra_handle h, int cap, const char **names, double *ms, int64_t *counts) {
  if (!h) return fail(LRA_EINVAL, "null handle");
  Prof &p = h->prof;
  int nd = 0;
  for (size_t i = 0; i + 1 < p.used; i += 2) {
    float t = 0.f;
    if (cudaEventSynchronize(p.ev[i + 1]) != cudaSuccess || cudaEventElapsedTime(&t, p.ev[i], p.ev[i + 1]) != cudaSuccess) {
      cudaGetLastError();
      return fail(LRA_ECUDA, "profile event read failed");
    }
    const char *nm = p.name[i / 2];
    int d = 0;
    while (d < nd && strcmp(names[d], nm) != 0) ++d;
    if (d == nd) {
      if (nd == cap) continue;
      names[nd] = nm;
      ms[nd] = 0.0;
      counts[nd] = 0;
      ++nd;
    }
    ms[d] += t;
    counts[d] += 1;
  }
  p.used = 0;
  return nd;
}

int64_t lra_launch_count(lra_handle h) { return h ? h->launches : 0; }

lra_status lra_debug_counters(uint64_t *out8, int reset) {
  if (!out8 /* 16 entries */) return fail(LRA_EINVAL, "null output");
  CK(read_ca_counters((unsigned long long *)out8, reset != 0));
  return LRA_OK;
}

lra_status lra_set_diagnostics(lra_handle h, int32_t level) {
  if (!h || level < 0) return fail(LRA_EINVAL, "need a handle and level >= 0");
  h->diag = level;
  return LRA_OK;
}

lra_status lra_debug_index_errors(int64_t *out4, int reset) {
  if (!out4) return fail(LRA_EINVAL, "null output");
  long long a[4], c[4];
  CK(read_idx_err_nuc(a, reset != 0));
  CK(read_idx_err_cc(c, reset != 0));
  for (int i = 0; i < 4; ++i) out4[i] = a[0] ? a[i] : c[i];
  return LRA_OK;
}

lra_status lra_debug_counters_residual(uint64_t *out16, int reset) {
  if (!out16) return fail(LRA_EINVAL, "null output");
  CK(read_rtc_counters((unsigned long long *)out16, reset != 0));
  return LRA_OK;
}

lra_status lra_preprocess(lra_handle h, const lra_operand *W, const lra_multiplier *M, void *Y, int64_t ldy,
                          void *stream) {
  lra_status s;
  if ((s = check_device(h)) != LRA_OK) return s;
  if ((s = check_operand(W)) != LRA_OK) return s;
  if (W->kind != LRA_OP_DENSE) return fail(LRA_EINVAL, "lra_preprocess needs a dense operand");
  if ((s = check_mult(M, W->n)) != LRA_OK) return s;
  if (!Y || ldy < W->m) return fail(LRA_EINVAL, "Y null or ldy < m");
  lra_multiplier Mr;
  if ((s = resolve_mult(h, M, W->n, (cudaStream_t)stream, &Mr)) != LRA_OK) return s;
  SketchArgs a = make_sketch(W, &Mr, Y, ldy);
  size_t per = 0;
  if ((s = sketch_scratch(h, &Mr, W->m, W->n, 1, 1, &per)) != LRA_OK) return s;
  CK(launch_sketch(a, 1, Mr.omega, Mr.ld_omega, (cudaStream_t)stream, &h->prof, per ? h->sk : nullptr, per));
  h->launches += per ? 2 : 1;
  return LRA_OK;
}

lra_status lra_preprocess_full(lra_handle h, const lra_operand *W, const lra_multiplier *M, void *Wout, int64_t ldo,
                               void *stream) {
  lra_status s;
  if ((s = check_device(h)) != LRA_OK) return s;
  if ((s = check_operand(W)) != LRA_OK) return s;
  if (W->kind != LRA_OP_DENSE || W->m_global > 0) return fail(LRA_EINVAL, "lra_preprocess_full needs an unsharded dense operand");
  if ((s = check_mult(M, W->n)) != LRA_OK) return s;
  if (M->kind != LRA_MUL_ARHT) return fail(LRA_EUNSUPPORTED, "full pre-processing is implemented for ARHT");
  if (M->lbar != W->n) return fail(LRA_EINVAL, "full pre-processing needs lbar == n (col = the whole permutation P)");
  if (M->depth > 5) return fail(LRA_EUNSUPPORTED, "full pre-processing supports depth <= 5");
  if (!Wout || ldo < W->m) return fail(LRA_EINVAL, "Wout null or ldo < m");
  if ((s = ws_reserve(h, (size_t)W->n * sizeof(int) + 256)) != LRA_OK) return s;
  SketchArgs a = make_sketch(W, M, Wout, ldo);
  CK(launch_transform_full(a, (int *)h->ws, Wout, ldo, (cudaStream_t)stream, &h->prof));
  h->launches += 2;
  return LRA_OK;
}

static lra_status check_ca_shape(const lra_operand *W, int64_t r, int64_t k, int64_t l, int32_t sweeps) {
  if (k != l) return fail(LRA_EINVAL, "v1 requires k == l (reading C9)");
  if (r < 1 || r > k) return fail(LRA_EINVAL, "need 0 < r <= k");
  const int64_t mg = W->m_global > 0 ? W->m_global : W->m;
  if (k > mg || l > W->n) return fail(LRA_EINVAL, "need k <= m and l <= n");
  if (k > LRA_QMAX_ALL) return fail(LRA_EUNSUPPORTED, "k > %d is outside this build's maxvol tiers", LRA_QMAX_ALL);
  if (sweeps < 1) return fail(LRA_EINVAL, "sweeps >= 1");
  return LRA_OK;
}

// The whole C-A -> nucleus -> factors chain for nb problems sharing shapes.
static lra_status run_chain(lra_handle h, const lra_operand *W, int64_t w_stride, const void *Y, int64_t ldy,
                            int64_t y_stride, int y_complex, const int64_t *I0, int64_t r, int64_t k,
                            int32_t sweeps, double tol, double tau, int32_t cap, int64_t *I, int64_t *J,
                            double *U, double *A, double *B, int64_t a_stride, int64_t b_stride,
                            lra_ca_stats *stats, int32_t *status, double *TS, double *Sr, int32_t *yinfo,
                            int64_t nb, cudaStream_t st) {
  CAArgs ca{};
  ca.op = make_view(W);
  ca.w_stride = w_stride;
  ca.Y = Y;
  ca.ldy = ldy;
  ca.y_stride = y_stride;
  ca.y_complex = y_complex;
  ca.I0 = I0;
  ca.i0_stride = k;
  ca.q = (int)k;
  ca.sweeps = sweeps;
  ca.cap = cap;
  ca.qp = (int)(k | 1);
  ca.tol = tol;
  ca.tau = tau;
  ca.I = I;
  ca.J = J;
  ca.stats = stats;
  ca.status = status;
  ca.yinfo = y_complex ? yinfo : nullptr;
  ca.grid = 0;
  ca.diag = (h->diag > 0 && !y_complex) ? 1 : 0;   // margins: measured on the global tier
  lra_status rs;
  if ((rs = buf_reserve(&h->gs, &h->gs_bytes, ca_grid_scratch_bytes(160), "the grid-tier exchange")) != LRA_OK)
    return rs;
  ca.gscratch = h->gs;
  int cs = 0;
  const int64_t maxN = W->m > W->n ? W->m : W->n;
  cudaError_t e;
  if (ca_needs_global(maxN, (int)k) || ca.diag) {
    if (y_complex) return fail(LRA_EUNSUPPORTED, "ARFT sketch with a block beyond the on-chip tiers");
    if ((rs = buf_reserve(&h->gm, &h->gm_bytes, ca_global_scratch_bytes(maxN, (int)k), "the global-memory C-A tier")) != LRA_OK)
      return rs;
    e = launch_ca_global(ca, nb, maxN, h->gm, st, &h->prof);
    if (e == cudaSuccess) h->launches += nb;
  } else {
    e = launch_ca(ca, nb, maxN, st, &cs, &h->prof);
    if (e == cudaSuccess) h->launches += 1;
  }
  if (e == cudaErrorInvalidConfiguration)
    return fail(LRA_EUNSUPPORTED, "block %lld x %lld exceeds the C-A tiers", (long long)maxN, (long long)k);
  CK(e);
  NucArgs na{};
  na.op = ca.op;
  na.w_stride = w_stride;
  na.I = I;
  na.J = J;
  na.k = (int)k;
  na.l = (int)k;
  na.r = (int)r;
  na.U = U;
  na.TS = TS;
  na.Sr = Sr;
  na.status = status;
  na.stats = stats;
  FacArgs fa{};
  fa.op = ca.op;
  fa.w_stride = w_stride;
  fa.I = I;
  fa.J = J;
  fa.k = (int)k;
  fa.l = (int)k;
  fa.r = (int)r;
  fa.TS = TS;
  fa.Sr = Sr;
  fa.A = A;
  fa.B = B;
  fa.a_stride = a_stride;
  fa.b_stride = b_stride;
  fa.status = status;
  int nl = 0;
  CK(launch_nucleus(na, fa, nb, st, &nl, &h->prof));
  h->launches += nl;
  return LRA_OK;
}

// ---------------------------------------------------------------- row-sharded C-A
// One standalone maxvol (Alg D.2 stage 1 / D.1) on a dense fp64 block (N x q col-major):
// cold (LUP) when start == nullptr, else warm from the slots `start`; slots -> out.
static lra_status maxvol_block(lra_handle h, const double *blk, int64_t N, int q, const int64_t *start, int64_t *out,
                               double tol, double tau, int32_t cap, lra_ca_stats *st_dev, int32_t *status,
                               int64_t *dummyJ, cudaStream_t st, const int32_t *skip = nullptr) {
  CAArgs ca{};
  ca.op.kind = LRA_OP_DENSE;
  ca.op.dtype = LRA_F64;
  ca.op.m = N;
  ca.op.n = N;
  ca.op.w = blk;
  ca.op.ldw = N;
  ca.Y = blk;
  ca.ldy = N;
  ca.I0 = start;
  ca.i0_stride = q;
  ca.y_warm = start ? 1 : 0;
  ca.q = q;
  ca.qp = q | 1;
  ca.sweeps = 0;
  ca.cap = cap;
  ca.tol = tol;
  ca.tau = tau;
  ca.I = out;
  ca.J = dummyJ;
  ca.stats = st_dev;
  ca.status = status;
  ca.skip = skip;
  cudaError_t e;
  const bool cluster = !ca_needs_global(N, q) && q <= 48 && N <= 16 * (q <= 24 ? 512 : 256);
  if (cluster) {
    int cs = 0;
    e = launch_ca_cluster(ca, 1, N, st, &cs, &h->prof);
  } else {
    lra_status rs;
    if ((rs = buf_reserve(&h->gm, &h->gm_bytes, ca_global_scratch_bytes(N, q), "the global-memory C-A tier")) != LRA_OK)
      return rs;
    e = launch_ca_global(ca, 1, N, h->gm, st, &h->prof);
  }
  if (e == cudaErrorInvalidConfiguration) return fail(LRA_EUNSUPPORTED, "block %lld x %d exceeds the C-A tiers", (long long)N, q);
  CK(e);
  h->launches += 1;
  return LRA_OK;
}

// The standard row split used by the allgather assembly: rank g holds rows [g cm, g cm + m_g),
// cm = ceil(m / G).  Other splits are accepted and assembled by the owner-scatter + sum path.
static bool standard_split(const lra_operand *W, int nranks, int rank, int64_t *cm_out) {
  const int64_t M = W->m_global, cm = (M + nranks - 1) / nranks;
  const int64_t r0 = (int64_t)rank * cm, ml = M - r0 < cm ? M - r0 : cm;
  *cm_out = cm;
  return W->row0 == r0 && W->m == ml;
}

static size_t sharded_scratch(int64_t M, int64_t n, int64_t r, int64_t q, int32_t sweeps, int nranks) {
  const int64_t Nmax = M > n ? M : n;
  const int64_t cm = (M + nranks - 1) / nranks;
  Carve probe{nullptr, 0};
  probe.take<double>((size_t)Nmax * q);         // assembled block
  probe.take<double>((size_t)n * q);            // R^T for the final factor B
  probe.take<double>((size_t)q * q);            // G
  probe.take<double>((size_t)q * r);            // TS
  probe.take<double>((size_t)q * r);            // Sr
  probe.take<lra_ca_stats>((size_t)(2 * sweeps + 1));
  probe.take<int32_t>(4);
  probe.take<int64_t>((size_t)q);               // dummy J output of standalone maxvol calls
  probe.take<int32_t>(4);                       // chain control flags
  probe.take<double>((size_t)cm * q);           // allgather: this rank's chunk
  probe.take<double>((size_t)nranks * cm * q);  // allgather: all chunks
  return probe.off + 256;
}

static lra_status allreduce_sum(lra_handle h, double *buf, size_t count, cudaStream_t st) {
  if (h->nranks == 1 && !h->comm) return LRA_OK;
  NK(nccl().AllReduce(buf, buf, count, ncclFloat64, ncclSum, h->comm, st));
  return LRA_OK;
}
static lra_status allgather(lra_handle h, const double *chunk, double *all, size_t count, cudaStream_t st) {
  if (h->nranks == 1 && !h->comm) {
    CK(cudaMemcpyAsync(all, chunk, count * sizeof(double), cudaMemcpyDeviceToDevice, st));
    return LRA_OK;
  }
  NK(nccl().AllGather(chunk, all, count, ncclFloat64, h->comm, st));
  return LRA_OK;
}

static lra_status sharded_cross_approx(lra_handle h, const lra_operand *W, const void *Y, int64_t ldy,
                                       const int64_t *I0, int64_t r, int64_t k, int32_t sweeps, double tol,
                                       double tau, int32_t cap, int64_t *I, int64_t *J, double *U, double *A,
                                       double *B, lra_ca_stats *stats, cudaStream_t st) {
  if (!h->comm && h->nranks > 1) return fail(LRA_ENCCL, "row-sharded operand needs an NCCL communicator");
  const int64_t M = W->m_global, n = W->n, q = k;
  const int64_t Nmax = M > n ? M : n;
  lra_status rs;
  if ((rs = buf_reserve(&h->sh, &h->sh_bytes, sharded_scratch(M, n, r, k, sweeps, h->nranks), "the sharded blocks")) !=
      LRA_OK)
    return rs;
  int64_t cm = 0;
  const bool gather = standard_split(W, h->nranks, h->rank, &cm);
  Carve cv{(char *)h->sh, 0};
  double *blk = cv.take<double>((size_t)Nmax * q);
  double *Rt = cv.take<double>((size_t)n * q);
  double *G = cv.take<double>((size_t)q * q);
  double *TS = cv.take<double>((size_t)q * r);
  double *Sr = cv.take<double>((size_t)q * r);
  lra_ca_stats *sts = cv.take<lra_ca_stats>((size_t)(2 * sweeps + 1));
  int32_t *status = cv.take<int32_t>(4);
  int64_t *dJ = cv.take<int64_t>((size_t)q);
  int32_t *ctl = cv.take<int32_t>(4);
  double *chunk = cv.take<double>((size_t)cm * q);
  double *chunks = cv.take<double>((size_t)h->nranks * cm * q);
  const OpView op = make_view(W);                 // local rows (op.m = m_local)
  lra_status s;
  // The whole chain is stream-ordered: maxvol calls after a failure or after convergence do
  // nothing (CAArgs::skip <- ctl), the early-exit rule and the statistics are evaluated on the
  // device (k_ctl_step / k_ctl_combine), so the call never synchronizes the host and can be
  // captured in a CUDA graph.  Every rank issues the same collectives in the same order.
  CK(cudaMemsetAsync(status, 0, 4 * sizeof(int32_t), st));
  CK(cudaMemsetAsync(ctl, 0, 4 * sizeof(int32_t), st));
  CK(cudaMemsetAsync(sts, 0, (size_t)(2 * sweeps + 1) * sizeof(lra_ca_stats), st));
  // blocks whose rows are the sharded rows: allgather of the packed local rows (standard
  // split), else owner scatter + sum
  auto assemble_rows = [&](bool from_y, const int64_t *Jc) -> lra_status {
    lra_status s2;
    if (gather) {
      if (from_y) CK(launch_pack_rows((const double *)Y, ldy, W->m, (int)q, cm, chunk, st));
      else CK(launch_pack_wcols(op, Jc, (int)q, cm, chunk, st));
      if ((s2 = allgather(h, chunk, chunks, (size_t)cm * q, st)) != LRA_OK) return s2;
      CK(launch_unpack_chunks(chunks, cm, (int)q, h->nranks, M, blk, st));
      h->launches += 2;
      return LRA_OK;
    }
    CK(cudaMemsetAsync(blk, 0, (size_t)M * q * sizeof(double), st));
    if (from_y) CK(launch_scatter_rows((const double *)Y, ldy, W->m, (int)q, W->row0, M, blk, st));
    else CK(launch_scatter_wcols(op, Jc, (int)q, W->row0, M, blk, st));
    h->launches += 1;
    return allreduce_sum(h, blk, (size_t)M * q, st);
  };
  int nst = 0;
  // stage 2: I <- maxvol(Y) on the assembled m_global x lbar sketch, or the given I0
  if (Y) {
    if ((s = assemble_rows(true, nullptr)) != LRA_OK) return s;
    if ((s = maxvol_block(h, blk, M, (int)q, nullptr, I, tol, tau, cap, sts + nst, status, dJ, st, ctl)) != LRA_OK)
      return s;
    CK(launch_ctl_step(sts, nst, 0, 0, ctl, st));
    ++nst;
  } else {
    CK(cudaMemcpyAsync(I, I0, q * sizeof(int64_t), cudaMemcpyDeviceToDevice, st));
  }
  for (int loop = 0; loop < sweeps; ++loop) {
    // horizontal: J <- maxvol(W[I,:]^T) (cold in loop 0, else warm from J); row I[s] is owned
    // by one rank: owner scatter + sum
    CK(cudaMemsetAsync(blk, 0, (size_t)n * q * sizeof(double), st));
    CK(launch_scatter_wrows(op, I, (int)q, W->row0, blk, st));
    if ((s = allreduce_sum(h, blk, (size_t)n * q, st)) != LRA_OK) return s;
    if ((s = maxvol_block(h, blk, n, (int)q, loop ? J : nullptr, J, tol, tau, cap, sts + nst, status, dJ, st, ctl)) !=
        LRA_OK)
      return s;
    CK(launch_ctl_step(sts, nst, 1, loop, ctl, st));
    ++nst;
    // vertical: I <- maxvol(W[:,J]) warm from I
    if ((s = assemble_rows(false, J)) != LRA_OK) return s;
    if ((s = maxvol_block(h, blk, M, (int)q, I, I, tol, tau, cap, sts + nst, status, dJ, st, ctl)) != LRA_OK) return s;
    CK(launch_ctl_step(sts, nst, 2, loop, ctl, st));
    ++nst;
    h->launches += 4;
  }
  if (stats) {   // the per-call statistics combined on the device as the fused kernel reports them
    CK(launch_ctl_combine(sts, ctl, Y ? 1 : 0, stats, st));
    h->launches += 1;
  }
  {
    // nucleus and factors: G = W[I,J] and R = W[I,:] assembled, the replicated Jacobi SVD
    // (skipped on device when a step failed: the kernels read `status`)
    CK(cudaMemsetAsync(Rt, 0, (size_t)n * q * sizeof(double), st));
    CK(launch_scatter_wrows(op, I, (int)q, W->row0, Rt, st));
    if ((s = allreduce_sum(h, Rt, (size_t)n * q, st)) != LRA_OK) return s;
    CK(cudaMemsetAsync(G, 0, (size_t)q * q * sizeof(double), st));
    CK(launch_scatter_g(op, I, J, (int)q, (int)q, W->row0, G, st));
    if ((s = allreduce_sum(h, G, (size_t)q * q, st)) != LRA_OK) return s;
    NucArgs na{};
    na.op = op;
    na.I = I;
    na.J = J;
    na.k = (int)q;
    na.l = (int)q;
    na.r = (int)r;
    na.U = U;
    na.TS = TS;
    na.Sr = Sr;
    na.status = status;
    na.Gd = G;
    na.stats = stats;
    FacArgs fa{};
    fa.op = op;
    fa.I = I;
    fa.J = J;
    fa.k = (int)q;
    fa.l = (int)q;
    fa.r = (int)r;
    fa.TS = TS;
    fa.Sr = Sr;
    fa.A = A;
    fa.B = B;
    fa.status = status;
    fa.Rt = Rt;
    int nl = 0;
    CK(launch_nucleus(na, fa, 1, st, &nl, &h->prof));
    h->launches += nl + 2;
  }
  return LRA_OK;
}

static size_t chain_scratch(int64_t r, int64_t k) {
  Carve probe{nullptr, 0};
  probe.take<int32_t>(1);
  probe.take<double>((size_t)k * r);
  probe.take<double>((size_t)k * r);
  probe.take<int32_t>(4);
  return probe.off + 256;
}

lra_status lra_cross_approx(lra_handle h, const lra_operand *W, const void *Y, int64_t ldy, int y_complex,
                            const int64_t *I0, int64_t r, int64_t k, int64_t l, int32_t sweeps, double swap_tol,
                            double tie_slack, int32_t swap_cap, int64_t *I, int64_t *J, double *U, double *A,
                            double *B, lra_ca_stats *stats, void *stream) {
  lra_status s;
  if ((s = check_device(h)) != LRA_OK) return s;
  if ((s = check_operand(W)) != LRA_OK) return s;
  if ((s = check_ca_shape(W, r, k, l, sweeps)) != LRA_OK) return s;
  if (!Y && !I0) return fail(LRA_EINVAL, "need a sketch Y or a start set I0");
  if (Y && ldy < W->m) return fail(LRA_EINVAL, "ldy < m");
  if (!I || !J || !A || !B) return fail(LRA_EINVAL, "null output");
  if (!(swap_tol >= 0.0) || !(tie_slack >= 0.0) || tie_slack >= 1.0 || swap_cap < 0)
    return fail(LRA_EINVAL, "bad swap_tol / tie_slack / swap_cap");
  if (W->m_global > 0) {
    if (y_complex) return fail(LRA_EUNSUPPORTED, "ARFT sketches are not row-sharded in this build");
    return sharded_cross_approx(h, W, Y, ldy, I0, r, k, sweeps, swap_tol, tie_slack, swap_cap, I, J, U, A, B,
                                stats, (cudaStream_t)stream);
  }
  if ((s = ws_reserve(h, chain_scratch(r, k))) != LRA_OK) return s;
  Carve cv{(char *)h->ws, 0};
  int32_t *status = cv.take<int32_t>(1);
  double *TS = cv.take<double>((size_t)k * r);
  double *Sr = cv.take<double>((size_t)k * r);
  int32_t *yinfo = cv.take<int32_t>(4);
  cudaStream_t st = (cudaStream_t)stream;
  CK(cudaMemsetAsync(status, 0, sizeof(int32_t), st));
  s = run_chain(h, W, 0, Y, ldy, 0, y_complex, Y ? nullptr : I0, r, k, sweeps, swap_tol, tie_slack, swap_cap, I, J,
                U, A, B, 0, 0, stats, status, TS, Sr, yinfo, 1, st);
  return s;
}

lra_status lra_cur_residual(lra_handle h, const lra_operand *W, const double *A, const double *B, int64_t r,
                            int32_t prec, int64_t nsamples, const int64_t *si, const int64_t *sj, double *num2,
                            double *den2, void *stream) {
  lra_status s;
  if ((s = check_device(h)) != LRA_OK) return s;
  if ((s = check_operand(W)) != LRA_OK) return s;
  if (prec != LRA_RECON_PRECISE && prec != LRA_RECON_FAST) return fail(LRA_EINVAL, "bad lra_recon");
  if (!A || !B || !num2 || !den2 || r < 1) return fail(LRA_EINVAL, "null A/B/num2/den2 or r < 1");
  cudaStream_t st = (cudaStream_t)stream;
  if (nsamples > 0) {
    if (W->m_global > 0) return fail(LRA_EUNSUPPORTED, "the sampled estimate is not row-sharded");
    if (!si || !sj) return fail(LRA_EINVAL, "sampled residual needs si, sj");
    const int nblk = 296;
    if ((s = ws_reserve(h, (size_t)2 * nblk * sizeof(double2) + 256)) != LRA_OK) return s;
    int nl = 0;
    CK(launch_sampled(make_view(W), A, B, (int)r, si, sj, nsamples, (double2 *)h->ws, nblk, num2, den2, st, &nl, &h->prof));
    h->launches += nl;
    return LRA_OK;
  }
  if (W->kind != LRA_OP_DENSE) return fail(LRA_EINVAL, "the full pass needs a dense operand (use nsamples > 0)");
  const int S = resid_slices(W->dtype, prec);
  if ((s = ws_reserve(h, resid_scratch(W->m, W->n, r, S, 1))) != LRA_OK) return s;
  ResArgs a{};
  a.dtype = W->dtype;
  a.m = W->m;
  a.n = W->n;
  a.ldw = W->ldw;
  a.w = W->w;
  a.A = A;
  a.B = B;
  a.r = (int)r;
  a.partial = (double2 *)h->ws;
  a.status = nullptr;
  int nl = 0;
  cudaError_t e = cudaErrorInvalidConfiguration;
  if (S) {
    char *tcs = (char *)h->ws + (((size_t)resid_partials(W->m, W->n) * sizeof(double2) + 255) & ~(size_t)255);
    e = launch_residual_tc(a, 1, S, tcs, num2, den2, st, &nl, &h->prof);
  }
  if (e == cudaErrorInvalidConfiguration) {   // no tensor-core configuration for this r: fp64 SIMT pass
    cudaGetLastError();
    e = launch_residual(a, 1, num2, den2, st, &nl, &h->prof);
  }
  CK(e);
  if (W->m_global > 0) {   // row-sharded: sum the partial norms over the ranks
    if ((s = allreduce_sum(h, num2, 1, st)) != LRA_OK) return s;
    if ((s = allreduce_sum(h, den2, 1, st)) != LRA_OK) return s;
  }
  h->launches += nl;
  return LRA_OK;
}

lra_status lra_error_sample(lra_handle h, const lra_operand *W, const double *A, const double *B, int64_t r,
                            const int64_t *rows, int64_t q, const int64_t *cols, int64_t s, double *stats3,
                            void *stream) {
  lra_status st;
  if ((st = check_device(h)) != LRA_OK) return st;
  if ((st = check_operand(W)) != LRA_OK) return st;
  if (W->m_global > 0) return fail(LRA_EUNSUPPORTED, "the sampled estimate is not row-sharded");
  if (!A || !B || !rows || !cols || !stats3 || r < 1 || q < 1 || s < 1) return fail(LRA_EINVAL, "bad arguments");
  if ((st = ws_reserve(h, (size_t)2 * q * s * sizeof(double) + 256)) != LRA_OK) return st;
  int nl = 0;
  CK(launch_error_sample(make_view(W), A, B, (int)r, rows, q, cols, s, (double *)h->ws, stats3,
                         (cudaStream_t)stream, &nl, &h->prof));
  h->launches += nl;
  return LRA_OK;
}

lra_status lra_cur_progressive(lra_handle h, const lra_operand *W, const lra_multiplier *Ms, int32_t nmult, int64_t r,
                               int64_t k, int32_t sweeps, double tol, const int64_t *rows, int64_t q,
                               const int64_t *cols, int64_t s, void *Y, int64_t *I, int64_t *J, double *U, double *A,
                               double *B, lra_ca_stats *stats, double *stats4, int32_t *depth, double *estimate,
                               void *stream) {
  lra_status st;
  if ((st = check_device(h)) != LRA_OK) return st;
  if ((st = check_operand(W)) != LRA_OK) return st;
  if (!Ms || nmult < 1 || !Y || !stats4 || !depth || !estimate) return fail(LRA_EINVAL, "bad arguments");
  if (!(tol >= 0.0)) return fail(LRA_EINVAL, "tol >= 0");
  cudaStream_t sm = (cudaStream_t)stream;
  for (int32_t d = 1;; ++d) {
    const lra_multiplier *M = &Ms[d - 1];
    if (M->kind == LRA_MUL_ARFT) return fail(LRA_EUNSUPPORTED, "progressive depth runs real multipliers");
    if ((st = lra_preprocess(h, W, M, Y, W->m, stream)) != LRA_OK) return st;
    if ((st = lra_cross_approx(h, W, Y, W->m, 0, nullptr, r, k, k, sweeps, 1e-12, 1e-12, (int32_t)(20 * k), I, J, U,
                               A, B, stats, stream)) != LRA_OK)
      return st;
    if ((st = lra_error_sample(h, W, A, B, r, rows, q, cols, s, stats4, stream)) != LRA_OK) return st;
    double v[4];
    CK(cudaMemcpyAsync(v, stats4, sizeof(v), cudaMemcpyDeviceToHost, sm));
    CK(cudaStreamSynchronize(sm));
    // the superfast estimate of rho (Section spstr): sqrt(sum g^2 / sum W^2) over the sample
    const double est = v[3] > 0.0 ? sqrt(v[2] / v[3]) : INFINITY;
    if (est <= tol || d >= nmult) {
      *depth = d;
      *estimate = est;
      return LRA_OK;
    }
  }
}

lra_status lra_cur_certificate(lra_handle h, const lra_operand *W, const int64_t *I, const int64_t *J, const double *U,
                               int64_t k, int64_t l, int64_t r, double delta, double *out4, void *stream) {
  lra_status st;
  if ((st = check_device(h)) != LRA_OK) return st;
  if ((st = check_operand(W)) != LRA_OK) return st;
  if (W->m_global > 0) return fail(LRA_EUNSUPPORTED, "the certificate is not row-sharded");
  if (!I || !J || !U || !out4 || k < 1 || l < 1 || r < 1 || r > (k < l ? k : l) || !(delta >= 0.0))
    return fail(LRA_EINVAL, "bad arguments");
  if ((st = ws_reserve(h, 3 * sizeof(double) + 256)) != LRA_OK) return st;
  cudaStream_t sm = (cudaStream_t)stream;
  CK(launch_cert_norms(make_view(W), I, J, (int)k, (int)l, U, (double *)h->ws, sm));
  double nn[3];
  CK(cudaMemcpyAsync(nn, h->ws, sizeof(nn), cudaMemcpyDeviceToHost, sm));
  CK(cudaStreamSynchronize(sm));
  h->launches += 1;
  const double nc = sqrt(nn[0]), nr = sqrt(nn[1]), nu = sqrt(nn[2]);
  const double eta = (r == (k < l ? k : l)) ? 1.0 : 2.0;
  const double theta = nu * eta * delta;       // ||U|| bounded by ||U||_F (reading C27)
  double bound = INFINITY;
  if (theta < 1.0) {
    const double xi = sqrt((double)k * (double)l) / (1.0 - theta);
    bound = delta * ((nr + nc + delta + eta * nc * nr * nu) * xi * nu + 1.0);
  }
  out4[0] = bound;
  out4[1] = nc;
  out4[2] = nr;
  out4[3] = nu;
  return LRA_OK;
}

lra_status lra_expand_columns(lra_handle h, const lra_operand *W, const int64_t *I, int64_t k, int64_t *J, int64_t g0,
                              int64_t l, double tie_slack, void *stream) {
  lra_status st;
  if ((st = check_device(h)) != LRA_OK) return st;
  if ((st = check_operand(W)) != LRA_OK) return st;
  if (W->m_global > 0) return fail(LRA_EUNSUPPORTED, "column expansion is not row-sharded");
  if (!I || !J || k < 1 || k > 128 || g0 < k || l < g0 || l > W->n || !(tie_slack >= 0.0 && tie_slack < 1.0))
    return fail(LRA_EINVAL, "need 1 <= k <= 128, k <= g0 <= l <= n");
  if ((st = ws_reserve(h, ((size_t)k * W->n + (size_t)k * k + W->n) * 8 + 512)) != LRA_OK) return st;
  int *ok = (int *)((char *)h->ws + (((size_t)k * W->n + (size_t)k * k + W->n) * 8 + 255) / 256 * 256);
  int nl = 0;
  CK(launch_expand_columns(make_view(W), I, (int)k, J, (int)g0, (int)l, tie_slack, h->ws, ok, (cudaStream_t)stream, &nl,
                           &h->prof));
  h->launches += nl;
  return LRA_OK;
}

lra_status lra_contract_columns(lra_handle h, const lra_operand *W, const int64_t *I, int64_t k, int64_t *J,
                                int64_t g0, int64_t l, double tie_slack, void *stream) {
  lra_status st;
  if ((st = check_device(h)) != LRA_OK) return st;
  if ((st = check_operand(W)) != LRA_OK) return st;
  if (W->m_global > 0) return fail(LRA_EUNSUPPORTED, "column contraction is not row-sharded");
  if (!I || !J || k < 1 || k > 128 || l < k || g0 < l || g0 > W->n || !(tie_slack >= 0.0 && tie_slack < 1.0))
    return fail(LRA_EINVAL, "need 1 <= k <= l <= g0 <= n, k <= 128");
  const size_t base = ((size_t)k * W->n + (size_t)k * k + W->n) * 8;
  if ((st = ws_reserve(h, base + 512)) != LRA_OK) return st;
  int *ok = (int *)((char *)h->ws + (base + 255) / 256 * 256);
  int nl = 0;
  CK(launch_contract_columns(make_view(W), I, (int)k, J, (int)g0, (int)l, tie_slack, h->ws, ok, (cudaStream_t)stream,
                             &nl, &h->prof));
  h->launches += nl;
  return LRA_OK;
}

lra_status lra_refine_columns(lra_handle h, const lra_operand *W, const int64_t *I, int64_t k, int64_t *J, int64_t l,
                              int32_t cycles, double tie_slack, int32_t *changed, void *stream) {
  lra_status st;
  if ((st = check_device(h)) != LRA_OK) return st;
  if ((st = check_operand(W)) != LRA_OK) return st;
  if (W->m_global > 0) return fail(LRA_EUNSUPPORTED, "column refinement is not row-sharded");
  if (!I || !J || !changed || k < 1 || k > 128 || l < k || l + 1 > W->n || cycles < 0 ||
      !(tie_slack >= 0.0 && tie_slack < 1.0))
    return fail(LRA_EINVAL, "need 1 <= k <= l < n, k <= 128, cycles >= 0");
  const size_t base = ((size_t)k * W->n + (size_t)k * k + W->n) * 8;
  const size_t off_i = (base + 255) / 256 * 256;
  if ((st = ws_reserve(h, off_i + 256 + (size_t)(l + 1) * 8 + 256)) != LRA_OK) return st;
  int *ok = (int *)((char *)h->ws + off_i);
  int *stop = ok + 1;
  int64_t *Jw = (int64_t *)((char *)h->ws + off_i + 256);
  cudaStream_t sm = (cudaStream_t)stream;
  CK(cudaMemsetAsync(stop, 0, sizeof(int), sm));
  CK(cudaMemsetAsync(changed, 0, sizeof(int32_t), sm));
  CK(cudaMemcpyAsync(Jw, J, (size_t)l * 8, cudaMemcpyDeviceToDevice, sm));
  int nl = 0;
  CK(launch_refine_columns(make_view(W), I, (int)k, Jw, (int)l, cycles, tie_slack, h->ws, ok, stop, changed, sm, &nl,
                           &h->prof));
  CK(cudaMemcpyAsync(J, Jw, (size_t)l * 8, cudaMemcpyDeviceToDevice, sm));
  h->launches += nl;
  return LRA_OK;
}

lra_status lra_nucleus_factors(lra_handle h, const lra_operand *W, const int64_t *I, const int64_t *J, int64_t k,
                               int64_t l, int64_t r, double *U, double *A, double *B, int32_t *status, void *stream) {
  lra_status st;
  if ((st = check_device(h)) != LRA_OK) return st;
  if ((st = check_operand(W)) != LRA_OK) return st;
  if (W->m_global > 0) return fail(LRA_EUNSUPPORTED, "use lra_cross_approx for row-sharded operands");
  if (!I || !J || !A || !B || !status || k < 1 || l < 1 || k > 128 || l > 128 || r < 1 || r > (k < l ? k : l))
    return fail(LRA_EINVAL, "need 0 < r <= min(k, l), k, l <= 128");
  if (!nucleus_fits((int)k, (int)l)) return fail(LRA_EUNSUPPORTED, "a %lld x %lld generator exceeds the nucleus's shared memory", (long long)k, (long long)l);
  if ((st = ws_reserve(h, (size_t)(k + l) * r * 8 + 512)) != LRA_OK) return st;
  double *TS = (double *)h->ws;
  double *Sr = TS + (size_t)l * r;
  cudaStream_t sm = (cudaStream_t)stream;
  CK(cudaMemsetAsync(status, 0, sizeof(int32_t), sm));
  NucArgs na{};
  na.op = make_view(W);
  na.I = I;
  na.J = J;
  na.k = (int)k;
  na.l = (int)l;
  na.r = (int)r;
  na.U = U;
  na.TS = TS;
  na.Sr = Sr;
  na.status = status;
  FacArgs fa{};
  fa.op = na.op;
  fa.I = I;
  fa.J = J;
  fa.k = (int)k;
  fa.l = (int)l;
  fa.r = (int)r;
  fa.TS = TS;
  fa.Sr = Sr;
  fa.A = A;
  fa.B = B;
  fa.status = status;
  int nl = 0;
  CK(launch_nucleus(na, fa, 1, sm, &nl, &h->prof));
  h->launches += nl;
  return LRA_OK;
}

// inverse of the standard normal CDF (Acklam's rational approximation, |rel err| < 1.2e-9)
static double norm_ppf(double p) {
  static const double a[] = {-3.969683028665376e+01, 2.209460984245205e+02, -2.759285104469687e+02,
                             1.383577518672690e+02, -3.066479806614716e+01, 2.506628277459239e+00};
  static const double b[] = {-5.447609879822406e+01, 1.615858368580409e+02, -1.556989798598866e+02,
                             6.680131188771972e+01, -1.328068155288572e+01};
  static const double c[] = {-7.784894002430293e-03, -3.223964580411365e-01, -2.400758277161838e+00,
                             -2.549732539343734e+00, 4.374664141464968e+00, 2.938163982698783e+00};
  static const double d[] = {7.784695709041462e-03, 3.224671290700398e-01, 2.445134137142996e+00,
                             3.754408661907416e+00};
  const double pl = 0.02425;
  if (p < pl) {
    const double q = sqrt(-2 * log(p));
    return (((((c[0] * q + c[1]) * q + c[2]) * q + c[3]) * q + c[4]) * q + c[5]) /
           ((((d[0] * q + d[1]) * q + d[2]) * q + d[3]) * q + 1);
  }
  if (p > 1 - pl) {
    const double q = sqrt(-2 * log(1 - p));
    return -(((((c[0] * q + c[1]) * q + c[2]) * q + c[3]) * q + c[4]) * q + c[5]) /
           ((((d[0] * q + d[1]) * q + d[2]) * q + d[3]) * q + 1);
  }
  const double q = p - 0.5, rr = q * q;
  return (((((a[0] * rr + a[1]) * rr + a[2]) * rr + a[3]) * rr + a[4]) * rr + a[5]) * q /
         (((((b[0] * rr + b[1]) * rr + b[2]) * rr + b[3]) * rr + b[4]) * rr + 1);
}

lra_status lra_variance_bound(double var_K, int64_t K, double alpha, double *bound) {
  if (!bound || K < 2 || !(alpha > 0.0 && alpha < 0.5) || !(var_K >= 0.0)) return fail(LRA_EINVAL, "bad arguments");
  // chi-square quantile chi2_{K-1}(alpha) by Wilson-Hilferty
  const double nu = (double)(K - 1), z = norm_ppf(alpha);
  const double t = 1.0 - 2.0 / (9.0 * nu) + z * sqrt(2.0 / (9.0 * nu));
  const double q = nu * t * t * t;
  *bound = (double)K * var_K / q;
  return LRA_OK;
}

static size_t batch_scratch(int64_t m, int64_t n, int64_t r, int64_t k, int64_t nb, size_t esz, int S) {
  Carve probe{nullptr, 0};
  probe.take<int32_t>(nb);
  probe.take<char>((size_t)nb * m * k * esz);
  probe.take<double>((size_t)nb * k * r);
  probe.take<double>((size_t)nb * k * r);
  probe.take<double>((size_t)nb * m * r);
  probe.take<double>((size_t)nb * r * n);
  probe.take<double2>((size_t)nb * resid_partials(m, n));
  probe.take<int32_t>((size_t)nb * 4);
  probe.take<char>(S ? residual_tc_scratch(m, n, (int)r, S, nb) : 0);
  return probe.off + 256;
}

lra_status lra_batch(lra_handle h, int64_t nb, const lra_operand *W0, int64_t w_stride, const lra_multiplier *M0,
                     int64_t m_stride, int64_t r, int64_t k, int64_t l, int32_t sweeps, double swap_tol,
                     double tie_slack, int32_t swap_cap, int32_t prec, int64_t *I, int64_t *J, double *U,
                     double *num2, double *den2, lra_ca_stats *stats, void *stream) {
  lra_status s;
  if ((s = check_device(h)) != LRA_OK) return s;
  if ((s = check_operand(W0)) != LRA_OK) return s;
  if (W0->kind != LRA_OP_DENSE) return fail(LRA_EINVAL, "lra_batch needs dense blocks");
  if (W0->m_global > 0) return fail(LRA_EINVAL, "lra_batch blocks are not row-sharded (deal blocks to ranks)");
  if (nb < 1) return fail(LRA_EINVAL, "nb >= 1");
  if (w_stride < W0->ldw * W0->n) return fail(LRA_EINVAL, "w_stride < ldw*n (blocks overlap)");
  if ((s = check_ca_shape(W0, r, k, l, sweeps)) != LRA_OK) return s;
  if ((s = check_mult(M0, W0->n)) != LRA_OK) return s;
  if (M0->lbar != k) return fail(LRA_EINVAL, "v1 requires lbar == k (reading C9)");
  if (m_stride != 0 && M0->kind != LRA_MUL_SPARSE_PM1)
    return fail(LRA_EINVAL, "per-block multipliers (m_stride != 0) are supported for SPARSE_PM1 only");
  if (prec != LRA_RECON_PRECISE && prec != LRA_RECON_FAST) return fail(LRA_EINVAL, "bad lra_recon");
  if (!I || !J || !num2 || !den2) return fail(LRA_EINVAL, "null output");
  const int64_t m = W0->m, n = W0->n;
  const bool cplx = M0->kind == LRA_MUL_ARFT;
  const size_t esz = cplx ? 16 : 8;
  const int64_t tiles = resid_partials(m, n);
  const int S = resid_slices(W0->dtype, prec);
  if ((s = ws_reserve(h, batch_scratch(m, n, r, k, nb, esz, S))) != LRA_OK) return s;
  Carve cv{(char *)h->ws, 0};
  int32_t *status = cv.take<int32_t>(nb);
  void *Y = cv.take<char>((size_t)nb * m * k * esz);
  double *TS = cv.take<double>((size_t)nb * k * r);
  double *Sr = cv.take<double>((size_t)nb * k * r);
  double *A = cv.take<double>((size_t)nb * m * r);
  double *B = cv.take<double>((size_t)nb * r * n);
  double2 *part = cv.take<double2>((size_t)nb * tiles);
  int32_t *yinfo = cv.take<int32_t>((size_t)nb * 4);
  char *tcs = S ? cv.take<char>(residual_tc_scratch(m, n, (int)r, S, nb)) : nullptr;
  cudaStream_t st = (cudaStream_t)stream;
  CK(cudaMemsetAsync(status, 0, sizeof(int32_t) * nb, st));
  // Blocks are processed in groups on the handle's side streams (fork/join on `stream` with
  // events, so the call stays stream-ordered and graph-capturable): the latency-bound C-A
  // and nucleus of one group overlap the bandwidth-bound sketch/residual of another.
  if ((s = ensure_streams(h)) != LRA_OK) return s;
  // Group size: as many problems as the cluster tier runs concurrently (one wave of co-resident
  // clusters; 7 for config 2 on a B200), so that one group's C-A fills the GPCs while the
  // previous group's nucleus / residual use the remaining SMs.  LRA_BATCH_GROUPS overrides.
  // The grid and global-memory tiers use the handle's single exchange / C-matrix buffers and
  // occupy every SM (cooperative grids), so their groups run in order on ONE side stream.
  const int64_t maxN = m > n ? m : n;
  if (cplx && ca_needs_global(maxN, (int)k))
    return fail(LRA_EUNSUPPORTED, "ARFT sketch with a block beyond the on-chip tiers");
  const int act = (ca_needs_global(maxN, (int)k) || (h->diag > 0 && !cplx))
                      ? 0
                      : (ca_small_fits(maxN, (int)k, cplx ? 1 : 0, 0) ? ca_small_max_active(maxN, (int)k)
                                                                       : ca_cluster_max_active(maxN, (int)k));
  // While profiling (lra_profile_enable), the groups also run in order on one stream: every
  // kernel's event interval is then its own device time, not time spent queued behind
  // another group's kernels (the isolation pass of bench.py).
  const int nside = (act >= 1 && !h->prof.on) ? LRA_NSIDE : 1;
  int64_t ngroups;
  if (h->groups_env > 0) {
    ngroups = nb < h->groups_env ? nb : h->groups_env;
  } else {
    const int64_t per = act >= 2 ? act : 4;
    ngroups = (nb + per - 1) / per;
    if (ngroups < 1) ngroups = 1;
  }
  const int64_t gsz = (nb + ngroups - 1) / ngroups;
  ngroups = (nb + gsz - 1) / gsz;
  lra_multiplier Mres;
  if ((s = resolve_mult(h, M0, n, st, &Mres)) != LRA_OK) return s;
  M0 = &Mres;
  // A Gaussian sketch runs once for the whole batch on the tensor cores (one stream-K launch
  // over every problem's tiles, before the fork); the other kinds are sketched per group.
  size_t skper = 0;
  if ((s = sketch_scratch(h, M0, m, n, nb, 1, &skper)) != LRA_OK) return s;
  if (skper) {
    SketchArgs sa = make_sketch(W0, M0, Y, m);
    sa.w_stride = w_stride;
    sa.y_stride = m * k;
    CK(launch_sketch(sa, nb, M0->omega, M0->ld_omega, st, &h->prof, h->sk, skper));
    h->launches += 2;
  }
  CK(cudaEventRecord(h->fork, st));
  for (int i = 0; i < nside; ++i) CK(cudaStreamWaitEvent(h->side[i], h->fork, 0));
  // Every exit after the fork joins the side streams back into `stream` (so a captured graph
  // stays joined and later work on `stream` is ordered after everything enqueued here).
  struct Join {
    lra_handle h;
    cudaStream_t st;
    int n;
    ~Join() {
      for (int i = 0; i < n; ++i) {
        cudaEventRecord(h->join[i], h->side[i]);
        cudaStreamWaitEvent(st, h->join[i], 0);
      }
    }
  } join{h, st, nside};
  const size_t wsz = W0->dtype == LRA_F32 ? 4 : 8;
  for (int64_t g = 0; g < ngroups; ++g) {
    const int64_t b0 = g * gsz, gn = (nb - b0) < gsz ? (nb - b0) : gsz;
    cudaStream_t gs = h->side[g % nside];
    lra_operand Wg = *W0;
    Wg.w = (const char *)W0->w + b0 * w_stride * wsz;
    lra_multiplier Mg = *M0;
    if (m_stride) {
      Mg.sp_row = M0->sp_row + b0 * m_stride;
      Mg.sp_sign = M0->sp_sign + b0 * m_stride;
    }
    char *Yg = (char *)Y + (size_t)b0 * m * k * esz;
    SketchArgs sa = make_sketch(&Wg, &Mg, Yg, m);
    sa.w_stride = w_stride;
    sa.m_stride = m_stride;
    sa.y_stride = m * k;
    if (!skper) {
      CK(launch_sketch(sa, gn, Mg.omega, Mg.ld_omega, gs, &h->prof));
      h->launches += 1;
    }
    s = run_chain(h, &Wg, w_stride, Yg, m, m * k, cplx ? 1 : 0, nullptr, r, k, sweeps, swap_tol, tie_slack, swap_cap,
                  I + b0 * k, J + b0 * k, U ? U + b0 * k * k : nullptr, A + b0 * m * r, B + b0 * r * n, m * r, r * n,
                  stats ? stats + b0 : nullptr, status + b0, TS + b0 * k * r, Sr + b0 * k * r, yinfo + 4 * b0, gn, gs);
    if (s != LRA_OK) return s;
    ResArgs ra{};
    ra.dtype = W0->dtype;
    ra.m = m;
    ra.n = n;
    ra.ldw = W0->ldw;
    ra.w_stride = w_stride;
    ra.w = Wg.w;
    ra.A = A + b0 * m * r;
    ra.B = B + b0 * r * n;
    ra.a_stride = m * r;
    ra.b_stride = r * n;
    ra.r = (int)r;
    ra.partial = part + b0 * tiles;
    ra.status = status + b0;
    int nl = 0;
    cudaError_t e = cudaErrorInvalidConfiguration;
    if (S) {   // each group uses its own slice of the tensor-core scratch
      char *g_tcs = tcs + (residual_tc_scratch(m, n, (int)r, S, nb) - 1024) / nb * b0;
      g_tcs = (char *)(((uintptr_t)g_tcs + 255) & ~(uintptr_t)255);
      e = launch_residual_tc(ra, gn, S, g_tcs, num2 + b0, den2 + b0, gs, &nl, &h->prof);
    }
    if (e == cudaErrorInvalidConfiguration) {   // fp64 SIMT pass (fp64 W PRECISE, or r beyond the TC tiles)
      cudaGetLastError();
      e = launch_residual(ra, gn, num2 + b0, den2 + b0, gs, &nl, &h->prof);
    }
    CK(e);
    h->launches += nl;
  }
  return LRA_OK;
}

lra_status lra_leverage_scores(lra_handle h, const lra_operand *W, const int64_t *idx, int64_t k, int32_t side,
                               int64_t r, double *p, int32_t *status, void *stream) {
  lra_status st;
  if ((st = check_device(h)) != LRA_OK) return st;
  if ((st = check_operand(W)) != LRA_OK) return st;
  if (W->m_global > 0) return fail(LRA_EUNSUPPORTED, "leverage scores are not row-sharded");
  if (!idx || !p || !status || (side != 0 && side != 1) || k < 1 || k > 112 || r < 1 || r > k ||
      (size_t)2 * k * r * 8 > 200 * 1024)
    return fail(LRA_EINVAL, "need side 0/1, 1 <= r <= k <= 112");
  const int64_t N = side ? W->m : W->n;
  if ((st = ws_reserve(h, leverage_scratch_bytes((int)k, (int)r, N))) != LRA_OK) return st;
  cudaStream_t sm = (cudaStream_t)stream;
  CK(cudaMemsetAsync(status, 0, sizeof(int32_t), sm));
  int nl = 0;
  CK(launch_leverage_scores(make_view(W), idx, (int)k, side, (int)r, p, status, h->ws, sm, &nl, &h->prof));
  h->launches += nl;
  return LRA_OK;
}

lra_status lra_sample_exactly(lra_handle h, const double *p, int64_t N, int64_t l, const double *u, int64_t *idx,
                              double *dscale, const int32_t *status, void *stream) {
  lra_status st;
  if ((st = check_device(h)) != LRA_OK) return st;
  if (!u || !idx || N < 1 || l < 1 || l > INT32_MAX) return fail(LRA_EINVAL, "need u, idx, N >= 1, 1 <= l < 2^31");
  if ((st = ws_reserve(h, (size_t)N * 8 + 256)) != LRA_OK) return st;
  int nl = 0;
  CK(launch_sample_exactly(p, N, (int)l, u, (double *)h->ws, idx, dscale, status, (cudaStream_t)stream, &nl,
                           &h->prof));
  h->launches += nl;
  return LRA_OK;
}

lra_status lra_sample_expected(lra_handle h, const double *p, int64_t N, int64_t l, const double *u, int64_t cap,
                               int64_t *idx, double *dscale, int64_t *count, const int32_t *status, void *stream) {
  lra_status st;
  if ((st = check_device(h)) != LRA_OK) return st;
  if (!u || !count || N < 1 || l < 1 || l > INT32_MAX || cap < 0 || (cap > 0 && !idx))
    return fail(LRA_EINVAL, "need u, count, N >= 1, 1 <= l < 2^31, cap >= 0 (idx when cap > 0)");
  int nl = 0;
  CK(launch_sample_expected(p, N, (int)l, u, cap, idx, dscale, count, status, (cudaStream_t)stream, &nl, &h->prof));
  h->launches += nl;
  return LRA_OK;
}

lra_status lra_maxvol(lra_handle h, const double *B, int64_t N, int64_t q, const int64_t *start, double swap_tol,
                      double tie_slack, int32_t swap_cap, int64_t *slots, lra_ca_stats *stats, void *stream) {
  lra_status st;
  if ((st = check_device(h)) != LRA_OK) return st;
  if (!B || !slots || q < 1 || N < q || q > LRA_QMAX_ALL) return fail(LRA_EINVAL, "need 1 <= q <= min(N, %d)", LRA_QMAX_ALL);
  if (!(swap_tol >= 0.0) || !(tie_slack >= 0.0) || tie_slack >= 1.0 || swap_cap < 0)
    return fail(LRA_EINVAL, "bad swap_tol / tie_slack / swap_cap");
  Carve probe{nullptr, 0};
  probe.take<int32_t>(4);
  probe.take<int64_t>((size_t)q);
  probe.take<lra_ca_stats>(1);
  if ((st = ws_reserve(h, probe.off + 256)) != LRA_OK) return st;
  Carve cv{(char *)h->ws, 0};
  int32_t *status = cv.take<int32_t>(4);
  int64_t *dJ = cv.take<int64_t>((size_t)q);
  lra_ca_stats *own = cv.take<lra_ca_stats>(1);
  cudaStream_t sm = (cudaStream_t)stream;
  CK(cudaMemsetAsync(status, 0, sizeof(int32_t), sm));
  return maxvol_block(h, B, N, (int)q, start, slots, swap_tol, tie_slack, swap_cap, stats ? stats : own, status, dJ, sm);
}

lra_status lra_qrp_columns(lra_handle h, const lra_operand *W, const int64_t *I, int64_t k, int64_t q,
                           double tie_slack, int64_t *piv, double *R, int64_t ldr, double *Rt, int32_t *status,
                           void *stream) {
  lra_status st;
  if ((st = check_device(h)) != LRA_OK) return st;
  if ((st = check_operand(W)) != LRA_OK) return st;
  if (W->m_global > 0) return fail(LRA_EUNSUPPORTED, "the QRP is not row-sharded");
  if (!I || !piv || !status || k < 1 || k > 128 || q < 1 || q > k || q > W->n || !(tie_slack >= 0.0 && tie_slack < 1.0))
    return fail(LRA_EINVAL, "need 1 <= q <= min(k, n), k <= 128");
  if (R && ldr < q) return fail(LRA_EINVAL, "ldr < q");
  if ((st = ws_reserve(h, qrp_scratch_bytes((int)k, W->n))) != LRA_OK) return st;
  cudaStream_t sm = (cudaStream_t)stream;
  CK(cudaMemsetAsync(status, 0, sizeof(int32_t), sm));
  int nl = 0;
  CK(launch_qrp(make_view(W), I, (int)k, (int)q, tie_slack, piv, R, ldr, Rt, status, h->ws, sm, &nl, &h->prof));
  h->launches += nl;
  return LRA_OK;
}

// Scratch for the calls of one workload shape (reading of SURVEY 8(b) "lra_workspace_query"):
// nb == 0 sizes lra_preprocess / lra_cross_approx / lra_cur_residual (either lra_recon) on W;
// nb >= 1 sizes lra_batch over nb blocks shaped like W.  All four handle-owned buffers count.
static lra_status workspace_sizes(lra_handle h, const lra_operand *W, int64_t r, int64_t k, int32_t sweeps,
                                  int64_t nb, size_t sz[4]) {
  lra_status s;
  if ((s = check_operand(W)) != LRA_OK) return s;
  if ((s = check_ca_shape(W, r, k, k, sweeps)) != LRA_OK) return s;
  if (nb < 0) return fail(LRA_EINVAL, "nb >= 0");
  const int64_t m = W->m, n = W->n, mg = W->m_global > 0 ? W->m_global : m;
  const int64_t maxN = mg > n ? mg : n;
  size_t ws = 0, gm = 0, sh = 0;
  const int Smax = W->dtype == LRA_F32 ? 6 : 3;
  if (nb == 0) {
    ws = chain_scratch(r, k);
    if (W->kind == LRA_OP_DENSE) {
      const size_t rs = resid_scratch(m, n, r, Smax, 1), r0 = resid_scratch(m, n, r, 0, 1);
      ws = ws > rs ? ws : rs;
      ws = ws > r0 ? ws : r0;
    }
    const size_t smp = (size_t)2 * 296 * sizeof(double2) + 256;
    ws = ws > smp ? ws : smp;
    if (W->m_global > 0) sh = sharded_scratch(mg, n, r, k, sweeps, h ? h->nranks : 1);
    if (ca_needs_global(maxN, (int)k) || W->m_global > 0) gm = ca_global_scratch_bytes(maxN, (int)k);
  } else {
    if (W->kind != LRA_OP_DENSE || W->m_global > 0) return fail(LRA_EINVAL, "lra_batch takes unsharded dense blocks");
    const size_t a = batch_scratch(m, n, r, k, nb, 16, Smax), b = batch_scratch(m, n, r, k, nb, 16, 0);
    ws = a > b ? a : b;
    if (ca_needs_global(maxN, (int)k)) gm = ca_global_scratch_bytes(maxN, (int)k);
  }
  sz[0] = ws + ws / 4;   // ws_reserve over-allocates by a quarter
  sz[1] = ca_grid_scratch_bytes(160);
  sz[2] = gm;
  sz[3] = sh;
  return LRA_OK;
}

lra_status lra_workspace_query(lra_handle h, const lra_operand *W, int64_t r, int64_t k, int32_t sweeps, int64_t nb,
                               size_t *bytes) {
  if (!h || !bytes) return fail(LRA_EINVAL, "null handle or bytes");
  size_t sz[4];
  lra_status s;
  if ((s = workspace_sizes(h, W, r, k, sweeps, nb, sz)) != LRA_OK) return s;
  *bytes = sz[0] + sz[1] + sz[2] + sz[3];
  return LRA_OK;
}

lra_status lra_workspace_reserve(lra_handle h, const lra_operand *W, int64_t r, int64_t k, int32_t sweeps, int64_t nb) {
  lra_status s;
  if ((s = check_device(h)) != LRA_OK) return s;
  size_t sz[4];
  if ((s = workspace_sizes(h, W, r, k, sweeps, nb, sz)) != LRA_OK) return s;
  if ((s = ws_reserve(h, sz[0] * 4 / 5)) != LRA_OK) return s;
  if ((s = buf_reserve(&h->gs, &h->gs_bytes, sz[1], "the grid-tier exchange")) != LRA_OK) return s;
  if (sz[2] && (s = buf_reserve(&h->gm, &h->gm_bytes, sz[2], "the global-memory C-A tier")) != LRA_OK) return s;
  if (sz[3] && (s = buf_reserve(&h->sh, &h->sh_bytes, sz[3], "the sharded blocks")) != LRA_OK) return s;
  return LRA_OK;
}

}  // extern "C"
