"""Thin ctypes binding of liblra.so (include/lra.h): same names, argument marshalling only.

Every step of the hot path runs in the library's CUDA kernels; PyTorch only supplies device
memory (tensors), the stream handle and, for multi-GPU runs, the process group.  There is
no CPU fallback: if liblra.so is missing or no CUDA device is present, calls raise.

Conventions: a dense m×n matrix W is a torch tensor ``Wt`` of shape (n, m), C-contiguous —
i.e. W column-major with ldw = m (``to_colmajor`` converts a numpy (m, n) array).  Batches
are (nb, n, m).  Index sets are int64 tensors, U is (k, l) storage of the l×k column-major
nucleus, A is (r, m) storage of the m×r column-major factor, B is (n, r) storage of the
r×n column-major factor.
"""
from __future__ import annotations

import ctypes as C
import os

import numpy as np

_HERE = os.path.dirname(os.path.abspath(__file__))
_SO = os.environ.get("LRA_SO") or os.path.join(_HERE, "liblra.so")   # LRA_SO: diagnostics (A/B builds)

LRA_OK, LRA_EINVAL, LRA_ESINGULAR, LRA_ENOMEM, LRA_ECUDA, LRA_ENCCL, LRA_EUNSUPPORTED = 0, -1, -2, -3, -4, -5, -6
LRA_F32, LRA_F64 = 0, 1
LRA_OP_DENSE, LRA_OP_FACTORED_CSR = 0, 1
LRA_MUL_NONE, LRA_MUL_GAUSSIAN, LRA_MUL_ARHT, LRA_MUL_ARFT, LRA_MUL_SPARSE_PM1, LRA_MUL_QGAUSS = 0, 1, 2, 3, 4, 5
LRA_RECON_FAST, LRA_RECON_PRECISE = 0, 1
MUL_KIND = {"none": LRA_MUL_NONE, "gaussian": LRA_MUL_GAUSSIAN, "arht": LRA_MUL_ARHT,
            "arft": LRA_MUL_ARFT, "sparse": LRA_MUL_SPARSE_PM1, "qgauss": LRA_MUL_QGAUSS}


class lra_operand(C.Structure):
    _fields_ = [("kind", C.c_int32), ("dtype", C.c_int32), ("m", C.c_int64), ("n", C.c_int64),
                ("w", C.c_void_p), ("ldw", C.c_int64), ("fa", C.c_void_p), ("fb", C.c_void_p),
                ("p", C.c_int64), ("e_rowptr", C.c_void_p), ("e_col", C.c_void_p), ("e_val", C.c_void_p),
                ("row0", C.c_int64), ("m_global", C.c_int64)]


class lra_multiplier(C.Structure):
    _fields_ = [("kind", C.c_int32), ("depth", C.c_int32), ("lbar", C.c_int64), ("dsign", C.c_void_p),
                ("col", C.c_void_p), ("sp_row", C.c_void_p), ("sp_sign", C.c_void_p),
                ("nnz_per_col", C.c_int32), ("omega", C.c_void_p), ("ld_omega", C.c_int64),
                ("qg_sign", C.c_void_p), ("qg_perm", C.c_void_p)]


STATS_DTYPE = np.dtype([("status", np.int32), ("loops_done", np.int32), ("lu_steps", np.int32),
                        ("swaps", np.int32), ("cap_hits", np.int32), ("sketch_swaps", np.int32),
                        ("cert_rows", np.float64), ("cert_cols", np.float64),
                        ("logvol_final", np.float64), ("min_pivot_margin", np.float64)])
assert STATS_DTYPE.itemsize == 56


class LibraryMissing(RuntimeError):
    pass


class LraError(RuntimeError):
    def __init__(self, status, msg):
        super().__init__(f"lra status {status}: {msg}")
        self.status = status


def _load():
    if not os.path.exists(_SO):
        raise LibraryMissing(f"{_SO} not built — run __graft_entry__.build() (no CPU fallback exists)")
    lib = C.CDLL(_SO)
    vp, i64, i32, dbl = C.c_void_p, C.c_int64, C.c_int32, C.c_double
    P = C.POINTER
    lib.lra_handle_create.argtypes = [P(vp), C.c_int, vp, C.c_int, C.c_int]
    lib.lra_handle_destroy.argtypes = [vp]
    lib.lra_handle_destroy.restype = None
    lib.lra_preprocess.argtypes = [vp, P(lra_operand), P(lra_multiplier), vp, i64, vp]
    lib.lra_cross_approx.argtypes = [vp, P(lra_operand), vp, i64, C.c_int, vp, i64, i64, i64, i32, dbl, dbl, i32,
                                     vp, vp, vp, vp, vp, vp, vp]
    lib.lra_cur_residual.argtypes = [vp, P(lra_operand), vp, vp, i64, i32, i64, vp, vp, vp, vp, vp]
    lib.lra_batch.argtypes = [vp, i64, P(lra_operand), i64, P(lra_multiplier), i64, i64, i64, i64, i32, dbl, dbl,
                              i32, i32, vp, vp, vp, vp, vp, vp, vp]
    lib.lra_last_error.restype = C.c_char_p
    lib.lra_preprocess_full.argtypes = [vp, P(lra_operand), P(lra_multiplier), vp, i64, vp]
    lib.lra_preprocess_full.restype = C.c_int
    lib.lra_error_sample.argtypes = [vp, P(lra_operand), vp, vp, i64, vp, i64, vp, i64, vp, vp]
    lib.lra_error_sample.restype = C.c_int
    lib.lra_cur_progressive.argtypes = [vp, P(lra_operand), P(lra_multiplier), i32, i64, i64, i32, dbl, vp, i64, vp,
                                        i64, vp, vp, vp, vp, vp, vp, vp, vp, P(i32), P(dbl), vp]
    lib.lra_cur_progressive.restype = C.c_int
    lib.lra_expand_columns.argtypes = [vp, P(lra_operand), vp, i64, vp, i64, i64, dbl, vp]
    lib.lra_expand_columns.restype = C.c_int
    lib.lra_nucleus_factors.argtypes = [vp, P(lra_operand), vp, vp, i64, i64, i64, vp, vp, vp, vp, vp]
    lib.lra_nucleus_factors.restype = C.c_int
    lib.lra_cur_certificate.argtypes = [vp, P(lra_operand), vp, vp, vp, i64, i64, i64, dbl, P(C.c_double), vp]
    lib.lra_cur_certificate.restype = C.c_int
    lib.lra_variance_bound.argtypes = [dbl, i64, dbl, P(C.c_double)]
    lib.lra_variance_bound.restype = C.c_int
    if hasattr(lib, "lra_leverage_scores"):
        lib.lra_leverage_scores.argtypes = [vp, P(lra_operand), vp, i64, i32, i64, vp, vp, vp]
        lib.lra_leverage_scores.restype = C.c_int
        lib.lra_sample_exactly.argtypes = [vp, vp, i64, i64, vp, vp, vp, vp, vp]
        lib.lra_sample_exactly.restype = C.c_int
        lib.lra_sample_expected.argtypes = [vp, vp, i64, i64, vp, i64, vp, vp, vp, vp, vp]
        lib.lra_sample_expected.restype = C.c_int
    if hasattr(lib, "lra_refine_columns"):
        lib.lra_contract_columns.argtypes = [vp, P(lra_operand), vp, i64, vp, i64, i64, dbl, vp]
        lib.lra_contract_columns.restype = C.c_int
        lib.lra_refine_columns.argtypes = [vp, P(lra_operand), vp, i64, vp, i64, i32, dbl, vp, vp]
        lib.lra_refine_columns.restype = C.c_int
    if hasattr(lib, "lra_qrp_columns"):
        lib.lra_maxvol.argtypes = [vp, vp, i64, i64, vp, dbl, dbl, i32, vp, vp, vp]
        lib.lra_maxvol.restype = C.c_int
        lib.lra_qrp_columns.argtypes = [vp, P(lra_operand), vp, i64, i64, dbl, vp, vp, i64, vp, vp, vp]
        lib.lra_qrp_columns.restype = C.c_int
    if hasattr(lib, "lra_workspace_query"):   # absent from older builds loaded through LRA_SO
        lib.lra_workspace_query.argtypes = [vp, P(lra_operand), i64, i64, i32, i64, P(C.c_size_t)]
        lib.lra_workspace_query.restype = C.c_int
        lib.lra_workspace_reserve.argtypes = [vp, P(lra_operand), i64, i64, i32, i64]
        lib.lra_workspace_reserve.restype = C.c_int
    lib.lra_nccl_unique_id.argtypes = [vp]
    lib.lra_nccl_unique_id.restype = C.c_int
    lib.lra_launch_count.argtypes = [vp]
    lib.lra_launch_count.restype = i64
    lib.lra_profile_enable.argtypes = [vp, C.c_int]
    lib.lra_profile_enable.restype = C.c_int
    lib.lra_profile_read.argtypes = [vp, C.c_int, P(C.c_char_p), P(C.c_double), P(i64)]
    lib.lra_profile_read.restype = C.c_int
    lib.lra_debug_counters.argtypes = [P(C.c_uint64), C.c_int]
    lib.lra_debug_counters.restype = C.c_int
    lib.lra_debug_counters_residual.argtypes = [P(C.c_uint64), C.c_int]
    lib.lra_debug_counters_residual.restype = C.c_int
    lib.lra_set_diagnostics.argtypes = [vp, i32]
    lib.lra_set_diagnostics.restype = C.c_int
    lib.lra_debug_index_errors.argtypes = [P(i64), C.c_int]
    lib.lra_debug_index_errors.restype = C.c_int
    for f in ("lra_handle_create", "lra_preprocess", "lra_cross_approx", "lra_cur_residual", "lra_batch"):
        getattr(lib, f).restype = C.c_int
    return lib


_lib = None


def lib():
    global _lib
    if _lib is None:
        _lib = _load()
    return _lib


EXPORTED = ["lra_handle_create", "lra_handle_destroy", "lra_preprocess", "lra_cross_approx",
            "lra_cur_residual", "lra_batch", "lra_last_error", "lra_launch_count", "lra_profile_enable",
            "lra_profile_read", "lra_debug_counters", "lra_debug_counters_residual", "lra_debug_index_errors", "lra_set_diagnostics",
            "lra_nccl_unique_id",
            "lra_preprocess_full", "lra_error_sample", "lra_cur_progressive", "lra_variance_bound",
            "lra_cur_certificate", "lra_expand_columns", "lra_nucleus_factors", "lra_workspace_query",
            "lra_workspace_reserve", "lra_maxvol", "lra_qrp_columns", "lra_contract_columns",
            "lra_refine_columns", "lra_leverage_scores", "lra_sample_exactly", "lra_sample_expected"]


def debug_counters(reset=True):
    out = (C.c_uint64 * 16)()
    _check(lib().lra_debug_counters(out, int(reset)))
    names = ["load", "cold_lu", "warm_gather", "gauss_jordan", "product", "swap_loop", "kernel", "pivot_steps",
             "exact_rounds", "pk_reduce", "pk_cluster_bar", "pk_decide", "take_row", "sw_update", "nuc_sweeps", "nuc_rotations"]
    return dict(zip(names, [int(x) for x in out]))


def debug_counters_residual(reset=True):
    out = (C.c_uint64 * 16)()
    _check(lib().lra_debug_counters_residual(out, int(reset)))
    names = ["mma_wait_b", "mma_wait_tmem", "mma_issue", "prod_wait_b", "prod_wait_a", "mma_wait_a",
             "epi_wait_tmem", "epi_work", "tiles", "epi_wait_w", "prod_wait_w"]
    return dict(zip(names, [int(x) for x in out]))


def debug_index_errors(reset=True):
    """First out-of-range data-dependent index (LRA_CHECK_IDX builds): (kernel id, problem, value, bound)."""
    out = (C.c_int64 * 4)()
    _check(lib().lra_debug_index_errors(out, int(reset)))
    return tuple(int(x) for x in out)


def _check(st):
    if st != LRA_OK:
        raise LraError(st, lib().lra_last_error().decode())


def _ptr(t):
    return None if t is None else C.c_void_p(t.data_ptr())


def _stream(stream):
    import torch
    s = torch.cuda.current_stream() if stream is None else stream
    return C.c_void_p(s.cuda_stream)


# ------------------------------------------------------------------ marshalling helpers
def to_colmajor(W_np, device="cuda"):
    """numpy (m, n) → torch (n, m) contiguous on ``device`` (column-major W, same bits)."""
    import torch
    return torch.from_numpy(np.ascontiguousarray(np.asarray(W_np).T)).to(device)


class Dense:
    """A dense operand: Wt is (n, m) [or (nb, n, m) for batches], fp32 or fp64.  A row shard
    of an m_global x n matrix: rows [row0, row0 + m) with m_global > 0 (multi-GPU)."""

    def __init__(self, Wt, row0=0, m_global=0):
        import torch
        assert Wt.is_cuda and Wt.is_contiguous() and Wt.dtype in (torch.float32, torch.float64)
        self.Wt = Wt
        self.n, self.m = Wt.shape[-2], Wt.shape[-1]
        self.row0, self.m_global = int(row0), int(m_global)

    def struct(self):
        import torch
        return lra_operand(LRA_OP_DENSE, LRA_F32 if self.Wt.dtype == torch.float32 else LRA_F64,
                           self.m, self.n, self.Wt.data_ptr(), self.m, None, None, 0, None, None, None,
                           self.row0, self.m_global)

    def block_stride(self):
        return self.m * self.n


class Factored:
    """Entry oracle W = A·B + E (config 4): A (p, m) storage of m×p col-major fp64, B (n, p)
    storage of p×n col-major fp64, CSR row_ptr (m+1), col, val on device."""

    def __init__(self, A_t, B_t, row_ptr, col, val, m, n, p):
        self.A_t, self.B_t, self.row_ptr, self.col, self.val = A_t, B_t, row_ptr, col, val
        self.m, self.n, self.p = m, n, p

    def struct(self):
        return lra_operand(LRA_OP_FACTORED_CSR, LRA_F64, self.m, self.n, None, self.m, self.A_t.data_ptr(),
                           self.B_t.data_ptr(), self.p, self.row_ptr.data_ptr(), self.col.data_ptr(),
                           self.val.data_ptr(), 0, 0)


class Multiplier:
    """Device copy of a realized multiplier (``synth.multiplier_*`` dict)."""

    def __init__(self, mult: dict, device="cuda"):
        import torch
        self.mult = mult
        self.kind = mult["kind"]
        self.t = {}
        for key in ("dsign", "col", "sp_row", "sp_sign", "qg_sign", "qg_perm"):
            if key in mult:
                self.t[key] = torch.from_numpy(np.ascontiguousarray(mult[key])).to(device)
        if "omega" in mult:   # (lbar, n) storage of the n×lbar col-major matrix
            self.t["omega"] = torch.from_numpy(np.ascontiguousarray(np.asarray(mult["omega"]).T)).to(device)
        self.lbar = mult["lbar"]
        self.n = mult["n"]

    def struct(self):
        om = self.t.get("omega")
        return lra_multiplier(MUL_KIND[self.kind], int(self.mult.get("depth", 0)), self.lbar,
                              _ptr(self.t.get("dsign")), _ptr(self.t.get("col")), _ptr(self.t.get("sp_row")),
                              _ptr(self.t.get("sp_sign")), int(self.mult.get("nnz", 0)), _ptr(om),
                              self.n if om is not None else 0, _ptr(self.t.get("qg_sign")),
                              _ptr(self.t.get("qg_perm")))

    def m_stride(self):
        """Per-block stride for lra_batch: stacked sparse multipliers (synth.multiplier_sparse_batch)
        advance by lbar·nnz entries per block; every other multiplier is shared (0)."""
        if self.kind == "sparse" and "nb" in self.mult:
            return self.lbar * int(self.mult["nnz"])
        return 0


# ------------------------------------------------------------------ the C-ABI, same names
def nccl_unique_id():
    """128-byte NCCL unique id (create on one rank, distribute with torch.distributed)."""
    buf = C.create_string_buffer(128)
    _check(lib().lra_nccl_unique_id(buf))
    return buf.raw


class Handle:
    """lra_handle_create: nccl_id (bytes from nccl_unique_id) + nranks/rank give the handle an
    NCCL communicator for row-sharded operands; None for single-GPU use."""

    def __init__(self, device=0, nccl_id=None, nranks=1, rank=0):
        h = C.c_void_p()
        idbuf = C.create_string_buffer(nccl_id, 128) if nccl_id is not None else None
        _check(lib().lra_handle_create(C.byref(h), int(device), idbuf, int(nranks), int(rank)))
        self.h = h

    def close(self):
        if self.h:
            lib().lra_handle_destroy(self.h)
            self.h = None

    def __del__(self):
        try:
            self.close()
        except Exception:
            pass

    def launches(self):
        return int(lib().lra_launch_count(self.h))

    def profile(self, enable=True):
        _check(lib().lra_profile_enable(self.h, int(bool(enable))))

    def profile_read(self, cap=32):
        """{kernel name: (total ms, launches)} since the last enable/read (synchronizes)."""
        names = (C.c_char_p * cap)()
        ms = (C.c_double * cap)()
        cnt = (C.c_int64 * cap)()
        nd = lib().lra_profile_read(self.h, cap, names, ms, cnt)
        if nd < 0:
            _check(nd)
        return {names[i].decode(): (ms[i], int(cnt[i])) for i in range(nd)}


def lra_handle_create(device=0):
    return Handle(device)


def lra_maxvol(h, B, slots, start=None, stats=None, swap_tol=1e-12, tie_slack=1e-12, swap_cap=None, stream=None):
    """maxvol (Alg D.2 stage 1 + D.1) of a dense fp64 block: B is a (q, N) tensor = the N x q
    column-major block; slots (q,) int64 device."""
    q, N = B.shape
    cap = 20 * q if swap_cap is None else swap_cap
    _check(lib().lra_maxvol(h.h, _ptr(B), N, q, _ptr(start), swap_tol, tie_slack, cap, _ptr(slots), _ptr(stats),
                            _stream(stream)))


def lra_qrp_columns(h, W, I, q, piv, status, R=None, Rt=None, tie_slack=1e-12, stream=None):
    """Householder QRP column selection (Alg D.3) on W[I,:]: piv (q,) int64; R a (n, ldr)
    tensor (= q x n column-major, ld ldr) or None; Rt a (q, n) tensor (= n x q column-major)."""
    ldr = R.shape[-1] if R is not None else q
    _check(lib().lra_qrp_columns(h.h, C.byref(W.struct()), _ptr(I), I.numel(), q, tie_slack, _ptr(piv), _ptr(R), ldr,
                                 _ptr(Rt), _ptr(status), _stream(stream)))


def lra_workspace_query(h, W, r, k, sweeps, nb=0):
    """Device scratch bytes of the calls of this shape (nb = 0: single problem; nb >= 1: lra_batch)."""
    out = C.c_size_t(0)
    _check(lib().lra_workspace_query(h.h, C.byref(W.struct()), int(r), int(k), int(sweeps), int(nb), C.byref(out)))
    return int(out.value)


def lra_workspace_reserve(h, W, r, k, sweeps, nb=0):
    """Allocate that scratch now (the calls of this shape then allocate nothing)."""
    _check(lib().lra_workspace_reserve(h.h, C.byref(W.struct()), int(r), int(k), int(sweeps), int(nb)))


def lra_preprocess(h, W, M, Y, stream=None):
    """Y (lbar, m) float64 [or (lbar, m, 2) for ARFT] receives Y = W·M (column-major)."""
    ldy = Y.shape[1]
    _check(lib().lra_preprocess(h.h, C.byref(W.struct()), C.byref(M.struct()), _ptr(Y), ldy, _stream(stream)))


def lra_preprocess_full(h, W, M, Wout, stream=None):
    """Wout (n, m) tensor of W's dtype receives W' = W·D·H_{n,d}·P (Alg 10.1 stage 1, u = n)."""
    _check(lib().lra_preprocess_full(h.h, C.byref(W.struct()), C.byref(M.struct()), _ptr(Wout), Wout.shape[-1],
                                     _stream(stream)))


def lra_cross_approx(h, W, Y, I0, r, k, l, sweeps, I, J, U, A, B, stats=None, y_complex=False,
                     swap_tol=1e-12, tie_slack=1e-12, swap_cap=None, stream=None):
    ldy = Y.shape[1] if Y is not None else 0
    cap = 20 * k if swap_cap is None else swap_cap
    _check(lib().lra_cross_approx(h.h, C.byref(W.struct()), _ptr(Y), ldy, int(bool(y_complex)), _ptr(I0), r, k, l,
                                  sweeps, swap_tol, tie_slack, cap, _ptr(I), _ptr(J), _ptr(U), _ptr(A), _ptr(B),
                                  _ptr(stats), _stream(stream)))


def lra_cur_residual(h, W, A, B, r, num2, den2, nsamples=0, si=None, sj=None, prec=LRA_RECON_PRECISE, stream=None):
    _check(lib().lra_cur_residual(h.h, C.byref(W.struct()), _ptr(A), _ptr(B), r, prec, nsamples, _ptr(si), _ptr(sj),
                                  _ptr(num2), _ptr(den2), _stream(stream)))


def lra_expand_columns(h, W, I, J, g0, tie_slack=1e-12, stream=None):
    """J (l,) int64 device tensor: first g0 entries given, the rest filled greedily (Alg D.4)."""
    _check(lib().lra_expand_columns(h.h, C.byref(W.struct()), _ptr(I), I.numel(), _ptr(J), g0, J.numel(), tie_slack,
                                    _stream(stream)))


def lra_leverage_scores(h, W, idx, side, r, p, status, stream=None):
    """Leverage scores of the columns of W[idx,:] (side 0) or of the rows of W[:,idx] (side 1)."""
    _check(lib().lra_leverage_scores(h.h, C.byref(W.struct()), _ptr(idx), idx.numel(), int(side), int(r), _ptr(p),
                                     _ptr(status), _stream(stream)))


def lra_set_diagnostics(h, level):
    """level >= 1: the C-A fills lra_ca_stats.min_pivot_margin (global tier; debugging mode)."""
    _check(lib().lra_set_diagnostics(h.h, int(level)))


def lra_sample_exactly(h, p, u, idx, dscale=None, status=None, stream=None, N=None):
    """Alg C.1: idx (l,) int64 picks from p (N,) with the uniforms u (l,); p None = uniform 1/N."""
    N = p.numel() if p is not None else int(N)
    _check(lib().lra_sample_exactly(h.h, _ptr(p), N, idx.numel(), _ptr(u), _ptr(idx), _ptr(dscale),
                                    _ptr(status), _stream(stream)))


def lra_sample_expected(h, p, l, u, idx, count, dscale=None, status=None, stream=None):
    """Alg C.2: keeps i iff u[i] < min(1, l p[i]) (u (N,)); the kept i in ascending order into idx
    (cap = idx.numel()), their number into count ((1,) int64); p None = uniform 1/N."""
    _check(lib().lra_sample_expected(h.h, _ptr(p), u.numel(), int(l), _ptr(u), idx.numel(), _ptr(idx), _ptr(dscale),
                                     _ptr(count), _ptr(status), _stream(stream)))


def lra_contract_columns(h, W, I, J, l, tie_slack=1e-12, stream=None):
    """J (g0,) int64 device tensor: on return its first l entries are the contracted set."""
    _check(lib().lra_contract_columns(h.h, C.byref(W.struct()), _ptr(I), I.numel(), _ptr(J), J.numel(), l, tie_slack,
                                      _stream(stream)))


def lra_refine_columns(h, W, I, J, cycles, changed, tie_slack=1e-12, stream=None):
    """J (l,) int64 device tensor refined in place by expand-contract cycles; changed (1,) int32."""
    _check(lib().lra_refine_columns(h.h, C.byref(W.struct()), _ptr(I), I.numel(), _ptr(J), J.numel(), int(cycles),
                                    tie_slack, _ptr(changed), _stream(stream)))


def lra_nucleus_factors(h, W, I, J, r, U, A, B, status, stream=None):
    """U (k, l) storage of the l x k nucleus, A (r, m), B (n, r); status (1,) int32."""
    _check(lib().lra_nucleus_factors(h.h, C.byref(W.struct()), _ptr(I), _ptr(J), I.numel(), J.numel(), r, _ptr(U),
                                     _ptr(A), _ptr(B), _ptr(status), _stream(stream)))


def lra_cur_certificate(h, W, I, J, U, k, l, r, delta, stream=None):
    """(bound, |C|_F, |R|_F, |U|_F) of Cor cowc1 for the Frobenius-tail bound delta."""
    out = (C.c_double * 4)()
    _check(lib().lra_cur_certificate(h.h, C.byref(W.struct()), _ptr(I), _ptr(J), _ptr(U), k, l, r, float(delta), out,
                                     _stream(stream)))
    return tuple(out)


def lra_cur_progressive(h, W, Ms, r, k, sweeps, tol, rows, cols, Y, I, J, U, A, B, stats, stats4, stream=None):
    """Progressive depth in the library: Ms = Multipliers of depth 1, 2, ... tried in order until
    the sampled estimate is <= tol.  Returns (depth, estimate)."""
    arr = (lra_multiplier * len(Ms))(*[M.struct() for M in Ms])
    d = C.c_int32(0)
    est = C.c_double(0.0)
    _check(lib().lra_cur_progressive(h.h, C.byref(W.struct()), arr, len(Ms), r, k, sweeps, float(tol), _ptr(rows),
                                     rows.numel(), _ptr(cols), cols.numel(), _ptr(Y), _ptr(I), _ptr(J), _ptr(U),
                                     _ptr(A), _ptr(B), _ptr(stats), _ptr(stats4), C.byref(d), C.byref(est),
                                     _stream(stream)))
    return int(d.value), float(est.value)


def lra_error_sample(h, W, A, B, r, rows, cols, stats3, stream=None):
    """stats3 (4,) float64 device tensor <- (mu_K, sigma_K^2, sum g^2, sum W^2) of E[rows, cols]."""
    _check(lib().lra_error_sample(h.h, C.byref(W.struct()), _ptr(A), _ptr(B), r, _ptr(rows), rows.numel(),
                                  _ptr(cols), cols.numel(), _ptr(stats3), _stream(stream)))


def lra_variance_bound(var_K, K, alpha):
    out = C.c_double()
    _check(lib().lra_variance_bound(float(var_K), int(K), float(alpha), C.byref(out)))
    return out.value


def lra_batch(h, nb, W, M, r, k, l, sweeps, I, J, U, num2, den2, stats=None, swap_tol=1e-12, tie_slack=1e-12,
              swap_cap=None, prec=LRA_RECON_PRECISE, stream=None):
    cap = 20 * k if swap_cap is None else swap_cap
    _check(lib().lra_batch(h.h, nb, C.byref(W.struct()), W.block_stride(), C.byref(M.struct()), M.m_stride(), r, k, l,
                           sweeps, swap_tol, tie_slack, cap, prec, _ptr(I), _ptr(J), _ptr(U), _ptr(num2), _ptr(den2),
                           _ptr(stats), _stream(stream)))


def stats_to_numpy(stats_t):
    """Device stats buffer (uint8 tensor of 56·nb bytes) → numpy structured array."""
    return np.frombuffer(stats_t.cpu().numpy().tobytes(), dtype=STATS_DTYPE)


def new_stats(nb=1, device="cuda"):
    import torch
    return torch.zeros(STATS_DTYPE.itemsize * nb, dtype=torch.uint8, device=device)
