"""End-to-end call sequence of the hot path through the C-ABI (user-facing convenience).

``cur`` runs Alg 10.2 + C-A (stages 1–3), the canonical nucleus and the a-posteriori
check on one dense matrix: lra_preprocess → lra_cross_approx → lra_cur_residual.
``cur_batch`` runs ``lra_batch`` on nb same-shape blocks.  All work happens in liblra.so.
"""
from __future__ import annotations

import torch

from . import lra as L


class CurBuffers:
    """Preallocated device outputs for one problem (reused across calls)."""

    def __init__(self, m, n, r, k, cplx=False, device="cuda"):
        f64 = dict(dtype=torch.float64, device=device)
        self.Y = torch.empty((k, m, 2) if cplx else (k, m), **f64)
        self.I = torch.empty(k, dtype=torch.int64, device=device)
        self.J = torch.empty(k, dtype=torch.int64, device=device)
        self.U = torch.empty((k, k), **f64)          # l×k column-major
        self.A = torch.empty((r, m), **f64)          # m×r column-major
        self.B = torch.empty((n, r), **f64)          # r×n column-major
        self.num2 = torch.empty(1, **f64)
        self.den2 = torch.empty(1, **f64)
        self.stats = L.new_stats(1, device)


def cur(h, W, M, r, k, sweeps, bufs=None, I0=None, swap_tol=1e-12, tie_slack=1e-12, stream=None):
    """W: lra.Dense (or lra.Factored with M None and I0 given); M: lra.Multiplier or None."""
    cplx = M is not None and M.kind == "arft"
    if bufs is None:
        bufs = CurBuffers(W.m, W.n, r, k, cplx)
    if M is not None:
        L.lra_preprocess(h, W, M, bufs.Y, stream=stream)
        Y = bufs.Y
    else:
        Y = None
    L.lra_cross_approx(h, W, Y, I0, r, k, k, sweeps, bufs.I, bufs.J, bufs.U, bufs.A, bufs.B, bufs.stats,
                       y_complex=cplx, swap_tol=swap_tol, tie_slack=tie_slack, stream=stream)
    if isinstance(W, L.Dense):
        L.lra_cur_residual(h, W, bufs.A, bufs.B, r, bufs.num2, bufs.den2, stream=stream)
    return bufs


class BatchBuffers:
    def __init__(self, nb, r, k, device="cuda"):
        self.I = torch.empty((nb, k), dtype=torch.int64, device=device)
        self.J = torch.empty((nb, k), dtype=torch.int64, device=device)
        self.U = torch.empty((nb, k, k), dtype=torch.float64, device=device)
        self.num2 = torch.empty(nb, dtype=torch.float64, device=device)
        self.den2 = torch.empty(nb, dtype=torch.float64, device=device)
        self.stats = L.new_stats(nb, device)


def cur_batch(h, W, M, r, k, sweeps, nb, bufs=None, swap_tol=1e-12, tie_slack=1e-12, stream=None):
    if bufs is None:
        bufs = BatchBuffers(nb, r, k)
    L.lra_batch(h, nb, W, M, r, k, k, sweeps, bufs.I, bufs.J, bufs.U, bufs.num2, bufs.den2, bufs.stats,
                swap_tol=swap_tol, tie_slack=tie_slack, stream=stream)
    return bufs


def cur_preprocessed(h, W, M_full, r, k, sweeps, I0, stream=None):
    """Alg 10.1 with C-A (the Table tb_fh protocol): W' = W·D·H_{n,d}·P (lra_preprocess_full),
    then lra_cross_approx (random start I0) and lra_cur_residual on W'.  C = W'[:,J], U and
    R = W[I,:] form the CUR LRA of W; the returned residual ratio (num2/den2 on W') equals the
    one of W in exact arithmetic (M M^T = 2^d I).  Returns (bufs, Wp)."""
    import torch
    Wp = torch.empty_like(W.Wt)
    L.lra_preprocess_full(h, W, M_full, Wp, stream=stream)
    Wpd = L.Dense(Wp)
    bufs = cur(h, Wpd, None, r, k, sweeps, I0=I0, stream=stream)
    return bufs, Wp


def cur_progressive(h, W, r, k, sweeps, tol, seed, rows, cols, dmax=6, stream=None):
    """Progressive-depth pre-processing through lra_cur_progressive: the ARHT
    multipliers of depth d = 1 .. D (realized by the seeded generator; D = dmax or the largest
    depth with 2^d | n) are handed to the library, which runs sketch -> C-A -> nucleus/factors ->
    superfast sampled estimate per depth and stops at the first estimate <= tol.
    Returns (d, bufs, estimate)."""
    import synth
    D = 1
    while D < dmax and W.n % (1 << (D + 1)) == 0:
        D += 1
    Ms = [L.Multiplier(synth.multiplier_abridged(seed, W.n, d, k, "arht")) for d in range(1, D + 1)]
    bufs = CurBuffers(W.m, W.n, r, k)
    stats4 = torch.empty(4, dtype=torch.float64, device=W.Wt.device)
    d, est = L.lra_cur_progressive(h, W, Ms, r, k, sweeps, tol, rows, cols, bufs.Y, bufs.I, bufs.J, bufs.U, bufs.A,
                                   bufs.B, bufs.stats, stats4, stream=stream)
    return d, bufs, est


def cur_rectangular(h, W, M, r, k, l, sweeps, stream=None):
    """k x l generators, l > k (NEXT-3): the square C-A (k = k) of Alg 10.2, Alg D.4 greedy
    expansion of J to l columns, then the canonical nucleus / factors of the k x l generator
    and the a-posteriori check.  Returns (square bufs, J (l,), U (k, l), A, B, num2, den2)."""
    bufs = cur(h, W, M, r, k, sweeps, stream=stream)
    dev = bufs.I.device
    J = torch.empty(l, dtype=torch.int64, device=dev)
    J[:k] = bufs.J
    L.lra_expand_columns(h, W, bufs.I, J, k, stream=stream)
    U = torch.empty((k, l), dtype=torch.float64, device=dev)
    A = torch.empty((r, W.m), dtype=torch.float64, device=dev)
    B = torch.empty((W.n, r), dtype=torch.float64, device=dev)
    status = torch.zeros(1, dtype=torch.int32, device=dev)
    L.lra_nucleus_factors(h, W, bufs.I, J, r, U, A, B, status, stream=stream)
    num2 = torch.empty(1, dtype=torch.float64, device=dev)
    den2 = torch.empty(1, dtype=torch.float64, device=dev)
    L.lra_cur_residual(h, W, A, B, r, num2, den2, stream=stream)
    return bufs, J, U, A, B, num2, den2


def cur_projective(h, W, M, r, k, l, sweeps, stream=None):
    """k x l generators of maximal r-projective volume (NEXT-3, Alg 7.1): the square C-A of
    Alg 10.2 gives the k rows I; on R = W[I,:] the Householder QRP (Alg D.3, r steps) gives
    R' (r x n); maxvol of R'^T gives r columns, Alg D.4 expands them to l; then the canonical
    nucleus / factors of the k x l generator and the a-posteriori check.
    Returns (square bufs, J (l,), U (k, l), A, B, num2, den2, piv (r,))."""
    cplx = M is not None and M.kind == "arft"
    bufs = CurBuffers(W.m, W.n, r, k, cplx)
    L.lra_preprocess(h, W, M, bufs.Y, stream=stream)
    L.lra_cross_approx(h, W, bufs.Y, None, r, k, k, sweeps, bufs.I, bufs.J, bufs.U, bufs.A, bufs.B, bufs.stats,
                       y_complex=cplx, stream=stream)
    dev = bufs.I.device
    piv = torch.empty(r, dtype=torch.int64, device=dev)
    status = torch.zeros(2, dtype=torch.int32, device=dev)
    Rp = torch.empty((W.n, r), dtype=torch.float64, device=dev)      # R' (r x n column-major)
    Rt = torch.empty((r, W.n), dtype=torch.float64, device=dev)      # R'^T (n x r column-major)
    L.lra_qrp_columns(h, W, bufs.I, r, piv, status[0:1], R=Rp, Rt=Rt, stream=stream)
    J = torch.empty(l, dtype=torch.int64, device=dev)
    L.lra_maxvol(h, Rt, J[:r], stream=stream)
    if l > r:
        rows = torch.arange(r, dtype=torch.int64, device=dev)
        L.lra_expand_columns(h, L.Dense(Rp), rows, J, r, stream=stream)
    U = torch.empty((k, l), dtype=torch.float64, device=dev)
    A = torch.empty((r, W.m), dtype=torch.float64, device=dev)
    B = torch.empty((W.n, r), dtype=torch.float64, device=dev)
    L.lra_nucleus_factors(h, W, bufs.I, J, r, U, A, B, status[1:2], stream=stream)
    num2 = torch.empty(1, dtype=torch.float64, device=dev)
    den2 = torch.empty(1, dtype=torch.float64, device=dev)
    L.lra_cur_residual(h, W, A, B, r, num2, den2, stream=stream)
    return bufs, J, U, A, B, num2, den2, piv


def cur_leverage(h, W, r, k, l, sweeps, I0, uniforms, stream=None):
    """C-A iterations with DMM08's leverage-score sampling as the subalgorithm (NEXT-4; Alg 9.1
    stages 1-2 with Alg C.1 in every horizontal and vertical step, section ststc-alvrg): from
    the rows I0, each sweep samples l columns from the leverage scores of W[I,:] and k rows from
    those of W[:,J]^T with the given uniforms (device tensors: uniforms[2s] (l,), [2s+1] (k,));
    then the canonical nucleus / factors and the a-posteriori check.
    Returns (I, J, U (k, l), A, B, num2, den2, status (3,))."""
    dev = I0.device
    I = I0.clone()
    J = torch.empty(l, dtype=torch.int64, device=dev)
    pc = torch.empty(W.n, dtype=torch.float64, device=dev)
    pr = torch.empty(W.m, dtype=torch.float64, device=dev)
    status = torch.zeros(3, dtype=torch.int32, device=dev)
    for s in range(sweeps):
        L.lra_leverage_scores(h, W, I, 0, r, pc, status[0:1], stream=stream)
        L.lra_sample_exactly(h, pc, uniforms[2 * s], J, status=status[0:1], stream=stream)
        L.lra_leverage_scores(h, W, J, 1, r, pr, status[1:2], stream=stream)
        L.lra_sample_exactly(h, pr, uniforms[2 * s + 1], I, status=status[1:2], stream=stream)
    U = torch.empty((k, l), dtype=torch.float64, device=dev)
    A = torch.empty((r, W.m), dtype=torch.float64, device=dev)
    B = torch.empty((W.n, r), dtype=torch.float64, device=dev)
    L.lra_nucleus_factors(h, W, I, J, r, U, A, B, status[2:3], stream=stream)
    num2 = torch.empty(1, dtype=torch.float64, device=dev)
    den2 = torch.empty(1, dtype=torch.float64, device=dev)
    L.lra_cur_residual(h, W, A, B, r, num2, den2, stream=stream)
    return I, J, U, A, B, num2, den2, status


def cur_uniform(h, W, r, k, l, u_cols, u_rows, sampler="exactly", stream=None):
    """Alg 9.1 with UNIFORM leverage scores (the superfast variant of section slrasmpav,
    P:3363-3575; NEXT-4): the columns J from p_j = 1/n and the rows I from 1/m, sampled by
    Alg C.1 (sampler "exactly": u_cols (l,), u_rows (k,)) or Alg C.2 ("expected": u_cols (n,),
    u_rows (m,)), then the canonical nucleus / factors and the a-posteriori check.  With
    "expected" the sample sizes are random: the counts are read back to size the nucleus call
    (one host sync).  Returns (I, J, U, A, B, num2, den2, status (1,))."""
    dev = u_cols.device
    status = torch.zeros(1, dtype=torch.int32, device=dev)
    if sampler == "exactly":
        J = torch.empty(l, dtype=torch.int64, device=dev)
        I = torch.empty(k, dtype=torch.int64, device=dev)
        L.lra_sample_exactly(h, None, u_cols, J, stream=stream, N=W.n)
        L.lra_sample_exactly(h, None, u_rows, I, stream=stream, N=W.m)
    else:
        J = torch.empty(W.n, dtype=torch.int64, device=dev)
        I = torch.empty(W.m, dtype=torch.int64, device=dev)
        cnt = torch.empty(2, dtype=torch.int64, device=dev)
        L.lra_sample_expected(h, None, l, u_cols, J, cnt[0:1], stream=stream)
        L.lra_sample_expected(h, None, k, u_rows, I, cnt[1:2], stream=stream)
        lc, kc = (int(x) for x in cnt.cpu())
        J, I = J[:lc].contiguous(), I[:kc].contiguous()
    U = torch.empty((I.numel(), J.numel()), dtype=torch.float64, device=dev)
    A = torch.empty((r, W.m), dtype=torch.float64, device=dev)
    B = torch.empty((W.n, r), dtype=torch.float64, device=dev)
    L.lra_nucleus_factors(h, W, I, J, r, U, A, B, status, stream=stream)
    num2 = torch.empty(1, dtype=torch.float64, device=dev)
    den2 = torch.empty(1, dtype=torch.float64, device=dev)
    L.lra_cur_residual(h, W, A, B, r, num2, den2, stream=stream)
    return I, J, U, A, B, num2, den2, status
