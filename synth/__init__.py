"""Seeded synthetic inputs for the superfast-CUR hot path (arXiv 1710.07946).

This module is the ONLY code shared by the CUDA product path (``paper_1710_07946_b200``)
and the CPU oracle (``oracle/``).  It holds none of the method's arithmetic: it draws
matrices W of the shapes / value distributions of BASELINE.json's configs, and it
*realizes* the randomness that the method consumes (the ±1 diagonal D, the sampled
column order σ = P·S, the sparse ±1 pattern, the Gaussian multiplier Ω, a random
starting row set I₀).  Both implementations receive these arrays as data.

Every generator is a counter-based Philox stream keyed by (seed, stream), so the same
call returns the same bits on every machine.  Matrices are returned COLUMN-MAJOR
(numpy ``order='F'``, shape (m, n)), the layout the library expects.

Recipes (DESIGN.md §4 states them with citations):
  cfg1  W = G1·G2 + N, 256², G ~ N(0,1), N ~ N(0,1e-20) (variance)   [P:4686 family]
  cfg2  W = U·diag(σ)·Vᵀ (fp32), 4096², U,V = Q factors of Gaussian    [BASELINE.json]
  cfg3  W_ij = 1/(s_i − t_j) (fp32), s ~ U[0,1], t ~ U[2,3], 512² blocks
  cfg4  W = A·B + E, factored, never materialized (see ``config4``)
  cfg5  W = U·diag(σ)·Vᵀ + N generated per row shard (see ``config5_factors``)
"""
from __future__ import annotations

import numpy as np

# Stream ids.
S_G1, S_G2, S_NOISE, S_MULT, S_U, S_V, S_I0, S_SAMPLES = 0, 1, 2, 3, 4, 5, 6, 7


def rng(seed: int, stream: int) -> np.random.Generator:
    """Counter-based Philox4x32 stream for (seed, stream)."""
    return np.random.Generator(np.random.Philox(key=[int(seed) & (2**64 - 1), int(stream)]))


def _normal_colmajor(g: np.random.Generator, m: int, n: int) -> np.ndarray:
    # draw column by column (column-major fill), so the first p columns of an m×n draw
    # are exactly an m×p draw from the same stream
    return np.asfortranarray(g.standard_normal(m * n).reshape(n, m).T)


def _q_factor(G: np.ndarray) -> np.ndarray:
    """Q of the QR factorization with R's diagonal > 0 (the unique Q), fp64."""
    Q, R = np.linalg.qr(G)
    s = np.sign(np.diag(R))
    s[s == 0] = 1.0
    return np.asfortranarray(Q * s[None, :])


# --------------------------------------------------------------------------- configs
def config1(seed: int = 0, n: int = 256, r: int = 8, noise_var: float = 1e-20) -> np.ndarray:
    """W = G1·G2 + N (fp64), the Table tb_ranrc input family at n, r."""
    G1 = _normal_colmajor(rng(seed, S_G1), n, r)
    G2 = _normal_colmajor(rng(seed, S_G2), r, n)
    N = _normal_colmajor(rng(seed, S_NOISE), n, n) * np.sqrt(noise_var)
    return np.asfortranarray(G1 @ G2 + N)


def factor_gaussian(seed: int, m: int, n: int, r: int, noise_var: float = 0.0) -> np.ndarray:
    """Generic perturbed factor-Gaussian m×n matrix of rank r (Def. defgsfc)."""
    G1 = _normal_colmajor(rng(seed, S_G1), m, r)
    G2 = _normal_colmajor(rng(seed, S_G2), r, n)
    W = G1 @ G2
    if noise_var:
        W = W + _normal_colmajor(rng(seed, S_NOISE), m, n) * np.sqrt(noise_var)
    return np.asfortranarray(W)


def config2_sigma(n: int = 4096, r: int = 32) -> np.ndarray:
    i = np.arange(1, n + 1, dtype=np.float64)
    return np.where(i <= r, 1.0, 1e-6 * 0.9 ** (i - r))


def config2(seed: int = 0, n: int = 4096, r: int = 32, p: int = 320) -> np.ndarray:
    """W = U·diag(σ)·Vᵀ rounded to fp32, σ_i = 1 (i ≤ 32), 1e-6·0.9^(i−32) beyond.

    U, V are Q factors of i.i.d. N(0,1) n×n matrices.  The first p columns of Q depend
    only on the first p columns of G (Householder QR with positive diag(R) is unique), and
    σ_p·max|u||v| for p = 320 is ~1e-19, far below the fp32 rounding of W (~1e-10), so only
    the first p columns are drawn (reading C20).
    """
    sig = config2_sigma(n, r)[:p]
    U = _q_factor(_normal_colmajor(rng(seed, S_U), n, p))
    V = _q_factor(_normal_colmajor(rng(seed, S_V), n, p))
    W = (U * sig[None, :]) @ V.T
    return np.asfortranarray(W.astype(np.float32))


def cauchy_params(seed: int, nb: int, m: int = 512, n: int = 512):
    """s_i ~ U[0,1] (m per block), t_j ~ U[2,3] (n per block), fp64; block b uses stream 100+b."""
    s = np.empty((nb, m))
    t = np.empty((nb, n))
    for b in range(nb):
        g = rng(seed, 100 + b)
        s[b] = g.random(m)
        t[b] = 2.0 + g.random(n)
    return s, t


def cauchy_block(s: np.ndarray, t: np.ndarray) -> np.ndarray:
    """W_ij = fl32(1/(s_i − t_j)) — elementwise IEEE ops only, so torch on any device
    produces identical bits (see ``cauchy_blocks_torch``)."""
    return np.asfortranarray((1.0 / (s[:, None] - t[None, :])).astype(np.float32))


def cauchy_blocks_torch(s, t, device):
    """All blocks at once on ``device``: returns a torch tensor (nb, n, m) contiguous, i.e.
    block b is a column-major m×n matrix.  Same IEEE elementwise ops as cauchy_block."""
    import torch
    st = torch.as_tensor(s, dtype=torch.float64, device=device)
    tt = torch.as_tensor(t, dtype=torch.float64, device=device)
    # element (b, j, i) = 1/(s[b,i] - t[b,j])
    return (1.0 / (st[:, None, :] - tt[:, :, None])).to(torch.float32).contiguous()


def config4(seed: int = 0, m: int = 65536, n: int = 65536, p: int = 16,
            dens_ab: float = 0.05, dens_e: float = 1e-4, var_e: float = 1e-6):
    """W = A·B + E, never materialized.  A m×p, B p×n Bernoulli(dens_ab)·N(0,1) (stored
    dense, column-major); E Bernoulli(dens_e) positions with N(0,var_e) values, in CSR
    over rows (row_ptr int64[m+1], col int64[nnz] ascending per row, val fp64)."""
    g = rng(seed, S_G1)
    A = np.where(g.random((p, m)).T < dens_ab, g.standard_normal((p, m)).T, 0.0)
    A = np.asfortranarray(A)
    g = rng(seed, S_G2)
    B = np.where(g.random((n, p)).T < dens_ab, g.standard_normal((n, p)).T, 0.0)
    B = np.asfortranarray(B)
    g = rng(seed, S_NOISE)
    # Bernoulli(dens_e) per entry == binomial count, then that many distinct uniform cells
    nnz_total = int(g.binomial(m * n, dens_e))
    flat = np.unique(g.integers(0, m * n, size=int(nnz_total * 1.01) + 64))
    if flat.size < nnz_total:
        raise RuntimeError("config4: not enough distinct cells drawn")
    flat = flat[np.sort(g.choice(flat.size, size=nnz_total, replace=False))]
    rows = flat // n
    cols = flat % n
    val = g.standard_normal(flat.size) * np.sqrt(var_e)
    row_ptr = np.zeros(m + 1, dtype=np.int64)
    np.add.at(row_ptr, rows + 1, 1)
    row_ptr = np.cumsum(row_ptr)
    # W entries are fp32 numbers: round each term's representation (cfg4)
    return dict(A=A.astype(np.float32).astype(np.float64), B=B.astype(np.float32).astype(np.float64),
                row_ptr=row_ptr, col=cols.astype(np.int64),
                val=val.astype(np.float32).astype(np.float64), m=m, n=n, p=p)


def config5_sigma(p: int = 64) -> np.ndarray:
    i = np.arange(1, p + 1, dtype=np.float64)
    return 10.0 ** (-3.0 * (i - 1) / 63.0)


# ------------------------------------------------------------ realized multipliers
def multiplier_abridged(seed: int, n: int, d: int, lbar: int, kind: str = "arht") -> dict:
    """Realized randomness of an abridged randomized Hadamard/Fourier multiplier
    D·H_{n,d}·P (resp. D·Ω_{n,d}·P) followed by sampling lbar columns:
    dsign ∈ {±1}^n (Rademacher, reading C5) and col = the first lbar entries of a uniform
    random permutation of [0, n) in draw order (P·S, reading C6)."""
    if n % (1 << d):
        raise ValueError("2^d must divide n")
    g = rng(seed, S_MULT)
    dsign = (g.integers(0, 2, size=n) * 2 - 1).astype(np.int8)
    col = g.permutation(n)[:lbar].astype(np.int64)
    return dict(kind=kind, depth=int(d), lbar=int(lbar), dsign=dsign, col=col, n=int(n))


def multiplier_sparse(seed: int, n: int, lbar: int, nnz: int = 4) -> dict:
    """Sparse ±1 multiplier: each of the lbar columns has nnz distinct uniform rows with
    Rademacher signs (reading C7).  Arrays are column-sliced: entry t of column c is at
    c·nnz + t, in draw order."""
    g = rng(seed, S_MULT)
    rows = np.empty(lbar * nnz, dtype=np.int64)
    for c in range(lbar):
        rows[c * nnz:(c + 1) * nnz] = g.choice(n, size=nnz, replace=False)
    signs = (g.integers(0, 2, size=lbar * nnz) * 2 - 1).astype(np.int8)
    return dict(kind="sparse", depth=0, lbar=int(lbar), sp_row=rows, sp_sign=signs, nnz=int(nnz), n=int(n))


def multiplier_sparse_batch(seed: int, nb: int, n: int, lbar: int, nnz: int = 4) -> dict:
    """One sparse multiplier per block, block b from stream 100000+b; arrays stacked."""
    rows = np.empty((nb, lbar * nnz), dtype=np.int64)
    signs = np.empty((nb, lbar * nnz), dtype=np.int8)
    for b in range(nb):
        g = rng(seed, 100000 + b)
        for c in range(lbar):
            rows[b, c * nnz:(c + 1) * nnz] = g.choice(n, size=nnz, replace=False)
        signs[b] = (g.integers(0, 2, size=lbar * nnz) * 2 - 1).astype(np.int8)
    return dict(kind="sparse", depth=0, lbar=int(lbar), sp_row=rows, sp_sign=signs, nnz=int(nnz), n=int(n), nb=nb)


def multiplier_gaussian(seed: int, n: int, lbar: int, round_fp32: bool = True) -> dict:
    """Gaussian n×lbar multiplier Ω, column-major fp64.  In fp32 mode its
    entries are rounded to fp32 values (then every product W_ij·Ω_jc is exact in fp64)."""
    om = _normal_colmajor(rng(seed, S_MULT), n, lbar)
    if round_fp32:
        om = om.astype(np.float32).astype(np.float64)
    return dict(kind="gaussian", depth=0, lbar=int(lbar), omega=np.asfortranarray(om), n=int(n))


def multiplier_qgauss(seed: int, n: int, q: int, lbar: int) -> dict:
    """Quasi-Gaussian multiplier (NEXT-4, section sqsgss / sgpbd, def11):
    G_q = M_0 M_1 ... M_{q-1} with M_i = B_i P_i, B_i the cyclic bidiagonal matrix with ones on
    the diagonal and random signs s_i[c] at (c + 1 mod n, c) (the corner is c = n - 1), P_i a
    uniform random permutation with P_i[perm_i[c], c] = 1; then lbar sampled columns (the
    first lbar of a uniform permutation, reading C30).  Arrays: sign (q, n) int8, perm (q, n)
    int64, col (lbar,)."""
    g = rng(seed, S_MULT)
    sign = (g.integers(0, 2, size=(q, n)) * 2 - 1).astype(np.int8)
    perm = np.stack([g.permutation(n) for _ in range(q)]).astype(np.int64)
    col = g.permutation(n)[:lbar].astype(np.int64)
    return dict(kind="qgauss", depth=int(q), lbar=int(lbar), qg_sign=sign, qg_perm=perm, col=col, n=int(n))


def leverage_uniforms(seed: int, sweeps: int, k: int, l: int):
    """The uniforms of the leverage-score sampling (Alg C.1) of cur_leverage: for sweep s,
    (l,) for the columns then (k,) for the rows, in [0, 1)."""
    g = rng(seed, S_MULT + 7)
    out = []
    for _ in range(sweeps):
        out.append(g.random(l))
        out.append(g.random(k))
    return out


def random_rows(seed: int, m: int, k: int) -> np.ndarray:
    """k distinct uniform row indices (Tests 2 random start I₀)."""
    return rng(seed, S_I0).permutation(m)[:k].astype(np.int64)


def sample_pairs(seed: int, m: int, n: int, q: int):
    """q i.i.d. uniform (i, j) pairs for the sampled a-posteriori check."""
    g = rng(seed, S_SAMPLES)
    return g.integers(0, m, size=q).astype(np.int64), g.integers(0, n, size=q).astype(np.int64)


# ------------------------------------------------------------ config 5 (device generator)
def config5_factors(seed: int, m: int, n: int, p: int = 64):
    """U (m×p), V (n×p) with orthonormal columns: Q factors (diag R > 0, reading C20) of
    i.i.d. N(0,1) matrices from Philox streams (seed, 50) / (seed, 51); fp64, host."""
    U = _q_factor(_normal_colmajor(rng(seed, 50), m, p))
    V = _q_factor(_normal_colmajor(rng(seed, 51), n, p))
    return U, V


def config5_torch(seed: int, m: int, n: int, row0: int = 0, rows: int = None, device="cuda",
                  noise_std: float = 1e-4, factors=None, block: int = 1024):
    """Row shard [row0, row0+rows) of W = U·diag(σ)·Vᵀ + N (BASELINE config 5; σ_i =
    10^(-3(i-1)/63), N i.i.d. N(0, 1e-8), i.e. std 1e-4 — reading C15), generated on
    ``device`` as a (n, rows) fp32 tensor = the column-major m_local×n shard.  The noise of
    every 1024-row block comes from its own seeded torch generator, so a shard's bits do not
    depend on how the rows are split over ranks."""
    import torch
    rows = m - row0 if rows is None else rows
    U, V = factors if factors is not None else config5_factors(seed, m, n)
    sig = config5_sigma(U.shape[1])
    Us = torch.from_numpy(np.ascontiguousarray((U[row0:row0 + rows] * sig[None, :]).T)).to(device, torch.float32)
    Vt = torch.from_numpy(np.ascontiguousarray(V)).to(device, torch.float32)
    out = torch.empty((n, rows), dtype=torch.float32, device=device)
    prev = torch.backends.cuda.matmul.allow_tf32
    torch.backends.cuda.matmul.allow_tf32 = False
    try:
        torch.matmul(Vt, Us, out=out)                       # (n, rows) = V · (U_shard σ)ᵀ
    finally:
        torch.backends.cuda.matmul.allow_tf32 = prev
    b0 = row0 // block
    for b in range(b0, (row0 + rows + block - 1) // block):
        lo, hi = max(b * block, row0), min((b + 1) * block, row0 + rows)
        g = torch.Generator(device=device).manual_seed(int(seed) * 1000003 + b)
        z = torch.randn((n, block), generator=g, device=device, dtype=torch.float32)
        out[:, lo - row0:hi - row0] += noise_std * z[:, lo - b * block:hi - b * block]
    return out


# ------------------------------------------------------------ NEXT-4: Table tb_Lp input
def laplacian_tb_lp(n: int) -> np.ndarray:
    """The discretized single-layer Laplacian of Table tb_Lp (after [HMT11, 7.1]):
    w_ij = psi * int_{Gamma_1,j} log|2 omega^i - y| dy, Gamma_1 the unit circle, Gamma_1,j its
    arc of angles [2 j pi / n, 2 (j+1) pi / n], omega = exp(2 pi sqrt(-1) / n) (the points
    2 omega^i lie on Gamma_2 = C(0, 2)), psi such that ||W|| = 1 (spectral norm).
    With phi = theta - 2 pi i / n, log|2 - e^{i phi}| = log 2 - sum_{k>=1} 2^-k cos(k phi) / k,
    so the arc integral is (b - a) log 2 - sum_k 2^-k (sin(k b) - sin(k a)) / k^2 over the
    shifted arc [a, b] (60 terms: below 2^-60).  W is circulant (w_ij depends on j - i mod n);
    psi = 1 / max |eigenvalue| (the DFT of its first row).  fp64, deterministic (no seed)."""
    a0 = 2.0 * np.pi * np.arange(n) / n                   # arc starts, i = 0
    b0 = a0 + 2.0 * np.pi / n
    kk = np.arange(1, 61, dtype=np.float64)
    c = (b0 - a0) * np.log(2.0) - np.sum((0.5 ** kk)[None, :] * (np.sin(kk[None, :] * b0[:, None]) -
                                                                 np.sin(kk[None, :] * a0[:, None])) / kk[None, :] ** 2,
                                           axis=1)         # first row: i = 0, j = 0..n-1
    W = np.empty((n, n))
    for i in range(n):
        W[i] = np.roll(c, i)                                # w_ij = c[(j - i) mod n]
    psi = 1.0 / np.max(np.abs(np.fft.fft(c)))
    return np.asfortranarray(W * psi)
