"""Abridged Hadamard / Fourier matrices (PAPER.md Appendix "sahaf").

TEST INFRASTRUCTURE (see oracle/__init__.py).  Dense builders follow the paper's
recursions literally (with readings C3/C4 of DESIGN.md); closed forms restate the same
matrices entrywise and are pinned against the recursions by tests/test_oracle_transforms.py.
"""
from __future__ import annotations

import numpy as np


# ----------------------------------------------------------------- Hadamard (eqrfd)
def hadamard_recursive(n: int, d: int) -> np.ndarray:
    """H_{n,d}: apply H_{2q} = [[H_q, H_q], [H_q, −H_q]] (eq. eqrfd) for
    q = s, 2s, …, n/2 starting from H_s = I_s, n = 2^d·s.

    Reading C3: the paper's index range "q = 2^h s, h = k−d…k−1" is taken as the d
    doublings from s to n (it equals eq. eqbschf for d = 1, 2)."""
    if d < 0 or n % (1 << d):
        raise ValueError("need 2^d | n")
    s = n >> d
    H = np.eye(s)
    for _ in range(d):
        H = np.block([[H, H], [H, -H]])
    return H


def hadamard_entry(n: int, d: int, k: np.ndarray, j: np.ndarray) -> np.ndarray:
    """Closed form of H_{n,d} = H_{2^d} ⊗ I_s:
    H[k, j] = [k ≡ j (mod s)] · (−1)^{popcount(⌊k/s⌋ & ⌊j/s⌋)}."""
    s = n >> d
    k = np.asarray(k)
    j = np.asarray(j)
    same = (k % s) == (j % s)
    a = (k // s) & (j // s)
    par = np.zeros(np.broadcast(a, a).shape, dtype=np.int64) + a
    pc = np.zeros_like(par)
    while np.any(par):
        pc += par & 1
        par >>= 1
    return np.where(same, np.where(pc % 2 == 0, 1.0, -1.0), 0.0)


def hadamard_column_support(n: int, d: int, sigma: int):
    """Nonzeros of column σ of H_{n,d}, in ascending row order:
    rows (σ mod s) + t·s, t = 0..2^d−1, values (−1)^{popcount(t & ⌊σ/s⌋)}."""
    s = n >> d
    t = np.arange(1 << d)
    rows = (sigma % s) + t * s
    return rows, hadamard_entry(n, d, rows, np.full_like(rows, sigma))


# ------------------------------------------------------------------ Fourier (eqfd)
def dft_matrix(n: int) -> np.ndarray:
    """Ω_n = (ω_n^{ij}), ω_n = exp(2π√−1/n) (eq. eqdft)."""
    i = np.arange(n)
    e = np.outer(i, i) % n
    return np.exp(2j * np.pi * e / n)


def even_odd_permutation(q2: int) -> np.ndarray:
    """P̂_{2q} as written: v_j = u_{2j}, v_{j+q} = u_{2j+1}."""
    P = np.zeros((q2, q2))
    q = q2 // 2
    for j in range(q):
        P[j, 2 * j] = 1.0
        P[j + q, 2 * j + 1] = 1.0
    return P


def fourier_recursive(n: int, d: int) -> np.ndarray:
    """Ω_{n,d}: apply the DIF step (eq. eqfd)
        Ω_{2q} = P̂_{2q}ᵀ [[Ω_q, Ω_q], [Ω_q D̂_q, −Ω_q D̂_q]]
    for q = s, 2s, …, n/2 from Ω_s = I_s.

    Reading C4: D̂_q = diag(ω_{2q}^i)_{i<q} (the paper prints ω_n^i with
    i < n, which is not q×q) and the output permutation is P̂ᵀ (interleave); with these
    two readings d = log2 n reproduces eq. eqdft exactly (pinned against the library DFT)."""
    if d < 0 or n % (1 << d):
        raise ValueError("need 2^d | n")
    s = n >> d
    Om = np.eye(s, dtype=complex)
    q = s
    for _ in range(d):
        Dq = np.diag(np.exp(2j * np.pi * np.arange(q) / (2 * q)))
        top = np.hstack([Om, Om])
        bot = np.hstack([Om @ Dq, -(Om @ Dq)])
        Om = even_odd_permutation(2 * q).T @ np.vstack([top, bot])
        q *= 2
    return Om


def fourier_column_support(n: int, d: int, sigma: int):
    """Closed form of column σ of Ω_{n,d} (pinned against fourier_recursive):
    rows 2^d·(σ mod s) + t, t = 0..2^d−1, values ω_n^{tσ} (exponent reduced mod n
    in integers before the trig call), evaluated as cos(a) + i sin(a) with a = fl(fl(2π e)/n)
    — DESIGN.md reading C32 (one fixed faithful rounding of ω_n^e)."""
    s = n >> d
    q = 1 << d
    t = np.arange(q)
    rows = q * (sigma % s) + t
    e = (t * sigma) % n
    ang = (2.0 * np.pi * e.astype(np.float64)) / float(n)   # fl(fl(2π·e)/n)
    return rows, np.cos(ang) + 1j * np.sin(ang)


def multiplier_dense(mult: dict, n: int) -> np.ndarray:
    """The n×lbar multiplier M = (D·T·P)[:, σ] materialized densely by the recursions
    (T = H_{n,d} or Ω_{n,d}), or the sparse/Gaussian multiplier as a dense matrix."""
    kind = mult["kind"]
    if kind in ("arht", "arft"):
        T = hadamard_recursive(n, mult["depth"]) if kind == "arht" else fourier_recursive(n, mult["depth"])
        D = mult["dsign"].astype(np.float64)
        return D[:, None] * T[:, mult["col"]]
    if kind == "sparse":
        lbar, nnz = mult["lbar"], mult["nnz"]
        M = np.zeros((n, lbar))
        for c in range(lbar):
            for t in range(nnz):
                M[mult["sp_row"][c * nnz + t], c] += float(mult["sp_sign"][c * nnz + t])
        return M
    if kind == "gaussian":
        return np.array(mult["omega"], dtype=np.float64)
    raise ValueError(kind)
