"""Pins of oracle/transforms.py and oracle.lra.sketch against what the paper fixes.

Every check here compares against something other than the oracle's own formula:
golden block patterns typed from the paper, the library DFT (numpy.fft), orthogonality
identities, brute-force dense products, and the closed forms vs the recursions."""
import os

import numpy as np
import pytest

import synth
from oracle import lra, transforms as T

GOLD = os.path.join(os.path.dirname(__file__), "golden")


def _load(name):
    return np.loadtxt(os.path.join(GOLD, name), comments="#")


@pytest.mark.parametrize("d,fname", [(1, "hadamard_blocks_d1.txt"), (2, "hadamard_blocks_d2.txt")])
@pytest.mark.parametrize("s", [1, 3, 5, 8])
def test_hadamard_displayed_matrices(d, fname, s):
    """H_{n,1}, H_{n,2} as displayed in eq. (eqbschf)."""
    pat = _load(fname)
    assert np.array_equal(T.hadamard_recursive((1 << d) * s, d), np.kron(pat, np.eye(s)))


@pytest.mark.parametrize("n,d", [(8, 1), (8, 3), (16, 2), (64, 6), (96, 5), (1000, 3), (800, 5), (1024, 4)])
def test_hadamard_closed_form_and_orthogonality(n, d):
    H = T.hadamard_recursive(n, d)
    k = np.arange(n)
    assert np.array_equal(H, T.hadamard_entry(n, d, k[:, None], k[None, :]))
    # orthogonal up to scaling with 2^d nonzeros per row / column
    assert np.array_equal(H.T @ H, (1 << d) * np.eye(n))
    assert np.all(np.count_nonzero(H, axis=0) == 1 << d)
    assert np.all(np.count_nonzero(H, axis=1) == 1 << d)
    for sig in [0, 1, n // 2 + 1, n - 1]:
        rows, vals = T.hadamard_column_support(n, d, sig)
        col = np.zeros(n)
        col[rows] = vals
        assert np.array_equal(col, H[:, sig])


@pytest.mark.parametrize("n", [2, 4, 8, 64, 256])
def test_full_hadamard_hht_is_nI(n):
    """d = log2 n: H_n H_nᵀ = n·I (north star's orthogonality pin)."""
    d = n.bit_length() - 1
    H = T.hadamard_recursive(n, d)
    assert np.array_equal(H @ H.T, n * np.eye(n))


@pytest.mark.parametrize("n", [2, 4, 8, 16, 64, 256])
def test_full_fourier_recursion_is_library_dft(n):
    """d = log2 n: the DIF recursion (eq. eqfd, readings C4) equals Ω_n = (ω^{ij}),
    ω = e^{+2πi/n} (eq. eqdft) — compared with numpy.fft (n·ifft of I = Σ_j ω^{ij} x_j)."""
    d = n.bit_length() - 1
    O = T.fourier_recursive(n, d)
    ref = n * np.fft.ifft(np.eye(n), axis=0)
    assert np.allclose(O, ref, atol=1e-12 * n)


@pytest.mark.parametrize("n,d", [(8, 1), (16, 2), (32, 3), (24, 3), (1000, 3), (256, 4)])
def test_abridged_fourier_closed_form_unitary(n, d):
    O = T.fourier_recursive(n, d)
    assert np.allclose(O.conj().T @ O, (1 << d) * np.eye(n), atol=1e-10)
    assert np.all(np.count_nonzero(np.abs(O) > 1e-12, axis=0) == 1 << d)
    for sig in range(n):
        rows, vals = T.fourier_column_support(n, d, sig)
        col = np.zeros(n, complex)
        col[rows] = vals
        assert np.allclose(col, O[:, sig], atol=1e-12)


def test_literal_fourier_recursion_is_not_dft():
    """Documents reading C4: the recursion exactly as printed (P̂ not transposed,
    D̂ = diag(ω_n^i)) does not reproduce Ω_8."""
    n = 8
    Om = np.eye(1, dtype=complex)
    q = 1
    while q < n:
        Dq = np.diag(np.exp(2j * np.pi * np.arange(q) / n))
        Om = T.even_odd_permutation(2 * q) @ np.vstack([np.hstack([Om, Om]), np.hstack([Om @ Dq, -(Om @ Dq)])])
        q *= 2
    assert not np.allclose(Om, T.dft_matrix(n))


@pytest.mark.parametrize("kind", ["arht", "arft"])
@pytest.mark.parametrize("m,n,d,lbar", [(40, 64, 3, 8), (33, 96, 5, 12), (20, 1000, 3, 6)])
def test_sketch_equals_dense_product(kind, m, n, d, lbar):
    """Y = W·(D·T_{n,d}·P)[:, σ] with T built by the paper's recursion (brute force)."""
    W = synth.factor_gaussian(5, m, n, 4, 1e-3)
    M = synth.multiplier_abridged(7, n, d, lbar, kind)
    Y = lra.sketch(W, M)
    ref = W @ T.multiplier_dense(M, n)
    assert np.allclose(Y, ref, rtol=0, atol=1e-13 * np.abs(W).max() * (1 << d))


def test_sketch_sparse_and_gaussian_dense_product():
    W = synth.factor_gaussian(1, 30, 50, 3, 1e-3)
    Ms = synth.multiplier_sparse(2, 50, 7)
    ref = W @ T.multiplier_dense(Ms, 50)
    assert np.allclose(lra.sketch(W, Ms), ref, atol=1e-13)
    # structure: 4 distinct rows, ±1 per column (reading C7)
    Md = T.multiplier_dense(Ms, 50)
    assert np.all(np.count_nonzero(Md, axis=0) == 4) and set(np.unique(Md)) <= {-1.0, 0.0, 1.0}
    Mg = synth.multiplier_gaussian(3, 50, 7)
    assert np.allclose(lra.sketch(W, Mg), W @ Mg["omega"], atol=1e-12)


def test_gaussian_sketch_fp32_products_exact():
    """fp32-mode Gaussian: every W_ij·Ω_jc is exact in fp64 (24+24 ≤ 53 bits), so the
    sequential fp64 sum is reproducible bit for bit with or without FMA."""
    from fractions import Fraction
    W = synth.config2(0, n=256, p=64)
    Mg = synth.multiplier_gaussian(3, 256, 5)
    for i, j, c in [(0, 7, 3), (17, 100, 0), (255, 255, 4)]:
        a = float(W[i, j])
        b = float(Mg["omega"][j, c])
        assert Fraction(a) * Fraction(b) == Fraction(a * b)
