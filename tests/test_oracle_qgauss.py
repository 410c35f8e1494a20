"""Pins of the quasi-Gaussian multiplier (NEXT-4): the factored application
against dense matrices built from def11, Thm thm2's closed-form limit for the averaging
factors (def2), and the Gaussian limit of Thm thm1 (moments and the Kolmogorov-Smirnov
distance shrinking with the number of factors, Fig LowRkTest1)."""
import numpy as np
import pytest
import scipy.stats

import synth
from oracle import lra


def _dense_factor(sign_i, perm_i, diag=1.0):
    n = len(sign_i)
    B = np.eye(n) * diag
    for c in range(n):
        B[(c + 1) % n, c] = sign_i[c]
    P = np.zeros((n, n))
    P[perm_i, np.arange(n)] = 1.0
    return B @ P


def test_qgauss_matches_dense_def11():
    mult = synth.multiplier_qgauss(3, 12, 3, 5)
    G = np.eye(12)
    for i in range(3):
        G = G @ _dense_factor(mult["qg_sign"][i], mult["qg_perm"][i])
    assert np.array_equal(lra.qgauss_omega(mult), G[:, mult["col"]])
    W = np.random.default_rng(4).standard_normal((7, 12))
    assert np.allclose(lra.sketch(W, mult), W @ G[:, mult["col"]], rtol=1e-13, atol=1e-13)


def test_averaging_factors_converge_to_uniform_thm2():
    """Thm thm2: products of A_t = (1/2)(I + cyclic shift) P_t converge to (1/n) ones."""
    n, T = 8, 400
    g = np.random.default_rng(5)
    perm = np.stack([g.permutation(n) for _ in range(T)])
    half = np.full((T, n), 0.5)
    Pi = lra.bidiag_product_columns(perm, half, half, np.arange(n))
    assert np.abs(Pi - 1.0 / n).max() < 1e-6
    assert np.allclose(Pi.sum(axis=0), 1.0)          # every factor is column-stochastic


def test_qgauss_entries_approach_gaussian_thm1():
    n = 256
    ks = {}
    for q in (2, 24):
        mult = synth.multiplier_qgauss(6, n, q, n)
        Om = lra.qgauss_omega(mult) / np.sqrt(2.0 ** q / n)
        x = Om.ravel()
        ks[q] = scipy.stats.kstest(x, "norm").statistic
        if q == 24:
            assert abs(x.mean()) < 0.02 and abs(x.var() - 1.0) < 0.05
    assert ks[2] > 0.3 and ks[24] < 0.02
