"""Pins of the leverage-score subalgorithm (NEXT-4; DMM08 as used by Alg 9.1 and §ststc-alvrg):
scores against an SVD-free projector (QR of the row space), their invariance, the
inverse-CDF sampling of Alg C.1 on a hand example and in frequency, and exact recovery of a
rank-r matrix by the leverage-score C-A."""
import numpy as np
import pytest

import synth
from oracle import lra


def test_leverage_scores_equal_projector_diagonal():
    g = np.random.default_rng(51)
    k, n, r = 6, 40, 4
    B = g.standard_normal((k, r)) @ g.standard_normal((r, n))
    p = lra.leverage_scores(B, r)
    Q, _ = np.linalg.qr(B.T)                     # n x k; the first r columns span the row space
    Qr = Q[:, :r]
    assert np.allclose(p, np.sum(Qr * Qr, axis=1) / r, rtol=1e-10, atol=1e-14)
    assert p.sum() == pytest.approx(1.0, rel=1e-13)
    M = g.standard_normal((k, k))                # invertible row mixing keeps the row space
    assert np.allclose(lra.leverage_scores(M @ B, r), p, rtol=1e-8, atol=1e-13)


def test_sample_exactly_inverse_cdf_and_frequencies():
    p = np.array([0.1, 0.2, 0.3, 0.4])
    idx, d = lra.sample_exactly(p, 6, np.array([0.05, 0.1, 0.29, 0.31, 0.99, 0.0]))
    assert list(idx) == [0, 1, 1, 2, 3, 0]
    assert np.allclose(d, 1 / np.sqrt(6 * p[idx]))
    u = np.random.default_rng(52).random(200000)
    idx, _ = lra.sample_exactly(p, len(u), u)
    freq = np.bincount(idx, minlength=4) / len(u)
    assert np.abs(freq - p).max() < 0.005


def test_cur_leverage_exact_recovery():
    W = synth.factor_gaussian(9, 300, 260, 5, 0.0)
    I0 = synth.random_rows(9, 300, 15)
    res = lra.cur_leverage(W, 5, 15, 15, 2, I0, synth.leverage_uniforms(9, 2, 15, 15))
    assert res.rho < 1e-10
