"""Pins of the NEXT-4 oracle pieces: Alg C.2 Expected(l) (reading C33), the
uniform-score Alg 9.1 and the Table tb_Lp Laplacian input
(P:4817-4826).  Every pin is a hand-evaluated value, a closed form or a probabilistic identity
of the algorithm — none retypes the oracle's own formula."""
import numpy as np
import pytest

import synth
from oracle import lra


# ------------------------------------------------------------------ Alg C.2 Expected(l)
def test_expected_hand_example():
    """p = (1/2, 1/4, 1/4), l = 2: pi = min(1, l p) = (1, 1/2, 1/2).  u = (.9, .3, .7):
    j = 0 kept (.9 < 1), j = 1 kept (.3 < .5), j = 2 not (.7 >= .5); the rescalings are
    1/min(1, sqrt(1)) = 1 and 1/sqrt(1/2) = sqrt 2."""
    idx, d = lra.sample_expected(np.array([0.5, 0.25, 0.25]), 2, np.array([0.9, 0.3, 0.7]))
    assert list(idx) == [0, 1]
    assert d[0] == 1.0 and d[1] == pytest.approx(np.sqrt(2.0), rel=1e-15)


def test_expected_boundary_u_equals_pi_not_kept():
    """Picked with probability pi_j: u uniform on [0, 1) is kept iff u < pi_j (so u = pi_j is
    not kept and pi_j = 1 keeps every u)."""
    p = np.array([0.125, 0.375, 0.5])
    idx, _ = lra.sample_expected(p, 2, np.array([0.25, 0.75, 0.999999]))
    assert list(idx) == [2]                             # pi = (.25, .75, 1): u = pi drops j = 0, 1
    idx, _ = lra.sample_expected(p, 2, np.array([0.2499, 0.7499, 0.0]))
    assert list(idx) == [0, 1, 2]


def test_expected_inclusion_frequencies_and_unbiased_rescaling():
    """Monte Carlo over 40000 draws of u: the inclusion frequency of j is pi_j = min(1, l p_j),
    the mean count is sum_j pi_j <= l, and the rescaled sampling is unbiased —
    E[1{j kept} d_j^2] = pi_j / min(1, l p_j) = 1 for every j (the property that makes
    S D D^T S^T an unbiased estimate of I, DMM08) — which fails if the min{1, .} is dropped
    (j with l p_j > 1) or d is not squared correctly."""
    g = np.random.default_rng(5)
    p = np.concatenate([[0.3, 0.2], g.random(30)])
    p[2:] *= 0.5 / p[2:].sum()
    l, R = 4, 40000
    pi = np.minimum(1.0, l * p)
    assert pi[0] == 1.0 and pi[1] < 1.0
    hits = np.zeros(len(p))
    w = np.zeros(len(p))
    cnt = 0
    for _ in range(R):
        idx, d = lra.sample_expected(p, l, g.random(len(p)))
        assert np.all(np.diff(idx) > 0)                  # ascending, no repeats
        hits[idx] += 1
        w[idx] += d ** 2
        cnt += len(idx)
    sd = np.sqrt(pi * (1 - pi) / R) + 1e-12
    assert np.all(np.abs(hits / R - pi) < 5 * sd + 1e-9)
    assert abs(cnt / R - pi.sum()) < 5 * np.sqrt(np.sum(pi * (1 - pi)) / R)
    assert pi.sum() <= l
    # E[1{kept} d^2] = 1: sd of the estimator is sqrt((1 - pi)/(pi R))
    assert np.all(np.abs(w / R - 1.0) < 5 * np.sqrt((1 - pi) / (pi * R)) + 1e-12)


def test_expected_all_kept_when_l_p_at_least_one():
    """l p_j >= 1 for all j (e.g. uniform p, l = n): every j is kept with d_j = 1 —
    Expected(n) on uniform scores is the identity sampling."""
    n = 17
    idx, d = lra.sample_expected(np.full(n, 1.0 / n), n, np.random.default_rng(1).random(n))
    assert list(idx) == list(range(n)) and np.all(d == 1.0)


# ------------------------------------------------------------------ uniform-score Alg 9.1
def test_uniform_exactly_picks_are_floor_u_n():
    """Uniform scores p_j = 1/n through Alg C.1: the inverse CDF of the uniform distribution on
    {0..n-1} is floor(u n); mid-cell uniforms (t + 1/2)/n pick t exactly, d = 1/sqrt(l/n)."""
    n, l = 640, 64
    t = np.random.default_rng(2).integers(0, n, l)
    idx, d = lra.sample_exactly(np.full(n, 1.0 / n), l, (t + 0.5) / n)
    assert list(idx) == list(t)
    assert np.allclose(d, np.sqrt(n / l), rtol=1e-14)


@pytest.mark.parametrize("sampler", ["exactly", "expected"])
def test_cur_uniform_exact_recovery_rank_r(sampler):
    """W of exact rank r (random Gaussian factors): any I, J with rank W[I,J] = r give
    W = CUR exactly (Thm scurhrd) — the uniform-score CUR has rho ~ 1e-14."""
    g = np.random.default_rng(7)
    m, n, r = 300, 260, 6
    W = g.standard_normal((m, r)) @ g.standard_normal((r, n))
    if sampler == "exactly":
        res = lra.cur_uniform(W, r, 24, 24, g.random(24), g.random(24))
    else:
        res = lra.cur_uniform(W, r, 24, 24, g.random(n), g.random(m), sampler="expected")
    assert len(res.I) >= r and len(res.J) >= r
    assert res.rho < 1e-12


def test_cur_uniform_expected_sizes_follow_l_over_n():
    """Expected(l) on uniform scores keeps j iff u_j < l/n: the sample sizes equal the numbers
    of uniforms below l/n and below k/m (counted directly)."""
    g = np.random.default_rng(8)
    m, n, r = 200, 180, 4
    W = g.standard_normal((m, r)) @ g.standard_normal((r, n))
    uc, ur = g.random(n), g.random(m)
    res = lra.cur_uniform(W, r, 30, 20, uc, ur, sampler="expected")
    assert len(res.J) == int(np.sum(uc < 20 / n)) and len(res.I) == int(np.sum(ur < 30 / m))


# ------------------------------------------------------------------ Table tb_Lp Laplacian
def _arc_integral_gl(i, j, n, nodes=48):
    """w_ij / psi by Gauss-Legendre quadrature of log|2 omega^i - e^{i theta}| over the arc
    [2 j pi / n, 2 (j + 1) pi / n] — direct numerical integration of P:4817-4826."""
    x, wt = np.polynomial.legendre.leggauss(nodes)
    a, b = 2 * np.pi * j / n, 2 * np.pi * (j + 1) / n
    th = 0.5 * (b - a) * x + 0.5 * (a + b)
    z = 2.0 * np.exp(2j * np.pi * i / n)
    return 0.5 * (b - a) * np.sum(wt * np.log(np.abs(z - np.exp(1j * th))))


def test_laplacian_entries_match_quadrature_and_norm_is_one():
    """Entries at random (i, j) equal psi x the Gauss-Legendre arc integral (no circulant or
    series assumption on that side) to 1e-13 relative; ||W||_2 = 1 by an SVD."""
    n = 256
    W = synth.laplacian_tb_lp(n)
    assert np.linalg.norm(W, 2) == pytest.approx(1.0, rel=1e-13)
    g = np.random.default_rng(3)
    ij = g.integers(0, n, (40, 2))
    q = np.array([_arc_integral_gl(i, j, n) for i, j in ij])
    w = np.array([W[i, j] for i, j in ij])
    psi = w[0] / q[0]
    assert np.allclose(w, psi * q, rtol=1e-13, atol=1e-16)


def test_laplacian_row_sums_mean_value_property():
    """The mean-value property of the harmonic function log|x - y| (|x| = 2 outside the unit
    circle): the integral over the whole circle is 2 pi log|x| = 2 pi log 2, for every row i.
    So every row sum of W is psi 2 pi log 2, the all-ones vector is the top singular vector
    (the row sum is the largest eigenvalue of the symmetric-spectrum circulant), and with
    ||W|| = 1 each row sums to exactly 1."""
    W = synth.laplacian_tb_lp(512)
    assert np.allclose(W.sum(axis=1), 1.0, rtol=1e-13)


def test_laplacian_spectrum_closed_form():
    """The singular values of the continuous operator (log|2 e^{ia} - e^{ib}| =
    log 2 - sum_k 2^-k cos(k (a - b)) / k) relative to the top one: sigma_f / sigma_0 =
    2^-f / (2 f log 2) for f >= 1, each twice (cos and sin modes); the arc discretization
    multiplies mode f by sinc(pi f / n) (1 - 4e-5 at n = 256, f = 2)."""
    n = 256
    sv = np.linalg.svd(synth.laplacian_tb_lp(n), compute_uv=False)
    assert sv[0] == pytest.approx(1.0, rel=1e-13)
    for f in (1, 2, 3, 4):
        want = 2.0 ** -f / (2 * f * np.log(2.0)) * np.sinc(f / n)
        assert sv[2 * f - 1] == pytest.approx(want, rel=1e-9)
        assert sv[2 * f] == pytest.approx(want, rel=1e-9)
