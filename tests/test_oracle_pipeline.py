"""Pins of the oracle's nucleus, residual and whole path (configs 1–3 recipes)."""
import os

import numpy as np
import pytest

import synth
from oracle import lra

GOLD = os.path.join(os.path.dirname(__file__), "golden")


# ------------------------------------------------------------------ nucleus (Alg 3.1)
def test_nucleus_spec_examples():
    """SPEC canonical_nucleus examples: [[5]] → 0.2; ones(2,2), r=1 → ones/4;
    diag(3, 1e-9), r = 1 → diag(1/3, 0)."""
    U, *_ = lra.canonical_nucleus(np.array([[5.0]]), 1)
    assert U[0, 0] == pytest.approx(0.2, rel=1e-15)
    U, *_ = lra.canonical_nucleus(np.ones((2, 2)), 1)
    assert np.allclose(U, np.ones((2, 2)) / 4, atol=1e-15)
    U, *_ = lra.canonical_nucleus(np.diag([3.0, 1e-9]), 1)
    assert np.allclose(U, np.diag([1 / 3, 0.0]), atol=1e-15)


def test_nucleus_is_inverse_when_k_eq_l_eq_r():
    """Remark reklr_kl: k = l = r ⇒ U = W_{r,r}⁻¹ (eq. eqnucinv)."""
    G = np.random.default_rng(1).standard_normal((6, 6))
    U, *_ = lra.canonical_nucleus(G, 6)
    assert np.allclose(U, np.linalg.inv(G), rtol=1e-12, atol=1e-12)


def test_nucleus_penrose_identities():
    """U = W_{k,l,r}⁺ satisfies the four Penrose identities with the truncation G_r."""
    g = np.random.default_rng(2)
    G = g.standard_normal((7, 5)) @ np.diag([5, 3, 1, 1e-3, 1e-4]) @ g.standard_normal((5, 7))
    U, Sr, sr, Tr = lra.canonical_nucleus(G, 3)
    s, sv, th = np.linalg.svd(G)
    Gr = (s[:, :3] * sv[:3]) @ th[:3]
    assert np.allclose(Gr @ U @ Gr, Gr, atol=1e-12)
    assert np.allclose(U @ Gr @ U, U, atol=1e-10)
    assert np.allclose((Gr @ U).T, Gr @ U, atol=1e-12)
    assert np.allclose((U @ Gr).T, U @ Gr, atol=1e-12)


# ------------------------------------------------------------------ residual
def test_residual_brute_force_loops():
    """num², den² against pure-Python triple loops on a tiny instance."""
    g = np.random.default_rng(4)
    W = g.standard_normal((7, 9)).astype(np.float32)
    A = g.standard_normal((7, 3))
    B = g.standard_normal((3, 9))
    num2 = den2 = 0.0
    for i in range(7):
        for j in range(9):
            s = 0.0
            for t in range(3):
                s += A[i, t] * B[t, j]
            num2 += (float(W[i, j]) - s) ** 2
            den2 += float(W[i, j]) ** 2
    n2, d2 = lra.cur_residual(W, A, B, row_block=3)
    assert n2 == pytest.approx(num2, rel=1e-13) and d2 == pytest.approx(den2, rel=1e-14)


# ------------------------------------------------------------------ whole path
@pytest.mark.parametrize("seed", range(10))
def test_exact_recovery_rank_r(seed):
    """Thm thcandec: rank-r W with a nonsingular generator ⇒ W = CUR."""
    W = synth.factor_gaussian(seed, 120, 96, 5, 0.0)
    M = synth.multiplier_abridged(seed, 96, 3, 5, "arht")
    res = lra.cur_pipeline(W, M, 5, 5, 5, 2)
    assert res.rho <= 1e-12


def test_recovery_canonical_truncation_k_gt_r():
    """k = l = 6 > r = 4 on rank-4 + 1e-12 noise: the canonical truncation (Alg 3.1)
    recovers W to the noise level (Cor. cowc1), above the Eckart–Young floor."""
    W = synth.factor_gaussian(3, 150, 128, 4, 1e-24)
    M = synth.multiplier_abridged(3, 128, 2, 6, "arht")
    res = lra.cur_pipeline(W, M, 4, 6, 6, 2)
    sv = np.linalg.svd(W, compute_uv=False)
    floor = np.sqrt(np.sum(sv[4:] ** 2) / np.sum(sv ** 2))
    assert floor * (1 - 1e-6) <= res.rho <= 1e3 * floor


def test_config1_baseline_expectations():
    """BASELINE.json config 1: ρ ≤ 1e-9 and maxvol dominance ≤ 1 + 1e-12."""
    W = synth.config1(0)
    M = synth.multiplier_abridged(0, 256, 3, 8, "arht")
    res = lra.cur_pipeline(W, M, 8, 8, 8, 2)
    assert res.rho <= 1e-9
    assert res.ca.cert_rows <= 1 + 1e-12 and res.ca.cert_cols <= 1 + 1e-12
    # Eckart–Young floor (eq. eqnsgmrfr): ρ ≥ sqrt(Σ_{i>r} σ_i²)/‖W‖_F
    sv = np.linalg.svd(W, compute_uv=False)
    assert res.rho >= np.sqrt(np.sum(sv[8:] ** 2) / np.sum(sv ** 2)) * (1 - 1e-9)


@pytest.mark.parametrize("kind", ["arht", "arft", "gaussian"])
def test_config2_small_floor_and_dominance(kind):
    """Config-2 recipe at n = 512: ρ above the Eckart–Young floor and within a modest
    factor of it; every maxvol ends dominant."""
    n = 512
    W = synth.config2(0, n=n, p=160)
    M = (synth.multiplier_gaussian(0, n, 48) if kind == "gaussian"
         else synth.multiplier_abridged(0, n, 4, 48, kind))
    res = lra.cur_pipeline(W, M, 32, 48, 48, 3)
    sv = np.linalg.svd(np.asarray(W, np.float64), compute_uv=False)
    floor = np.sqrt(np.sum(sv[32:] ** 2) / np.sum(sv ** 2))
    assert floor * (1 - 1e-9) <= res.rho <= 20 * floor
    assert res.ca.cert_rows <= 1 + 1e-12 and res.ca.cert_cols <= 1 + 1e-12


def test_config3_block_floor():
    s, t = synth.cauchy_params(0, 2)
    for b in range(2):
        W = synth.cauchy_block(s[b], t[b])
        M = synth.multiplier_sparse_batch(0, 2, 512, 20)
        Mb = dict(M, sp_row=M["sp_row"][b], sp_sign=M["sp_sign"][b])
        res = lra.cur_pipeline(W, Mb, 16, 20, 20, 2)
        sv = np.linalg.svd(np.asarray(W, np.float64), compute_uv=False)
        floor = np.sqrt(np.sum(sv[16:] ** 2) / np.sum(sv ** 2))
        assert floor * (1 - 1e-6) <= res.rho <= 1e-6


def test_delta_matrices_defeat_superfast_ca():
    """Example exdlt: a ±δ matrix whose nonzero lies outside the rows and
    columns the algorithm reads gives a singular generator — reported, not hidden."""
    pats = np.loadtxt(os.path.join(GOLD, "delta_matrices_2x2.txt"), comments="#")
    assert pats.shape == (8, 4) and np.all(np.abs(pats).sum(axis=1) == 1)
    W = np.zeros((8, 8))
    W[6, 5] = 1.0
    with pytest.raises(lra.Singular):
        lra.cross_approx(lra.DenseOperand(W), 1, 1, 2, I0=[0])


def test_sampled_residual_unbiased():
    """num²_est = (mn/Q)Σd² over uniform samples tracks the full num²."""
    W = synth.factor_gaussian(1, 300, 200, 4, 1e-4)
    M = synth.multiplier_abridged(1, 200, 3, 4, "arht")
    res = lra.cur_pipeline(W, M, 4, 4, 4, 2)
    ii, jj = synth.sample_pairs(9, 300, 200, 200000)
    est = lra.sampled_residual(lra.DenseOperand(W), res.A, res.B, ii, jj)
    assert est == pytest.approx(res.num2, rel=0.02)


def test_factored_operand_matches_dense():
    """Config-4 entry oracle on a downsized instance equals the dense materialization;
    the factored ‖W‖_F² identity equals the dense one."""
    c4 = synth.config4(0, m=384, n=320, p=5, dens_ab=0.3, dens_e=0.01)
    op = lra.FactoredOperand(c4["A"], c4["B"], c4["row_ptr"], c4["col"], c4["val"])
    Wd = c4["A"] @ c4["B"]
    for i in range(op.m):
        lo, hi = c4["row_ptr"][i], c4["row_ptr"][i + 1]
        Wd[i, c4["col"][lo:hi]] += c4["val"][lo:hi]
    I = np.array([3, 100, 7])
    J = np.array([0, 319, 31, 5])
    assert np.allclose(op.rows(I), Wd[I], atol=1e-14)
    assert np.allclose(op.cols(J), Wd[:, J], atol=1e-14)
    assert lra.factored_den2(op) == pytest.approx(float(np.sum(Wd * Wd)), rel=1e-12)


def test_factored_entries_vectorized():
    """The vectorized entry oracle equals the dense materialization at sampled pairs."""
    c4 = synth.config4(1, m=300, n=250, p=4, dens_ab=0.3, dens_e=0.02)
    op = lra.FactoredOperand(c4["A"], c4["B"], c4["row_ptr"], c4["col"], c4["val"])
    Wd = c4["A"] @ c4["B"]
    for i in range(op.m):
        lo, hi = c4["row_ptr"][i], c4["row_ptr"][i + 1]
        Wd[i, c4["col"][lo:hi]] += c4["val"][lo:hi]
    ii, jj = synth.sample_pairs(3, 300, 250, 5000)
    assert np.allclose(op.entries(ii, jj), Wd[ii, jj], atol=1e-14)


# ------------------------------------------------------------ NEXT-1: Alg 10.1 full pre-processing
def test_preprocess_full_equals_dense_hadamard_product():
    """d = log2 n: W' = W·D·H_n·P with the Sylvester Hadamard matrix from scipy (a library
    routine, not the oracle's recursion); integer-valued W so every sum is exact and the fp32
    rounding is the identity."""
    import scipy.linalg
    g = np.random.default_rng(3)
    n, d = 64, 6
    W = g.integers(-50, 50, size=(37, n)).astype(np.float32)
    mult = synth.multiplier_abridged(2, n, d, n, "arht")
    H = scipy.linalg.hadamard(n).astype(np.float64)
    M = (mult["dsign"].astype(np.float64)[:, None] * H)[:, mult["col"]]
    ref = (W.astype(np.float64) @ M).astype(np.float32)
    assert np.array_equal(lra.preprocess_full(W, mult), ref)


def test_preprocess_full_norm_and_abridged_blocks():
    """d < log2 n (n = 2^d·s, s not a power of two): ||W'||_F^2 = 2^d ||W||_F^2 (M M^T = 2^d I)
    and W' equals the dense product with the closed-form H_{n,d} = H_{2^d} ⊗ I_s."""
    from oracle.transforms import hadamard_recursive
    g = np.random.default_rng(4)
    n, d = 1000, 3
    W = g.standard_normal((23, n))
    mult = synth.multiplier_abridged(5, n, d, n, "arht")
    Wp = lra.preprocess_full(W, mult)
    assert np.sum(Wp * Wp) == pytest.approx(8 * np.sum(W * W), rel=1e-13)
    M = (mult["dsign"].astype(np.float64)[:, None] * hadamard_recursive(n, d))[:, mult["col"]]
    assert np.allclose(Wp, W @ M, rtol=0, atol=1e-12 * np.abs(W).max())


def test_alg101_backmap_residual_identity():
    """Alg 10.1 with R = R_H H^+ = W[I,:]: the relative residual of the CUR LRA of W equals the
    one computed on W' (M M^T = 2^d I); fp64 data so W' is exact."""
    W = synth.factor_gaussian(8, 300, 256, 5, 1e-12)
    mult = synth.multiplier_abridged(8, 256, 3, 256, "arht")
    I0 = synth.random_rows(8, 300, 5)
    res, rho_w = lra.cur_preprocessed(W, mult, 5, 5, 3, I0)
    assert rho_w == pytest.approx(res.rho, rel=1e-9)
    assert res.rho < 1e-5


# ------------------------------------------------------------ NEXT-2: superfast a-posteriori estimate
def test_error_sample_full_grid_equals_residual():
    """rows = all, cols = all: the sampled sum of squares is the full a-posteriori numerator."""
    W = synth.factor_gaussian(11, 120, 90, 4, 1e-6)
    mult = synth.multiplier_abridged(11, 90, 1, 4, "arht")
    res = lra.cur_pipeline(W, mult, 4, 4, 4, 2)
    mu, var, ss, sw = lra.error_sample(lra.DenseOperand(W), res.A, res.B, np.arange(120), np.arange(90))
    assert ss == pytest.approx(res.num2, rel=1e-12)
    assert sw == pytest.approx(res.den2, rel=1e-13)
    E = (W - res.A @ res.B).ravel()
    assert mu == pytest.approx(E.mean(), rel=1e-9, abs=1e-18)          # numpy's own mean / var
    assert var == pytest.approx(E.var(), rel=1e-9)


def test_error_sample_recovers_known_noise_variance():
    """W = A·B + E with E i.i.d. N(0, s²) and the exact factors: the q×s sample estimates s²
    within its statistical error (sqrt(2/K) relative) and the chi-square bound covers it."""
    g = np.random.default_rng(5)
    m, n, r, sd = 2000, 1500, 6, 1e-3
    A = g.standard_normal((m, r))
    B = g.standard_normal((r, n))
    W = A @ B + sd * g.standard_normal((m, n))
    rows = g.choice(m, 100, replace=False)
    cols = g.choice(n, 100, replace=False)
    mu, var, _, _ = lra.error_sample(lra.DenseOperand(W), A, B, rows, cols)
    assert abs(var / sd ** 2 - 1) < 5 * np.sqrt(2 / 1e4)
    assert abs(mu) < 5 * sd / 100
    assert lra.variance_upper_bound(var, 10000, 0.05) >= sd ** 2


def test_variance_bound_coverage():
    """Coverage of the one-sided 95 % chi-square bound over 400 independent samples of K = 200
    standard normals (binomial 95 % ± 4.4 % at 4 sigma)."""
    g = np.random.default_rng(6)
    hits = 0
    for _ in range(400):
        x = g.standard_normal(200)
        v = float(np.sum((x - x.mean()) ** 2)) / 200
        hits += lra.variance_upper_bound(v, 200, 0.05) >= 1.0
    assert abs(hits / 400 - 0.95) < 0.045


def test_certificate_holds_and_vanishes():
    """Cor cowc1 (ii): with Δ = σ̃_{r+1} (the Frobenius tail of W's spectrum, eq. eqnsgmrfr)
    the certificate bounds ||W − CUR||_F on random perturbed low-rank inputs; for an exactly
    rank-r W (Δ = 0) it is 0 and W = CUR (thm thcandec)."""
    for seed in range(6):
        W = synth.factor_gaussian(40 + seed, 200, 150, 5, 1e-8 * (seed + 1))
        mult = synth.multiplier_abridged(seed, 150, 1, 7, "arht")
        res = lra.cur_pipeline(W, mult, 5, 7, 7, 2)
        sv = np.linalg.svd(W, compute_uv=False)
        delta = float(np.sqrt(np.sum(sv[5:] ** 2)))
        op = lra.DenseOperand(W)
        bound, nc, nr, nu = lra.cur_certificate(op.cols(res.J), op.rows(res.I), res.U, 5, delta)
        assert np.sqrt(res.num2) <= bound
        assert nc == pytest.approx(np.linalg.norm(W[:, res.J])) and nu == pytest.approx(np.linalg.norm(res.U))
    b0, *_ = lra.cur_certificate(np.ones((4, 2)), np.ones((2, 4)), np.eye(2), 2, 0.0)
    assert b0 == 0.0


def test_certificate_hand_evaluated_eqnrm11():
    """Two-sided pin of eq. (eqnrm11), on hand-evaluated cases (Frobenius norm,
    mu = 1, (1 - theta) xi = sqrt(kl), theta = ||U|| eta Delta with ||U|| <= ||U||_F, C27).

    Case 1: C = ones(4,2), R = ones(2,4), U = I_2, k = l = r = 2 (eta = 1), Delta = 0.01:
      |C| = |R| = sqrt 8, |U| = sqrt 2, theta = 0.01 sqrt 2 = 0.0141421356...,
      xi = 2 / (1 - theta) = 2.02869000924931...,
      bound = 0.01 ((2 sqrt 8 + 0.01 + 8 sqrt 2) xi sqrt 2 + 1) = 0.497172502312...
    Case 2: C = ones(4,3), R = ones(3,4), U = I_3 / 2, k = l = 3, r = 2 (eta = 2), Delta = 0.05:
      |C| = |R| = sqrt 12, |U| = sqrt 3 / 2, theta = 2 (0.05) sqrt 3 / 2 = 0.0866025403...,
      xi = 3 / (1 - theta), bound = 0.05 ((2 sqrt 12 + 0.05 + 2 (12) sqrt 3 / 2) xi sqrt 3 / 2 + 1)
           = 3.99844013691766...
    Case 3: theta >= 1 (|U| eta Delta = 2 sqrt 2 * 0.5 > 1): no certificate (inf)."""
    b1, nc, nr, nu = lra.cur_certificate(np.ones((4, 2)), np.ones((2, 4)), np.eye(2), 2, 0.01)
    assert b1 == pytest.approx(0.49717250231232796, rel=1e-13, abs=0)
    assert (nc, nr, nu) == pytest.approx((8 ** 0.5, 8 ** 0.5, 2 ** 0.5), rel=1e-15)
    b2, *_ = lra.cur_certificate(np.ones((4, 3)), np.ones((3, 4)), 0.5 * np.eye(3), 2, 0.05)
    assert b2 == pytest.approx(3.9984401369176634, rel=1e-13, abs=0)
    b3, *_ = lra.cur_certificate(np.ones((4, 2)), np.ones((2, 4)), 2 * np.eye(2), 2, 0.5)
    assert b3 == float("inf")


def test_progressive_depth_stops_at_first_passing_depth():
    """d = 1 already passes on a generic perturbed low-rank input; an impossible
    tolerance runs to dmax; the estimate is the sampled ratio."""
    W = synth.factor_gaussian(3, 256, 256, 6, 1e-10)
    g = np.random.default_rng(0)
    rows, cols = g.choice(256, 40, replace=False), g.choice(256, 40, replace=False)
    d, res, est = lra.cur_progressive(W, 6, 8, 2, 1e-3, 1, rows, cols, dmax=4)
    assert d == 1 and est <= 1e-3
    d2, _, est2 = lra.cur_progressive(W, 6, 8, 2, 1e-30, 1, rows, cols, dmax=3)
    assert d2 == 3 and est2 > 1e-30
