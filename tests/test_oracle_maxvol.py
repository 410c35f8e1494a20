"""Pins of the oracle's maxvol (Alg D.2 stage 1 + Alg D.1) and C-A loops.

Brute force over all q-row subsets, LAPACK's partial pivoting, the dominance and volume
statements of the paper, and hand traces — not the oracle's own formulas."""
import itertools

import numpy as np
import pytest
import scipy.linalg

import synth
from oracle import lra


def _absdet(B, S):
    return abs(np.linalg.det(B[list(S), :]))


def test_q1_is_argmax_with_smallest_index_tie():
    """q = 1: the 1×1 volume is |entry| (SPEC lup_ca example); ties → smallest index."""
    B = np.array([[0.5], [-3.0], [2.0], [3.0], [-1.0]])
    r = lra.maxvol(B)
    assert list(r.S) == [1] and r.swaps == 0


def test_hand_trace_swap():
    """SPEC dominant_submatrix example A = [[1, 2]] (transposed): start {0} → one swap
    → {1}, certificate 1/2 (Alg D.1 by hand)."""
    B = np.array([[1.0], [2.0]])
    r = lra.maxvol(B, start=[0])
    assert list(r.S) == [1] and r.swaps == 1 and r.cert == pytest.approx(0.5)


@pytest.mark.parametrize("seed", range(6))
def test_lup_pivots_match_lapack_getrf(seed):
    """Cold start = LU with partial pivoting; LAPACK dgetrf (max |pivot|, first on ties)
    selects the same rows when there are no near-ties."""
    g = np.random.default_rng(seed)
    B = g.standard_normal((40, 7))
    S = lra.lup_pivots(B)
    lu, piv = scipy.linalg.lu_factor(B)
    perm = np.arange(40)
    for i, p in enumerate(piv):
        perm[[i, p]] = perm[[p, i]]
    assert list(S) == list(perm[:7])


@pytest.mark.parametrize("seed", range(20))
@pytest.mark.parametrize("N,q", [(8, 2), (10, 3), (12, 3)])
def test_maxvol_vs_brute_force(seed, N, q):
    """Exit state is dominant (|C'| ≤ 1+tol, Alg D.1 stage 1), locally maximal (no single
    row swap raises |det| by more than 1+tol, Def. defmxv), and globally within q^{q/2}
    of the maximum volume (Thm thlclglb with h = 1)."""
    g = np.random.default_rng(1000 + seed)
    B = g.standard_normal((N, q))
    r = lra.maxvol(B)
    C = B @ np.linalg.inv(B[r.S, :])
    mask = np.ones(N, bool)
    mask[r.S] = False
    assert np.abs(C[mask]).max() <= 1 + 1e-12
    v = _absdet(B, r.S)
    vmax = max(_absdet(B, S) for S in itertools.combinations(range(N), q))
    assert v >= vmax / q ** (q / 2) * (1 - 1e-12)
    for j in range(q):
        for i in range(N):
            if i in r.S:
                continue
            S2 = list(r.S)
            S2[j] = i
            assert _absdet(B, S2) <= v * (1 + 1e-9)


@pytest.mark.parametrize("seed", range(5))
def test_each_swap_multiplies_volume_by_c(seed):
    """Each swap multiplies |det B[S,:]| by |c_{i*j*}| > 1: log-volume
    strictly increases."""
    g = np.random.default_rng(seed)
    B = g.standard_normal((200, 10))
    r = lra.maxvol(B, start=list(range(10)))
    assert r.swaps > 0
    assert all(b > a for a, b in zip(r.logdet, r.logdet[1:]))


def test_dominant_start_is_fixed_point():
    """A = (I_r | small) → the identity block is kept with 0 swaps (SPEC example)."""
    g = np.random.default_rng(0)
    B = np.vstack([np.eye(4), 0.1 * g.standard_normal((30, 4))])
    r = lra.maxvol(B)
    assert sorted(r.S) == [0, 1, 2, 3] and r.swaps == 0


def test_singular_block_raises():
    B = np.zeros((10, 3))
    B[:, 0] = 1.0
    with pytest.raises(lra.Singular):
        lra.maxvol(B)


def test_swap_cap_reported_not_error():
    g = np.random.default_rng(3)
    B = g.standard_normal((300, 8))
    r = lra.maxvol(B, start=list(range(8)), cap=1)
    assert r.swaps == 1 and r.cap_hit


# ------------------------------------------------------------------ C-A loops
def test_ca_two_step_volume_bound_brute_force():
    """Thm th111 with thlclglb: after a C-A loop whose steps end dominant,
    W[I,J] is (r^{r/2})²-maximal over ALL k×l submatrices (5×5, r = 2, brute force)."""
    for seed in range(10):
        W = np.random.default_rng(50 + seed).standard_normal((5, 5))
        op = lra.DenseOperand(W)
        ca = lra.cross_approx(op, 2, 2, 3, I0=[0, 1])
        v = abs(np.linalg.det(op.block(ca.I, ca.J)))
        vmax = max(abs(np.linalg.det(W[np.ix_(I, J)]))
                   for I in itertools.combinations(range(5), 2) for J in itertools.combinations(range(5), 2))
        assert v >= vmax / (2.0 ** 1) ** 2 * (1 - 1e-12)


@pytest.mark.parametrize("seed", range(4))
def test_ca_log_volume_monotone_and_fixed_point(seed):
    """Reading C10: warm starts make log|det W[I,J]| non-decreasing across C-A steps, and
    a converged loop is a fixed point (0 swaps on the next loop)."""
    W = synth.factor_gaussian(seed, 300, 200, 6, 1e-6)
    op = lra.DenseOperand(W)
    I0 = synth.random_rows(seed, 300, 6)
    ca = lra.cross_approx(op, 6, 6, 6, I0=I0)
    ld = ca.logdet_steps
    assert all(b >= a - 1e-9 for a, b in zip(ld, ld[1:]))
    assert ca.steps[-1][1] == 0 and ca.steps[-2][1] == 0
    ca2 = lra.cross_approx(op, 6, 6, 2, I0=ca.I, J0=ca.J)
    assert list(ca2.I) == list(ca.I) and list(ca2.J) == list(ca.J)
    assert all(sw == 0 for _, sw in ca2.steps)


# ------------------------------------------------------------ NEXT-3: greedy expansion (Alg D.4)
def test_expand_columns_volume_identity_and_brute_force():
    """Each appended column multiplies v2(C)^2 = det(C C^T) by exactly 1 + score (eq. eqbun),
    and is the argmax of det over all candidates (brute force)."""
    g = np.random.default_rng(12)
    R = g.standard_normal((4, 30))
    J0 = [3, 7, 11, 20]
    J, scores = lra.expand_columns(R, J0, 8)
    assert list(J[:4]) == J0 and len(set(J.tolist())) == 8
    for step in range(4):
        cur = list(J[:4 + step])
        C = R[:, cur]
        d0 = np.linalg.det(C @ C.T)
        dets = np.full(30, -np.inf)
        for j in range(30):
            if j not in cur:
                Cj = R[:, cur + [j]]
                dets[j] = np.linalg.det(Cj @ Cj.T)
        assert int(np.argmax(dets)) == J[4 + step]
        assert dets[J[4 + step]] / d0 == pytest.approx(1 + scores[step], rel=1e-10)


def test_rectangular_generator_exact_recovery_and_improvement():
    """k x l generators (l > k) still reproduce a rank-r W exactly (thm thcandec) and the
    expansion never lowers v2 of the generator."""
    W = synth.factor_gaussian(6, 200, 180, 5, 0.0)
    mult = synth.multiplier_abridged(6, 180, 2, 5, "arht")
    res = lra.cur_rectangular(W, mult, 5, 5, 9, 2)
    assert len(res.J) == 9 and res.rho < 1e-12
    G5 = W[np.ix_(res.I, res.J[:5])]
    G9 = W[np.ix_(res.I, res.J)]
    assert np.linalg.det(G9 @ G9.T) >= np.linalg.det(G5 @ G5.T) * (1 - 1e-12)


# ------------------------------------------------------------ NEXT-3: QRP (Alg D.3) and Alg 7.1
def test_qrp_pivots_are_greedy_volume_expansions():
    """Alg D.3: every pivot maximizes the distance of the appended column to the span of the
    previous pivots (= the greedy expansion of Def defgrd, since v2(C|b) = v2(C)·dist(b, C)),
    checked by least squares over all candidates; the reflected matrix keeps every column's
    norm and the Gram matrix (orthogonal transform), is upper triangular on the pivots, and
    its diagonal magnitudes are non-increasing."""
    g = np.random.default_rng(21)
    R = g.standard_normal((6, 17))
    piv, X = lra.qrp_columns(R, 6)
    assert len(set(piv.tolist())) == 6
    for step in range(6):
        prev = list(piv[:step])
        dist = np.full(17, -1.0)
        for j in range(17):
            if j in prev:
                continue
            if prev:
                coef = np.linalg.lstsq(R[:, prev], R[:, j], rcond=None)[0]
                dist[j] = np.linalg.norm(R[:, j] - R[:, prev] @ coef)
            else:
                dist[j] = np.linalg.norm(R[:, j])
        assert int(np.argmax(dist)) == piv[step]
        assert abs(X[step, piv[step]]) == pytest.approx(dist[piv[step]], rel=1e-12)
    assert np.allclose(np.linalg.norm(X, axis=0), np.linalg.norm(R, axis=0), rtol=1e-13)
    assert np.allclose(X.T @ X, R.T @ R, atol=1e-12 * np.abs(R.T @ R).max())
    T = X[:, piv]
    assert np.all(np.tril(T, -1) == 0.0)
    d = np.abs(np.diag(T))
    assert np.all(d[:-1] >= d[1:])


def test_qrp_rank_deficient_raises():
    g = np.random.default_rng(22)
    R = g.standard_normal((5, 3)) @ g.standard_normal((3, 12))
    lra.qrp_columns(R, 3)
    R2 = np.zeros((4, 6))
    R2[0, 2] = 1.0
    with pytest.raises(lra.Singular):
        lra.qrp_columns(R2, 2)


def test_projective_columns_volume_identity_and_brute_force():
    """Alg 7.1 on a rank-r matrix: the r-projective volume of W[:,J] (product of its r largest
    singular values) equals v2(R'[:,J]) (Lemma leprwnmp with the unitary Q of the QRP), and for
    l = r the chosen set is within the factor r^(r/2) of the best r-subset (Thm thlclglb
    through the maxvol black box), by brute force over all subsets."""
    g = np.random.default_rng(23)
    k, n, r = 5, 11, 3
    W = g.standard_normal((k, r)) @ g.standard_normal((r, n))
    for l in (3, 5):
        J, piv, Rp = lra.projective_columns(W, r, l)
        assert len(set(J.tolist())) == l
        sv = np.linalg.svd(W[:, J], compute_uv=False)
        vol_r = float(np.prod(sv[:r]))
        vol_Rp = float(np.sqrt(np.linalg.det(Rp[:, J] @ Rp[:, J].T)))
        assert vol_r == pytest.approx(vol_Rp, rel=1e-9)
    J, _, _ = lra.projective_columns(W, r, r)
    best = max(float(np.prod(np.linalg.svd(W[:, list(c)], compute_uv=False)[:r]))
               for c in itertools.combinations(range(n), r))
    got = float(np.prod(np.linalg.svd(W[:, J], compute_uv=False)[:r]))
    assert got >= best / r ** (r / 2) * (1 - 1e-12)


def test_projective_generator_exact_recovery():
    """k×l generators of maximal r-projective volume reproduce a rank-r W up to its noise
    (thm thcandec with the canonical nucleus) — Alg 7.1 after the square C-A (k > r needs the
    noise: an exactly rank-r W has no nonsingular k×k generator)."""
    W = synth.factor_gaussian(7, 160, 150, 4, 1e-20)
    mult = synth.multiplier_abridged(7, 150, 1, 6, "arht")
    res = lra.cur_projective(W, mult, 4, 6, 8, 2)
    assert len(res.J) == 8 and len(set(res.J.tolist())) == 8
    assert res.rho < 1e-8


def test_contract_columns_brute_force_and_identity():
    """Greedy contraction: the removed column maximizes the remaining det(C C^T) over all
    choices (brute force), and det drops by exactly 1 - leverage (eq. eqbtr)."""
    g = np.random.default_rng(24)
    R = g.standard_normal((4, 25))
    J0 = [1, 4, 6, 9, 13, 17, 21, 24]
    J = list(J0)
    for target in range(7, 3, -1):
        C = R[:, J]
        d0 = np.linalg.det(C @ C.T)
        dets = []
        for t in range(len(J)):
            Ct = R[:, J[:t] + J[t + 1:]]
            dets.append(np.linalg.det(Ct @ Ct.T))
        Jn = list(lra.contract_columns(R, J, target))
        removed = [t for t in range(len(J)) if J[t] not in Jn]
        assert len(removed) == 1 and removed[0] == int(np.argmax(dets))
        lev = R[:, J[removed[0]]] @ np.linalg.solve(C @ C.T, R[:, J[removed[0]]])
        assert dets[removed[0]] / d0 == pytest.approx(1 - lev, rel=1e-9)
        assert Jn == [j for j in J if j != J[removed[0]]]      # slot order kept
        J = Jn


def test_refine_columns_monotone_and_fixed_point():
    """Expand-contract cycles (p = 1): the volume never decreases, and at exit the greedy
    expansion's column is the greedy contraction's choice (fixed point), checked by brute
    force over all single additions and removals."""
    g = np.random.default_rng(25)
    R = g.standard_normal((5, 40))
    J0 = np.array([0, 1, 2, 3, 4, 5, 6], dtype=np.int64)
    vol = lambda J: np.linalg.det(R[:, J] @ R[:, J].T)
    J, done = lra.refine_columns(R, J0, 50)
    assert done >= 1 and vol(J) >= vol(J0) * (1 - 1e-12)
    cand = [j for j in range(40) if j not in J]
    jstar = max(cand, key=lambda j: vol(list(J) + [j]))
    Jx = list(J) + [jstar]
    best_removal = max(range(len(Jx)), key=lambda t: vol(Jx[:t] + Jx[t + 1:]))
    assert Jx[best_removal] == jstar


# ------------------------------------------- stats: top-2 pivot margins, final log-volume
def test_pivot_margins_hand_examples():
    """Top-2 margin (M − M₂)/M of each decision (reading C35), hand-evaluated:
    LUP on (1, 1/2, 1/4)ᵀ: one step, M = 1, M₂ = 1/2 -> 1/2;  an exact tie (1, 1, .2)ᵀ -> 0;
    a tie inside the slack window (1, 1 − 1e-13, .2)ᵀ: row 0 chosen, margin 1e-13;
    maxvol of (4, 2, 1)ᵀ from S = [2]: C = (4, 2, 1), swap to row 0 with margin (4 − 2)/4,
    then C = (1, 1/2, 1/4) is dominant — one margin, 1/2."""
    r = lra.maxvol(np.array([[1.0], [0.5], [0.25]]))
    assert r.margins == [0.5]
    r = lra.maxvol(np.array([[1.0], [1.0], [0.2]]))
    assert list(r.S) == [0] and r.margins == [0.0]
    r = lra.maxvol(np.array([[1.0], [1.0 - 1e-13], [0.2]]))
    assert list(r.S) == [0] and r.margins[0] == pytest.approx(1e-13, rel=1e-3)
    r = lra.maxvol(np.array([[4.0], [2.0], [1.0]]), start=np.array([2]))
    assert list(r.S) == [0] and r.swaps == 1 and r.margins == [0.5]


def test_pivot_margin_two_columns_tie_across_columns():
    """A swap decision over a 2-column C': the two largest entries in different columns and
    rows, equal -> the smallest row-major index wins and the margin is 0."""
    B = np.array([[1.0, 0.0], [0.0, 1.0], [3.0, 0.5], [0.5, 3.0]])
    r = lra.maxvol(B, start=np.array([0, 1]))
    assert r.margins[0] == 0.0 and list(r.S)[0] == 2


def _det_bareiss(M):
    """Exact integer determinant (fraction-free Bareiss elimination, Python ints)."""
    A = [[int(x) for x in row] for row in M]
    n = len(A)
    sign, prev = 1, 1
    for k in range(n - 1):
        if A[k][k] == 0:
            sw = next((i for i in range(k + 1, n) if A[i][k] != 0), None)
            if sw is None:
                return 0
            A[k], A[sw] = A[sw], A[k]
            sign = -sign
        for i in range(k + 1, n):
            for j in range(k + 1, n):
                A[i][j] = (A[i][j] * A[k][k] - A[i][k] * A[k][j]) // prev
        prev = A[k][k]
    return sign * A[n - 1][n - 1]


def test_logvol_final_equals_exact_integer_determinant():
    """logvol_final = log|det W[I,J]| of the final generator (eq. eqvol with k = l): on an
    integer-valued W it equals the log of the exact Bareiss determinant of W[I,J] to 1e-12."""
    g = np.random.default_rng(12)
    W = g.integers(-9, 10, (60, 50)).astype(np.float64)
    ca = lra.cross_approx(lra.DenseOperand(W), 6, 6, 3, I0=np.arange(6))
    d = _det_bareiss(W[np.ix_(ca.I, ca.J)])
    assert d != 0
    assert ca.logvol_final == pytest.approx(np.log(abs(float(d))), rel=1e-12)
    assert 0.0 <= ca.min_pivot_margin <= 1.0 and len(ca.margins) == ca.lu_steps + ca.swaps
