"""fp64 oracle of the hot path: Alg 10.2 (algrhtcur) with C-A iterations at stage 3
(Remark rerfnhmt), maxvol by Alg D.2 stage 1 + Alg D.1, canonical nucleus (Alg 3.1),
and the a-posteriori check ρ = ‖W − CUR‖_F / ‖W‖_F.

TEST INFRASTRUCTURE (see oracle/__init__.py).  Plain numpy, fp64 / complex128, no
blocking or fusion beyond what each cited definition states.  W is an (m, n) array whose
values are converted exactly to fp64.  Index sets are int64 arrays in *slot order*.
"""
from __future__ import annotations

from dataclasses import dataclass, field

import numpy as np

from .transforms import fourier_column_support, hadamard_column_support

TAU = 1e-12   # tie slack of the pivot rule (reading C11 / R6)
TOL = 1e-12   # dominance tolerance |c_ij| <= 1 + TOL (reading C12; BASELINE.json)


class Singular(Exception):
    """Exactly-zero / non-finite pivot, or σ_r(W[I,J]) = 0 (SPEC's 'singular generator')."""


# ================================================================ stage 1: sketch
def sketch(W: np.ndarray, mult: dict) -> np.ndarray:
    """Y = W·M (Alg 10.2 stage 1; M = the realized multiplier).

    ARHT: M = (D·H_{n,d}·P)[:, σ]; column c of Y is
          Σ_{t<2^d} D_k·H[k,σ_c]·W[:,k] over the 2^d nonzeros k of column σ_c,
          summed in ascending t (= ascending k).
    ARFT: the same with Ω_{n,d} (complex128 result).
    sparse: Σ_{t<nnz} sgn_{t,c}·W[:, row_{t,c}] in draw order (reading C7).
    gaussian: Σ_{k<n} W[:,k]·Ω[k,:], accumulated sequentially in k.
    The SRHT scale √(n/l̄) is omitted (reading C8: pivoting is scale-invariant)."""
    W = np.asarray(W, dtype=np.float64)
    m, n = W.shape
    kind, lbar = mult["kind"], mult["lbar"]
    if kind == "qgauss":                      # NEXT-4: Y = W·Ω with Ω = G_q[:, σ] (exact integers)
        return sketch(W, dict(kind="gaussian", lbar=lbar, omega=qgauss_omega(mult), n=mult["n"]))
    if kind == "arht":
        Y = np.zeros((m, lbar))
        for c, sig in enumerate(mult["col"]):
            rows, vals = hadamard_column_support(n, mult["depth"], int(sig))
            for k, h in zip(rows, vals):
                coef = float(mult["dsign"][k]) * h            # ±1
                Y[:, c] = Y[:, c] + coef * W[:, k]
        return Y
    if kind == "arft":
        Yr = np.zeros((m, lbar))
        Yi = np.zeros((m, lbar))
        for c, sig in enumerate(mult["col"]):
            rows, vals = fourier_column_support(n, mult["depth"], int(sig))
            for k, w in zip(rows, vals):
                dk = float(mult["dsign"][k])
                Yr[:, c] = Yr[:, c] + W[:, k] * (dk * w.real)
                Yi[:, c] = Yi[:, c] + W[:, k] * (dk * w.imag)
        return Yr + 1j * Yi
    if kind == "sparse":
        nnz = mult["nnz"]
        Y = np.zeros((m, lbar))
        for c in range(lbar):
            for t in range(nnz):
                k = int(mult["sp_row"][c * nnz + t])
                Y[:, c] = Y[:, c] + float(mult["sp_sign"][c * nnz + t]) * W[:, k]
        return Y
    if kind == "gaussian":
        Om = np.asarray(mult["omega"], dtype=np.float64)
        Y = np.zeros((m, lbar))
        for k in range(n):
            Y = Y + np.outer(W[:, k], Om[k, :])
        return Y
    raise ValueError(kind)


def bidiag_product_columns(perm, diag, sub, col) -> np.ndarray:
    """Columns `col` of G = M_0 M_1 ... M_{q-1}, M_i = B_i P_i (def11 / def2):
    B_i has diag[i][c] at (c, c) and sub[i][c] at (c + 1 mod n, c); P_i[perm[i][c], c] = 1.
    Applied right to left to the selection S (G S = M_0 (M_1 (... (M_{q-1} S)))):
    (P V)[perm[c]] = V[c], then (B U)[r] = diag[r] U[r] + sub[r-1] U[r-1] (cyclic).
    Exact for integer entries below 2^53."""
    q, n = np.asarray(perm).shape
    V = np.zeros((n, len(col)))
    V[np.asarray(col), np.arange(len(col))] = 1.0
    for i in reversed(range(q)):
        U = np.empty_like(V)
        U[np.asarray(perm[i]), :] = V
        V = np.asarray(diag[i], dtype=np.float64)[:, None] * U + np.roll(np.asarray(sub[i], dtype=np.float64)[:, None] * U, 1, axis=0)
    return V


def qgauss_omega(mult: dict) -> np.ndarray:
    """Ω = G_q[:, σ] of the quasi-Gaussian multiplier (ones on the diagonal, random signs on
    the cyclic subdiagonal, NEXT-4); the sketch is then Y = W·Ω as for a Gaussian Ω."""
    q, n = mult["qg_perm"].shape
    return bidiag_product_columns(mult["qg_perm"], np.ones((q, n)), mult["qg_sign"], mult["col"])


def preprocess_full(W: np.ndarray, mult: dict) -> np.ndarray:
    """Alg 10.1 stage 1 with u = n and the abridged randomized Hadamard multiplier
    (the Table tb_fh protocol P:4882-4914):
    W' = W·D·H_{n,d}·P with ALL n columns, column c = (W D H_{n,d})[:, perm[c]] — the same
    ascending-t signed sum as `sketch` with lbar = n — stored in W's precision (reading C25:
    fp32 W -> fl32 of the fp64 sum, fp64 W -> the fp64 sum)."""
    W = np.asarray(W)
    if mult["kind"] != "arht" or mult["lbar"] != W.shape[1]:
        raise ValueError("full pre-processing: ARHT multiplier with lbar = n")
    Wp = sketch(W, mult)
    return Wp.astype(np.float32) if W.dtype == np.float32 else Wp


def cur_preprocessed(W, mult_full, r: int, k: int, sweeps: int, I0):
    """Alg 10.1 with C-A as its CUR subalgorithm (the Table tb_fh protocol, P:4882-4914;
    SURVEY NEXT-1): W' = W·D·H_{n,d}·P, C-A ("Tests 2": random I0) and the
    canonical nucleus on W', so C = W'[:,J], U = W'_{k,l,r}^+ and R = R_H·H^+ = W[I,:]
    (R = R_H H^+, H square and invertible).  The relative residual on W' equals the
    one on W because M M^T = 2^d I (so ||X M||_F = 2^{d/2} ||X||_F).  Returns the CurResult
    on W' and rho_W = ||W - C U W[I,:]||_F / ||W||_F computed directly."""
    Wp = preprocess_full(W, mult_full)
    res = cur_pipeline(Wp, None, r, k, k, sweeps, I0=I0)
    Wd = np.asarray(W, dtype=np.float64)
    C = np.asarray(Wp, dtype=np.float64)[:, res.J]
    D = Wd - C @ res.U @ Wd[res.I, :]
    rho_w = float(np.sqrt(np.sum(D * D) / np.sum(Wd * Wd)))
    return res, rho_w


# ====================================================== maxvol (Alg D.2 + Alg D.1)
@dataclass
class MaxvolResult:
    S: np.ndarray                 # slot-ordered selected rows
    cert: float                   # max |C| at exit (dominance certificate)
    swaps: int
    lu_steps: int
    cap_hit: bool
    logdet: list = field(default_factory=list)   # log|det B[S,:]| after start and each swap
    margins: list = field(default_factory=list)  # top-2 margin of every pivot decision (see pivot_margin)


def pivot_margin(cand: np.ndarray, chosen: int) -> float:
    """Top-2 margin of one pivot decision (SURVEY §8(b) `min_pivot_margin`, reading C35):
    (M − M₂)/M with M the largest candidate magnitude and M₂ the largest magnitude among the
    candidates other than the chosen one (0 if there is none): 0 when the index rule broke a
    tie inside the slack window (the chosen entry is not the unique maximum), small when a
    rounding-level change could reorder the top two."""
    a = np.asarray(cand, dtype=np.float64).copy()
    M = float(a.max())
    a[chosen] = -np.inf
    M2 = float(a.max()) if len(a) > 1 else 0.0
    M2 = max(M2, 0.0)
    return (M - M2) / M


def lup_pivots(B: np.ndarray, tau: float = TAU, margins=None) -> np.ndarray:
    """Cold start = Alg D.2 stage 1 on the tall block B (N×q): LU with
    partial (row) pivoting.  Step t: M_t = max over unchosen rows of |B'[i,t]|;
    p = smallest unchosen i with |B'[i,t]| ≥ (1−τ)·M_t (reading C11); then for every
    unchosen i: B'[i,t:] −= (B'[i,t]/B'[p,t])·B'[p,t:]  (one IEEE multiply, one subtract)."""
    Bp = np.array(B, dtype=np.complex128 if np.iscomplexobj(B) else np.float64)
    N, q = Bp.shape
    chosen = np.zeros(N, dtype=bool)
    S = np.empty(q, dtype=np.int64)
    for t in range(q):
        a = np.abs(Bp[:, t])
        a[chosen] = -1.0
        M = a.max()
        if not np.isfinite(M) or M <= 0.0:
            raise Singular(f"LUP: zero/non-finite pivot at step {t}")
        p = int(np.flatnonzero(a >= (1.0 - tau) * M)[0])
        if margins is not None:
            margins.append(pivot_margin(a[~chosen], int(np.sum(~chosen[:p]))))
        S[t] = p
        chosen[p] = True
        rest = ~chosen
        f = Bp[rest, t] / Bp[p, t]
        Bp[rest, t:] = Bp[rest, t:] - f[:, None] * Bp[p, t:][None, :]
    return S


def maxvol(B: np.ndarray, start=None, tau: float = TAU, tol: float = TOL, cap=None) -> MaxvolResult:
    """Dominant q×q submatrix of the tall N×q block B (Alg D.1, transposed
    to rows): from the start slots S (LUP cold start if None),
      1. C = B·B[S,:]⁻¹ (from scratch); m* = max|C|; stop if m* ≤ 1+tol or cap reached;
      2. (i*, j*) = smallest row-major index i·q+j with |C[i,j]| ≥ (1−τ)m*; S[j*] ← i*.
    Each swap multiplies |det B[S,:]| by |C[i*,j*]| > 1."""
    B = np.asarray(B)
    N, q = B.shape
    cap = 20 * q if cap is None else cap
    margins = []
    if start is None:
        S = lup_pivots(B, tau, margins)
        lu_steps = q
    else:
        S = np.array(start, dtype=np.int64).copy()
        lu_steps = 0
    swaps = 0
    logdet = []
    while True:
        BS = B[S, :]
        sign, ld = np.linalg.slogdet(BS)
        if sign == 0 or not np.isfinite(ld):
            raise Singular("maxvol: singular B[S,:]")
        logdet.append(float(ld))
        C = np.linalg.solve(BS.T, B.T).T          # C = B · B[S,:]⁻¹
        absC = np.abs(C)
        # C[S,:] = I_q exactly (Alg D.2 stage 2: C = (I_r | C')); the test and the swap
        # search run over the non-selected rows C' only (stage 3, "||A'_1||_C <= 1").
        absC[S, :] = 0.0
        mstar = float(absC.max())
        if mstar <= 1.0 + tol or swaps >= cap:
            return MaxvolResult(S, mstar, swaps, lu_steps, mstar > 1.0 + tol, logdet, margins)
        flat = int(np.flatnonzero(absC.ravel() >= (1.0 - tau) * mstar)[0])
        keep = np.ones(N, dtype=bool)
        keep[S] = False                                  # candidates: the rows outside S
        margins.append(pivot_margin(absC[keep, :].ravel(), int(np.sum(keep[:flat // q])) * q + flat % q))
        i, j = divmod(flat, q)
        S[j] = i
        swaps += 1


# ======================================================= operands ("W or an entry oracle")
class DenseOperand:
    """W given densely (m×n)."""

    def __init__(self, W):
        self.W = np.asarray(W, dtype=np.float64)
        self.m, self.n = self.W.shape

    def rows(self, I):
        return self.W[np.asarray(I), :]

    def cols(self, J):
        return self.W[:, np.asarray(J)]

    def block(self, I, J):
        return self.W[np.ix_(np.asarray(I), np.asarray(J))]

    def entries(self, ii, jj):
        return self.W[np.asarray(ii), np.asarray(jj)]


class FactoredOperand:
    """Entry oracle W_ij = A_{i,:}·B_{:,j} + E_ij with E in CSR (config 4); W never formed."""

    def __init__(self, A, B, row_ptr, col, val):
        self.A = np.asarray(A, dtype=np.float64)
        self.B = np.asarray(B, dtype=np.float64)
        self.row_ptr, self.col, self.val = np.asarray(row_ptr), np.asarray(col), np.asarray(val, dtype=np.float64)
        self.m, self.n = self.A.shape[0], self.B.shape[1]

    def _e_rows(self, I):
        out = np.zeros((len(I), self.n))
        for a, i in enumerate(I):
            lo, hi = self.row_ptr[i], self.row_ptr[i + 1]
            out[a, self.col[lo:hi]] = self.val[lo:hi]
        return out

    def rows(self, I):
        I = np.asarray(I)
        return self.A[I, :] @ self.B + self._e_rows(I)

    def cols(self, J):
        J = np.asarray(J)
        out = self.A @ self.B[:, J]
        pos = {int(j): c for c, j in enumerate(J)}
        for i in range(self.m):
            for e in range(self.row_ptr[i], self.row_ptr[i + 1]):
                c = pos.get(int(self.col[e]))
                if c is not None:
                    out[i, c] += self.val[e]
        return out

    def block(self, I, J):
        return self.rows(I)[:, np.asarray(J)]

    def entries(self, ii, jj):
        """W(i_q, j_q) = A[i_q,:]·B[:,j_q] + E(i_q, j_q) for arrays of pairs."""
        ii = np.asarray(ii, dtype=np.int64)
        jj = np.asarray(jj, dtype=np.int64)
        w = np.einsum("qt,tq->q", self.A[ii, :], self.B[:, jj])
        rows = np.repeat(np.arange(self.m, dtype=np.int64), np.diff(self.row_ptr))
        keys = rows * self.n + self.col
        qk = ii * self.n + jj
        pos = np.searchsorted(keys, qk)
        pos = np.minimum(pos, len(keys) - 1)
        hit = keys[pos] == qk if len(keys) else np.zeros(len(qk), bool)
        return w + np.where(hit, self.val[pos] if len(keys) else 0.0, 0.0)


# ============================================================ C-A loops (stage 3)
@dataclass
class CAResult:
    I: np.ndarray
    J: np.ndarray
    loops_done: int
    lu_steps: int
    swaps: int
    cap_hits: int
    cert_rows: float
    cert_cols: float
    logdet_steps: list      # log|det W[I,J]| after every C-A step (start of each maxvol)
    steps: list             # per-maxvol (side, swaps)
    margins: list = field(default_factory=list)   # top-2 margins of every pivot decision

    @property
    def logvol_final(self) -> float:
        """log v₂(W[I,J]) = log|det W[I,J]| of the final generator (eq. eqvol)."""
        return self.logdet_steps[-1]

    @property
    def min_pivot_margin(self) -> float:
        return min(self.margins) if self.margins else float("nan")


def cross_approx(op, k: int, l: int, sweeps: int, Y=None, I0=None, J0=None,
                 tau: float = TAU, tol: float = TOL, cap=None) -> CAResult:
    """Alg 10.2 stages 2–3 with C-A iterations at stage 3 (Remark rerfnhmt):
      I ← maxvol(Y) cold (stage 2), or I ← I₀ given (Tests 2);
      loop 1..T:  J ← maxvol(W[I,:]ᵀ, start = J if loop > 1)        (horizontal step)
                  I ← maxvol(W[:,J],  start = I)                      (vertical step)
                  stop early if neither step swapped (fixed point, reading C13).
    J0 (optional) warm-starts the first horizontal step (restart from a previous result).
    Reading C9: v1 requires k = l (square generators)."""
    if k != l:
        raise ValueError("v1 requires k == l")
    if Y is not None:
        res = maxvol(Y, None, tau, tol, cap)
        I = res.S
        lu, sw, ch = res.lu_steps, res.swaps, int(res.cap_hit)
        steps = [("sketch", res.swaps)]
        margins = list(res.margins)
    else:
        I = np.array(I0, dtype=np.int64)
        lu = sw = ch = 0
        steps = []
        margins = []
    J = None if J0 is None else np.array(J0, dtype=np.int64)
    logdet_steps = []
    cert_r = cert_c = float("nan")
    loops = 0
    for loop in range(sweeps):
        rh = maxvol(op.rows(I).T, J, tau, tol, cap)
        rv = maxvol(op.cols(rh.S), I, tau, tol, cap)
        loops += 1
        lu += rh.lu_steps + rv.lu_steps
        sw += rh.swaps + rv.swaps
        ch += int(rh.cap_hit) + int(rv.cap_hit)
        steps += [("h", rh.swaps), ("v", rv.swaps)]
        logdet_steps += rh.logdet + rv.logdet
        margins += rh.margins + rv.margins
        J, I = rh.S, rv.S
        cert_c, cert_r = rh.cert, rv.cert
        if loop > 0 and rh.swaps == 0 and rv.swaps == 0:
            break
    return CAResult(I, J, loops, lu, sw, ch, cert_r, cert_c, logdet_steps, steps, margins)


# ============================================ rectangular generators (Alg D.4, NEXT-3)
def expand_columns(R: np.ndarray, J, l: int, tau: float = TAU):
    """Greedy expansion of the k×g submatrix C_g = R[:, J] of the k×n matrix R (g ≥ k, full
    row rank) to k×l (Alg D.4 "algrup"): the column b appended at each step
    maximizes v₂(C_g | b)² = v₂(C_g)²·(1 + bᵀ(C_g C_gᵀ)⁻¹ b) (eq. eqbun), i.e. the score
    ‖L⁻¹ b‖² with L Lᵀ = C_g C_gᵀ (Cholesky, then forward substitution — the "orthogonalizing
    pre-multiplication R_g" of stage 1 is L⁻¹).  Ties: smallest column among scores ≥
    (1 − τ)·max (reading C11).  Returns (J extended to l columns, list of scores)."""
    import scipy.linalg
    R = np.asarray(R, dtype=np.float64)
    J = [int(j) for j in J]
    scores = []
    n = R.shape[1]
    while len(J) < l:
        C = R[:, J]
        L = np.linalg.cholesky(C @ C.T)
        Z = scipy.linalg.solve_triangular(L, R, lower=True)
        sc = np.sum(Z * Z, axis=0)
        sc[J] = -1.0
        mx = float(sc.max())
        j = int(np.flatnonzero(sc >= (1.0 - tau) * mx)[0])
        J.append(j)
        scores.append(mx)
    return np.array(J, dtype=np.int64), scores


def contract_columns(R: np.ndarray, J, l: int, tau: float = TAU):
    """Greedy contraction (Def defgrdc) of C_g = R[:, J] (k×g) down to k×l
    (l ≥ k): each step removes the column whose removal leaves the largest volume.  Since
    v₂(C_{g,j})² = v₂(C_g)²·(1 − c_jᵀ(C_g C_gᵀ)⁻¹c_j) (eq. eqbtr), that is the column of
    minimal leverage ‖L⁻¹c_j‖² (L Lᵀ = C_g C_gᵀ); ties: the smallest slot with leverage ≤
    (1 + τ)·min (reading C11).  The remaining columns keep their slot order."""
    import scipy.linalg
    R = np.asarray(R, dtype=np.float64)
    J = [int(j) for j in J]
    k = R.shape[0]
    if l < k:
        raise ValueError("contraction needs l >= k (C C^T nonsingular)")
    while len(J) > l:
        C = R[:, J]
        L = np.linalg.cholesky(C @ C.T)
        Z = scipy.linalg.solve_triangular(L, C, lower=True)
        lev = np.sum(Z * Z, axis=0)
        mn = float(lev.min())
        t = int(np.flatnonzero(lev <= (1.0 + tau) * mn)[0])
        del J[t]
    return np.array(J, dtype=np.int64)


def refine_columns(R: np.ndarray, J, cycles: int, tau: float = TAU):
    """The expand–contract search of §scrsorth with p = 1: append the greedy
    expansion's column (Alg D.4), then remove the greedy contraction's column (Def defgrdc);
    stop when the contraction removes the column just appended (a fixed point), else repeat
    (the volume never decreases: eqs. eqbun, eqbtr).  Returns (J, cycles that changed J)."""
    J = np.asarray(J, dtype=np.int64)
    l = len(J)
    done = 0
    for _ in range(cycles):
        Jx, _ = expand_columns(R, J, l + 1, tau)
        Jc = contract_columns(R, Jx, l, tau)
        if list(Jc) == list(J):
            break
        J = Jc
        done += 1
    return J, done


def leverage_scores(B: np.ndarray, r: int) -> np.ndarray:
    """SVD-based leverage scores of the n columns of the k×n matrix B (eq. eqlevsc with β = 1,
    eq. eqlevsc1): p_j = ‖(V_r)_{j,:}‖² / r with V_r the r top right singular
    vectors (numpy's SVD as the library step).  Σ p_j = 1."""
    B = np.asarray(B, dtype=np.float64)
    _, sv, Vt = np.linalg.svd(B, full_matrices=False)
    if not 0 < r <= len(sv) or not sv[r - 1] > 0.0:
        raise Singular("leverage scores need rank >= r")
    V = Vt[:r, :].T
    return np.sum(V * V, axis=1) / r


def sample_exactly(p: np.ndarray, l: int, u: np.ndarray):
    """Alg C.1 (algsmplex, "Exactly(l)"): l independent picks with
    Probability(i_t = i) = p_i and the rescaling d_t = 1/sqrt(l·p_{i_t}).  The random picks are
    the caller's uniforms u_t ∈ [0, 1) through the inverse CDF: i_t = the smallest i with
    u_t·P_{n-1} < P_i, P_i = p_0 + … + p_i summed sequentially (reading C31)."""
    p = np.asarray(p, dtype=np.float64)
    P = np.cumsum(p)
    idx = np.searchsorted(P, np.asarray(u, dtype=np.float64) * P[-1], side="right").astype(np.int64)
    idx = np.minimum(idx, len(p) - 1)
    return idx, 1.0 / np.sqrt(l * p[idx])


def sample_expected(p: np.ndarray, l: int, u: np.ndarray):
    """Alg C.2 (algsmplexp, "Expected(l)"), reading C33: ONE pass over j = 0..n-1
    in ascending order; j is picked independently with probability π_j = min{1, l·p_j}, the
    caller's uniform u_j ∈ [0, 1) deciding (picked iff u_j < π_j); the picked j, in ascending
    order, are the sampled columns t = 0, 1, … (their number is random, expected Σ_j π_j ≤ l)
    with the rescaling d_t = 1 / min{1, √(l·p_j)}."""
    p = np.asarray(p, dtype=np.float64)
    u = np.asarray(u, dtype=np.float64)
    pi = np.minimum(1.0, l * p)
    idx = np.nonzero(u < pi)[0].astype(np.int64)
    return idx, 1.0 / np.minimum(1.0, np.sqrt(l * p[idx]))


def cur_uniform(W, r: int, k: int, l: int, u_cols, u_rows, sampler: str = "exactly") -> "CurResult":
    """Alg 9.1 (algcurlevsc) with UNIFORM leverage scores, the superfast variant of
    §slrasmpav ("choosing the norms v_j^{(r)} equal to each other for all j",
    so p_j = 1/n and p̄_i = 1/m): stage 2 samples the columns J with Alg C.1 (Exactly(l)) or
    Alg C.2 (Expected(l)) from p_j = 1/n and the caller's uniforms u_cols; stages 3-4 sample the
    rows I from p̄_i = 1/m (u_rows) — with uniform scores the scores of (C D)ᵀ are uniform too,
    so no SVD is needed; stage 6: the constant rescalings D, D̄ cancel in D M⁺ D̄ and the
    nucleus is the canonical U = W_{I,J,r}⁺ (reading C31).  Then CUR = A·B and ρ."""
    W = np.asarray(W)
    m, n = W.shape
    op = DenseOperand(W)
    pc = np.full(n, 1.0 / n)
    pr = np.full(m, 1.0 / m)
    if sampler == "exactly":
        J, _ = sample_exactly(pc, l, u_cols)
        I, _ = sample_exactly(pr, k, u_rows)
    else:
        J, _ = sample_expected(pc, l, u_cols)
        I, _ = sample_expected(pr, k, u_rows)
    U, Sr, sr, Tr = canonical_nucleus(op.block(I, J), r)
    A, B = rank_r_factors(op.cols(J), op.rows(I), Sr, sr, Tr)
    num2, den2 = cur_residual(W, A, B)
    return CurResult(I, J, U, A, B, num2, den2, None, None)


def cur_leverage(W, r: int, k: int, l: int, sweeps: int, I0, uniforms) -> "CurResult":
    """C-A iterations with the leverage-score sampling of DMM08 (stages 1–2 of Alg 9.1
    "algcurlevsc", with Alg C.1) as the subalgorithm of every horizontal and
    vertical step (§ststc-alvrg): from the rows I0, sweep s samples l columns from
    the leverage scores of W[I,:] with uniforms[2s] and then k rows from those of W[:,J]ᵀ with
    uniforms[2s+1]; the nucleus is the canonical U = W_{I,J,r}⁺ (Remark resmplfc's unscaled
    form, reading C31), CUR = A·B and ρ."""
    W = np.asarray(W)
    op = DenseOperand(W)
    I = np.asarray(I0, dtype=np.int64)
    J = None
    for s in range(sweeps):
        J, _ = sample_exactly(leverage_scores(op.rows(I), r), l, uniforms[2 * s])
        I, _ = sample_exactly(leverage_scores(op.cols(J).T, r), k, uniforms[2 * s + 1])
    U, Sr, sr, Tr = canonical_nucleus(op.block(I, J), r)
    A, B = rank_r_factors(op.cols(J), op.rows(I), Sr, sr, Tr)
    num2, den2 = cur_residual(W, A, B)
    return CurResult(I, J, U, A, B, num2, den2, None, None)


def qrp_columns(R: np.ndarray, q: int, tau: float = TAU):
    """Alg D.3 (alg1tor): greedy expansions from a vector to a k×q submatrix of the
    k×n matrix R by Householder reflections with column pivoting.  Step g = 0..q−1:
      1. for every column not yet chosen, the squared norm of its last k−g coordinates,
         summed in ascending row order (one rounded product, one rounded add per term);
      2. pivot b_g = the column of maximal norm (ties: the smallest column among the norms
         ≥ (1 − τ)·max, reading C11);
      3. H'_g = I − β v vᵀ with v = x + sign(x₀)‖x‖e₁, x = the pivot's last k−g coordinates,
         β = 2 / vᵀv (vᵀv summed in ascending order): the pivot's trailing part becomes
         −sign(x₀)‖x‖e₁ (set exactly), every other column y ← y − (β·vᵀy)·v (vᵀy summed in
         ascending order, no fused operations);
      4. W_{g+1} = H_g W_g.
    The paper normalises the diagonal of R_g to 1 (reading C29: column scaling, which changes
    neither the pivots nor the volumes' ratios; R keeps the reflected values here).
    Returns (pivots (q,), the transformed k×n matrix H_{q−1}···H_0 R in the original column
    order).  Raises Singular when the maximal trailing norm is 0 (rank < q)."""
    X = np.array(R, dtype=np.float64, copy=True)
    k, n = X.shape
    if not 0 < q <= min(k, n):
        raise ValueError("need 0 < q <= min(k, n)")
    chosen = np.zeros(n, dtype=bool)
    piv = []
    for g in range(q):
        nrm2 = np.zeros(n)
        for i in range(g, k):
            nrm2 = nrm2 + X[i, :] * X[i, :]
        nrm2[chosen] = -1.0
        mx = float(nrm2.max())
        if not mx > 0.0 or not np.isfinite(mx):
            raise Singular("rank < q in the QRP")
        p = int(np.flatnonzero(nrm2 >= (1.0 - tau) * mx)[0])
        x = X[g:, p].copy()
        alpha = float(np.sqrt(nrm2[p]))
        sgn = 1.0 if x[0] >= 0.0 else -1.0
        v = x.copy()
        v[0] = x[0] + sgn * alpha
        vtv = 0.0
        for i in range(k - g):
            vtv = vtv + v[i] * v[i]
        beta = 2.0 / vtv
        w = np.zeros(n)
        for i in range(k - g):
            w = w + v[i] * X[g + i, :]
        t = beta * w
        for i in range(k - g):
            X[g + i, :] = X[g + i, :] - t * v[i]
        X[g:, p] = 0.0
        X[g, p] = -sgn * alpha
        chosen[p] = True
        piv.append(p)
    return np.array(piv, dtype=np.int64), X


def projective_columns(R: np.ndarray, r: int, l: int, tau: float = TAU, tol: float = TOL):
    """Alg 7.1 (algprjvlm): a column set J (l ≥ r columns) of the k×n matrix R
    with maximal r-projective volume: (1) rank-revealing QRP R = QRP (Alg D.3, r steps), R′ =
    the first r rows of the reflected matrix (r×n); (2) a maximal-volume r×l submatrix of R′:
    the black box is maxvol (Alg D.2 stage 1 + D.1) on R′ᵀ for r columns, then Alg D.4 greedy
    expansion to l columns.  Returns (J, piv, R′)."""
    piv, X = qrp_columns(R, r, tau)
    Rp = X[:r, :].copy()
    mv = maxvol(Rp.T, None, tau, tol)
    J = mv.S
    if l > r:
        J, _ = expand_columns(Rp, J, l, tau)
    return np.asarray(J, dtype=np.int64), piv, Rp


def cur_projective(W, mult, r: int, k: int, l: int, sweeps: int, I0=None) -> "CurResult":
    """NEXT-3 r-projective generators: the square C-A of Alg 10.2 gives the k rows I; Alg 7.1
    on R = W[I,:] picks l ≥ r columns of maximal r-projective volume; then the canonical
    nucleus U = W_{k,l,r}^+ of the k×l generator, CUR = A·B and ρ."""
    op = DenseOperand(W)
    Y = sketch(W, mult) if mult is not None else None
    ca = cross_approx(op, k, k, sweeps, Y=Y, I0=I0)
    J, _, _ = projective_columns(op.rows(ca.I), r, l)
    U, Sr, sr, Tr = canonical_nucleus(op.block(ca.I, J), r)
    A, B = rank_r_factors(op.cols(J), op.rows(ca.I), Sr, sr, Tr)
    num2, den2 = cur_residual(W, A, B)
    return CurResult(ca.I, J, U, A, B, num2, den2, ca, Y)


def cur_rectangular(W, mult, r: int, k: int, l: int, sweeps: int, I0=None) -> "CurResult":
    """k×l generators with l > k (NEXT-3): the square C-A of Alg 10.2 (k = k) gives (I, J),
    Alg D.4 expands J greedily to l columns on R = W[I,:], then the canonical nucleus
    U = W_{k,l,r}^+ (Alg 3.1, rectangular) and CUR = A·B with A = W[:,J] T_r Σ_r⁻¹,
    B = S_rᵀ W[I,:]."""
    op = DenseOperand(W)
    Y = sketch(W, mult) if mult is not None else None
    ca = cross_approx(op, k, k, sweeps, Y=Y, I0=I0)
    J, _ = expand_columns(op.rows(ca.I), ca.J, l)
    U, Sr, sr, Tr = canonical_nucleus(op.block(ca.I, J), r)
    A, B = rank_r_factors(op.cols(J), op.rows(ca.I), Sr, sr, Tr)
    num2, den2 = cur_residual(W, A, B)
    return CurResult(ca.I, J, U, A, B, num2, den2, ca, Y)


# ============================================================ canonical nucleus
def canonical_nucleus(G: np.ndarray, r: int):
    """Alg 3.1 (algcnnncl): U = W_{k,l,r}⁺ from the SVD G = S Σ Tᵀ truncated to
    the r largest singular values: U = T_r Σ_r⁻¹ S_rᵀ (l×k).  Returns (U, S_r, σ_r, T_r)."""
    G = np.asarray(G, dtype=np.float64)
    if not 0 < r <= min(G.shape):
        raise ValueError("need 0 < r <= min(k, l)")
    S, sv, Th = np.linalg.svd(G)
    if not sv[r - 1] > 0.0:
        raise Singular("sigma_r(W[I,J]) = 0")
    Sr, sr, Tr = S[:, :r], sv[:r], Th[:r, :].T
    U = (Tr / sr[None, :]) @ Sr.T
    return U, Sr, sr, Tr


def rank_r_factors(C: np.ndarray, R: np.ndarray, Sr, sr, Tr):
    """CUR = A·B with A = C·T_r·Σ_r⁻¹ (m×r) and B = S_rᵀ·R (r×n)."""
    A = (np.asarray(C, dtype=np.float64) @ Tr) / sr[None, :]
    Bf = Sr.T @ np.asarray(R, dtype=np.float64)
    return A, Bf


# ============================================================ a-posteriori checks
def cur_residual(W: np.ndarray, A: np.ndarray, B: np.ndarray, row_block: int = 1024):
    """num² = Σ_ij (W_ij − (A·B)_ij)², den² = Σ_ij W_ij² in fp64 (eq. eqcur0, P:1153-1155;
    the "dense audit"), row-block partials summed in block order.  ρ = √(num²/den²)."""
    W = np.asarray(W)
    m = W.shape[0]
    num2 = 0.0
    den2 = 0.0
    for i0 in range(0, m, row_block):
        Wb = np.asarray(W[i0:i0 + row_block], dtype=np.float64)
        D = Wb - A[i0:i0 + row_block] @ B
        num2 += float(np.sum(D * D))
        den2 += float(np.sum(Wb * Wb))
    return num2, den2


def sampled_residual(op, A, B, ii, jj):
    """Sampled estimate num²_est = (mn/Q)·Σ_q d_q², d_q = W(i_q,j_q) − A[i_q,:]·B[:,j_q]
    over Q i.i.d. uniform pairs (the mn/Q extrapolation is SPEC S:280-288)."""
    Q = len(ii)
    w = op.entries(ii, jj)
    d = w - np.einsum("qt,tq->q", A[ii, :], B[:, jj])
    return op.m * op.n / Q * float(np.sum(d * d))


def error_sample(op, A, B, rows, cols):
    """Superfast a-posteriori estimation (Section spstr): the
    q×s submatrix E[rows, cols] of E = W − CUR (CUR = A·B) gives K = q·s observed values g_i;
    μ_K = (1/K) Σ g_i and σ_K² = (1/K) Σ |g_i − μ_K|² (reading C26: the paper's |g_i| in μ_K is
    read as g_i, the sample mean of the variable whose variance is tested), and Σ g_i², which
    extrapolates to ‖E‖_F² ≈ (mn/K) Σ g_i², and Σ W_ij² over the same entries (the superfast
    estimate of ‖W‖_F² used by the progressive mode).  `op` is a DenseOperand or
    FactoredOperand."""
    rows = np.asarray(rows, dtype=np.int64)
    cols = np.asarray(cols, dtype=np.int64)
    Wb = op.block(rows, cols)
    Es = Wb - np.asarray(A, dtype=np.float64)[rows, :] @ np.asarray(B, dtype=np.float64)[:, cols]
    g = Es.ravel()
    K = g.size
    mu = float(np.sum(g)) / K
    var = float(np.sum((g - mu) ** 2)) / K
    return mu, var, float(np.sum(g * g)), float(np.sum(Wb * Wb))


def variance_upper_bound(var_K: float, K: int, alpha: float) -> float:
    """One-sided (1−α) upper confidence bound on the variance σ² of a Gaussian variable from
    the biased sample variance σ_K² of K observations (the customary chi-square rule the paper
    refers to): K σ_K² / σ² ~ χ²_{K−1}, so σ² ≤ K σ_K² / χ²_{K−1}(α)."""
    from scipy.stats import chi2
    return K * var_K / chi2.ppf(alpha, K - 1)


def cur_certificate(C, R, U, r: int, delta: float):
    """A-priori error certificate of Corollary cowc1 (ii), eq. (eqnrm11), in
    the Frobenius norm: |W − CUR| ≤ Δ·((|R| + |C| + Δ + μη|C||R||U|)·ξ|U| + 1) with μ = 1,
    η = 1 if r = min(k, l) else 2, (1 − θ)ξ = √(kl), θ = ‖U‖ Δ_{k,l,r} ≤ ‖U‖ η Δ (Lemmas
    leprtpsdinv, leprtinv), where Δ ≥ σ̃_{r+1} (eq. eqnsgmrfr) is the caller's bound.  ‖U‖ is
    bounded by ‖U‖_F (reading C27).  Returns (bound or inf when θ ≥ 1, |C|_F, |R|_F, |U|_F)."""
    C = np.asarray(C, dtype=np.float64)
    R = np.asarray(R, dtype=np.float64)
    U = np.asarray(U, dtype=np.float64)
    l, k = U.shape
    nc, nr, nu = float(np.linalg.norm(C)), float(np.linalg.norm(R)), float(np.linalg.norm(U))
    eta = 1.0 if r == min(k, l) else 2.0
    theta = nu * eta * delta
    if theta >= 1.0:
        return float("inf"), nc, nr, nu
    xi = np.sqrt(k * l) / (1.0 - theta)
    bound = delta * ((nr + nc + delta + eta * nc * nr * nu) * xi * nu + 1.0)
    return float(bound), nc, nr, nu


def cur_progressive(W, r: int, k: int, sweeps: int, tol: float, seed: int, rows, cols, dmax: int = 6):
    """Progressive-depth pre-processing: for d = 1, 2, 3, … apply Alg 10.2 with
    the ARHT multiplier of depth d (Philox seed `seed`) and accept the first CUR LRA whose
    superfast estimate ((mn/K) Σ g²)/((mn/K) Σ W²) over the sampled rows × cols is ≤ tol²
    (Section spstr).  Returns (d, CurResult, rho_estimate) (d = dmax result if none passes)."""
    import synth
    W = np.asarray(W)
    m, n = W.shape
    op = DenseOperand(W)
    d = 1
    while True:
        mult = synth.multiplier_abridged(seed, n, d, k, "arht")
        res = cur_pipeline(W, mult, r, k, k, sweeps, residual=False)
        _, _, ss, sw = error_sample(op, res.A, res.B, rows, cols)
        est = float(np.sqrt(ss / sw)) if sw > 0 else float("inf")
        if est <= tol or d >= dmax or n % (1 << (d + 1)):
            return d, res, est
        d += 1


def factored_den2(op: FactoredOperand) -> float:
    """Exact ‖W‖_F² for W = A·B + E:  tr((AᵀA)(BBᵀ)) + 2·Σ_{(i,j)∈E} E_ij (A·B)_ij + Σ E_ij²."""
    G1 = op.A.T @ op.A
    G2 = op.B @ op.B.T
    t = float(np.sum(G1 * G2))
    cross = 0.0
    for i in range(op.m):
        lo, hi = op.row_ptr[i], op.row_ptr[i + 1]
        if hi > lo:
            cross += float(np.dot(op.val[lo:hi], op.A[i, :] @ op.B[:, op.col[lo:hi]]))
    return t + 2.0 * cross + float(np.dot(op.val, op.val))


# ============================================================ whole path
@dataclass
class CurResult:
    I: np.ndarray
    J: np.ndarray
    U: np.ndarray
    A: np.ndarray
    B: np.ndarray
    num2: float
    den2: float
    ca: CAResult
    Y: object = None

    @property
    def rho(self):
        return float(np.sqrt(self.num2 / self.den2))


def cur_pipeline(W, mult, r: int, k: int, l: int, sweeps: int, I0=None, residual=True) -> CurResult:
    """Alg 10.2 + Remark rerfnhmt + Alg 3.1 + the full a-posteriori check, on dense W."""
    op = DenseOperand(W)
    Y = sketch(W, mult) if mult is not None else None
    ca = cross_approx(op, k, l, sweeps, Y=Y, I0=I0)
    U, Sr, sr, Tr = canonical_nucleus(op.block(ca.I, ca.J), r)
    A, B = rank_r_factors(op.cols(ca.J), op.rows(ca.I), Sr, sr, Tr)
    num2, den2 = cur_residual(W, A, B) if residual else (float("nan"), float("nan"))
    return CurResult(ca.I, ca.J, U, A, B, num2, den2, ca, Y)
