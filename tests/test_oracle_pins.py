"""Pins for the CPU oracle (oracle/): each check ties it to something other than itself.

Every test here is CPU-only.  A plausible mistake in the oracle -- a dropped term in a
dot product, a wrong sign in a substitution, a transposed operand, an off-by-one in the
X_R column of problem i, X_L/X_R coefficient order swapped -- fails at least one of:

* the SPEC/paper worked examples (tests/golden/spec_examples.json, cited per entry);
* exact rational brute force of Eq. (1) with explicit inverses;
* the M = I ordinary-least-squares closed form (p = 2) and LAPACK lstsq (Alg. 1 route,
  PAPER.md:140-145);
* scaling invariance b(cM) = b(M) (bitwise for c = 4);
* planted beta: noise-free y = X_L beta => b_i = (beta, 0) for every i;
* M^-1-orthogonality: x_R with X_L^T M^-1 x_R = 0 and y^T M^-1 x_R = 0 => b_B = 0;
* whitening invariance against scipy's Cholesky;
* a LAPACK (scipy) cross-check of the whole sequence on a config-0-shaped problem;
* rank-deficiency isolation (reading A4) and NotSPD pivot reporting (reading A5).
"""
from fractions import Fraction

import numpy as np
import pytest
import scipy.linalg as sla

import gen
import oracle


# ----------------------------------------------------------------------------- helpers
def frac_inverse(A):
    """Exact inverse of a square Fraction matrix by Gauss-Jordan elimination."""
    n = len(A)
    M = [[Fraction(A[i][j]) for j in range(n)] + [Fraction(int(i == j)) for j in range(n)]
         for i in range(n)]
    for c in range(n):
        piv = next(r for r in range(c, n) if M[r][c] != 0)
        M[c], M[piv] = M[piv], M[c]
        pv = M[c][c]
        M[c] = [v / pv for v in M[c]]
        for r in range(n):
            if r != c and M[r][c] != 0:
                f = M[r][c]
                M[r] = [a - f * b for a, b in zip(M[r], M[c])]
    return [row[n:] for row in M]


def frac_matmul(A, B):
    return [[sum(A[i][k] * B[k][j] for k in range(len(B))) for j in range(len(B[0]))]
            for i in range(len(A))]


def frac_T(A):
    return [list(r) for r in zip(*A)]


def exact_gls(M, X, y):
    """b = (X^T M^-1 X)^-1 X^T M^-1 y exactly (Eq. (1), explicit inverses)."""
    Mi = frac_inverse(M)
    Xt = frac_T(X)
    XtMi = frac_matmul(Xt, Mi)
    S = frac_matmul(XtMi, X)
    r = frac_matmul(XtMi, [[v] for v in y])
    b = frac_matmul(frac_inverse(S), r)
    return [row[0] for row in b]


def col_major(cols):
    """list of length-n columns -> (k, n) array (column-major n x k)."""
    return np.ascontiguousarray(np.array(cols, dtype=np.float64))


# ----------------------------------------------------------------------------- examples
def test_spec_cholesky_examples(golden):
    for ex in golden["cholesky"]:
        L = oracle.cholesky(np.array(ex["M"], dtype=float))
        np.testing.assert_allclose(L, np.array(ex["L"]), rtol=0, atol=1e-15, err_msg=ex["cite"])


def test_spec_not_spd(golden):
    for ex in golden["cholesky_not_spd"]:
        with pytest.raises(oracle.NotSPD) as ei:
            oracle.cholesky(np.array(ex["M"], dtype=float))
        assert ei.value.pivot == ex["pivot"], ex["cite"]


def test_not_spd_reports_first_failing_pivot():
    # SPD leading 3x3 block, then a row that makes the 4th pivot negative.
    A = np.array([[4, 1, 0, 2], [1, 3, 0, 1], [0, 0, 2, 0], [2, 1, 0, 0.5]], dtype=float)
    with pytest.raises(oracle.NotSPD) as ei:
        oracle.cholesky(A)
    assert ei.value.pivot == 3
    # zero pivot counts as failure (threshold 2^-52 * max diag, reading A5)
    with pytest.raises(oracle.NotSPD) as ei:
        oracle.cholesky(np.array([[1.0, 1.0], [1.0, 1.0]]))
    assert ei.value.pivot == 1


def test_spec_forward(golden):
    for ex in golden["forward"]:
        x = oracle.forward(np.array(ex["L"], dtype=float), np.array(ex["b"], dtype=float))
        np.testing.assert_array_equal(x, np.array(ex["x"], dtype=float), err_msg=ex["cite"])


def test_spec_spd_solve(golden):
    for ex in golden["spd_solve"]:
        b, st = oracle.spd_solve(np.array(ex["S"], dtype=float), np.array(ex["r"], dtype=float))
        assert st == 0
        np.testing.assert_allclose(b, ex["b"], rtol=1e-15, atol=0, err_msg=ex["cite"])
    for ex in golden["spd_solve_rank_deficient"]:
        b, st = oracle.spd_solve(np.array(ex["S"], dtype=float), np.array(ex["r"], dtype=float))
        assert st == 1 and np.all(np.isnan(b)), ex["cite"]


def test_spec_gls_identity_e1(golden):
    ex = golden["gls_identity_e1"]
    n = ex["n"]
    y = np.array(ex["y"])
    e1 = np.zeros((1, n)); e1[0, 0] = 1.0
    b, st = oracle.solve(np.eye(n), np.zeros((0, n)), y, e1, pR=1)
    assert st[0] == 0 and b[0, 0] == y[0], ex["cite"]


def test_orthonormal_X_identity_M():
    # M = I with orthonormal columns => b = X^T y.
    rng = np.random.default_rng(1)
    n = 9
    Q, _ = np.linalg.qr(rng.standard_normal((n, 3)))
    y = rng.standard_normal(n)
    XL = col_major([Q[:, 0], Q[:, 1]])
    XR = col_major([Q[:, 2]])
    b, st = oracle.solve(np.eye(n), XL, y, XR, pR=1)
    np.testing.assert_allclose(b[0], Q.T @ y, rtol=0, atol=1e-14)


# ----------------------------------------------------------------------------- Cholesky
def test_cholesky_residual_and_lapack():
    rng = np.random.default_rng(7)
    for n in (8, 33, 120):
        A = rng.standard_normal((n, n))
        M = A @ A.T + 8 * np.eye(n)
        L = oracle.cholesky(M)
        assert np.allclose(np.triu(L, 1), 0)
        res = np.linalg.norm(L @ L.T - M) / np.linalg.norm(M)
        assert res <= 1e-13
        np.testing.assert_allclose(L, sla.cholesky(M, lower=True), rtol=1e-11, atol=1e-13)


def test_forward_against_lapack_and_column_separable():
    rng = np.random.default_rng(8)
    n = 64
    A = rng.standard_normal((n, n))
    L = oracle.cholesky(A @ A.T + n * np.eye(n))
    B = rng.standard_normal((5, n))
    for j in range(5):
        x = oracle.forward(L, B[j])
        np.testing.assert_allclose(x, sla.solve_triangular(L, B[j], lower=True), rtol=1e-12, atol=1e-13)


# ----------------------------------------------------------------------------- Eq. (1)
@pytest.mark.parametrize("n,pL,pR,m,seed", [(5, 1, 1, 4, 0), (7, 2, 1, 5, 1), (8, 0, 2, 3, 2),
                                           (6, 3, 1, 6, 3), (8, 1, 3, 3, 4), (4, 0, 1, 4, 5)])
def test_exact_rational_brute_force(n, pL, pR, m, seed):
    """Eq. (1) evaluated exactly in rationals with explicit inverses."""
    rng = np.random.default_rng(100 + seed)
    A = rng.integers(-3, 4, size=(n, n))
    Mi = (A @ A.T + n * np.eye(n, dtype=np.int64)).astype(np.int64)   # SPD, integer
    XLi = rng.integers(-2, 3, size=(pL, n))
    if pL:
        XLi[0] = 1
    XRi = rng.integers(0, 3, size=(m * pR, n))
    yi = rng.integers(-5, 6, size=n)
    Mf = [[Fraction(int(v)) for v in row] for row in Mi]
    b_or, st = oracle.solve(Mi.astype(float), XLi.astype(float), yi.astype(float),
                            XRi.astype(float), pR)
    checked = 0
    for i in range(m):
        cols = [XLi[k] for k in range(pL)] + [XRi[i * pR + k] for k in range(pR)]
        X = [[Fraction(int(c[r])) for c in cols] for r in range(n)]
        # skip exactly singular designs (the oracle must flag them)
        Xf = np.array(cols, dtype=float).T
        if np.linalg.matrix_rank(Xf) < pL + pR:
            assert st[i] == 1
            continue
        b_ex = np.array([float(v) for v in exact_gls(Mf, X, [Fraction(int(v)) for v in yi])])
        assert st[i] == 0
        err = np.max(np.abs(b_or[i] - b_ex)) / max(np.max(np.abs(b_ex)), 1e-300)
        assert err <= 1e-13, (i, b_or[i], b_ex)
        checked += 1
    assert checked >= 1


def test_identity_M_ols_closed_form_p2():
    """M = I, X = (1 | x): slope = sum (x-xb)(y-yb) / sum (x-xb)^2, intercept = yb - slope xb."""
    cfg = gen.CONFIGS[0]
    n = 300
    x_all = gen.make_XR(gen.DEFAULT_SEED, n, 0, 20)
    y = gen.normals(gen.DEFAULT_SEED, 4, 0, n) + 0.3 * x_all[3]
    ones = np.ones((1, n))
    b, st = oracle.solve(np.eye(n), ones, y, x_all, pR=1)
    for i in range(20):
        x = x_all[i]
        xb, yb = x.mean(), y.mean()
        slope = np.sum((x - xb) * (y - yb)) / np.sum((x - xb) ** 2)
        icpt = yb - slope * xb
        np.testing.assert_allclose(b[i], [icpt, slope], rtol=1e-11, atol=1e-13)
    assert cfg.n == 500  # config table sanity


def test_identity_M_lstsq_pL3():
    """M = I, pL = 3: Alg. 1 reduces GLS to least squares; LAPACK gelsd."""
    P = gen.make_problem(200, 3, 1, with_sex=True, seed=11)
    XR = gen.make_XR(11, 200, 0, 10)
    b, st = oracle.solve(np.eye(200), P.XL, P.y, XR, pR=1)
    for i in range(10):
        X = np.column_stack([P.XL.T, XR[i]])
        ref = np.linalg.lstsq(X, P.y, rcond=None)[0]
        np.testing.assert_allclose(b[i], ref, rtol=1e-10, atol=1e-12)


def test_scaling_invariance():
    """b(cM) = b(M): bitwise for c = 4 (chol(4M) = 2 chol(M) exactly), <= 1e-13 norm-wise for c = 3."""
    P = gen.make_problem(120, 3, 1, seed=5)
    XR = gen.make_XR(5, 120, 0, 40)
    b1, s1 = oracle.solve(P.M, P.XL, P.y, XR, 1)
    b4, s4 = oracle.solve(4.0 * P.M, P.XL, P.y, XR, 1)
    b3, s3 = oracle.solve(3.0 * P.M, P.XL, P.y, XR, 1)
    assert np.all(s1 == 0)
    np.testing.assert_array_equal(b1, b4)
    rel = np.max(np.linalg.norm(b3 - b1, axis=1) / np.linalg.norm(b1, axis=1))   # norm-wise per b_i
    assert rel <= 1e-13


@pytest.mark.parametrize("pL,pR,sex", [(3, 1, True), (5, 2, False)])
def test_planted_beta_noise_free(pL, pR, sex):
    """y = X_L beta (no noise) lies in span(X_L) subset span(X_i) => b_i = (beta, 0) exactly."""
    n = 150
    P = gen.make_problem(n, pL, pR, with_sex=sex, seed=21, noise=0.0)
    XR = gen.make_XR(21, n, 0, 30 * pR)
    b, st = oracle.solve(P.M, P.XL, P.y, XR, pR)
    assert np.all(st == 0)
    ref = np.concatenate([P.beta_L, np.zeros(pR)])
    err = np.max(np.abs(b - ref)) / np.max(np.abs(P.beta_L))
    assert err <= 1e-12


def test_planted_snp_effect():
    """y = X_L beta + x_{i*} beta_R (no noise) => b_{i*} = (beta, beta_R)."""
    n = 140
    P = gen.make_problem(n, 3, 1, seed=22, noise=0.0)
    XR = gen.make_XR(22, n, 0, 8)
    y = P.y + 0.75 * XR[5]
    b, st = oracle.solve(P.M, P.XL, y, XR, 1, sel=[5])
    np.testing.assert_allclose(b[0], np.concatenate([P.beta_L, [0.75]]), rtol=1e-12, atol=1e-12)


def test_orthogonality_gives_zero_bB():
    """x_R = M v with v ⟂ X_L, y: X_L^T M^-1 x_R = 0, y^T M^-1 x_R = 0 => b_B = 0,
    and b_T equals the GLS estimate on X_L alone (computed here with LAPACK)."""
    n = 90
    P = gen.make_problem(n, 3, 1, seed=23)
    rng = np.random.default_rng(23)
    B = np.column_stack([P.XL.T, P.y])
    v = rng.standard_normal(n)
    v -= B @ np.linalg.lstsq(B, v, rcond=None)[0]
    xr = (P.M @ v)[None, :]
    b, st = oracle.solve(P.M, P.XL, P.y, xr, 1)
    assert abs(b[0, 3]) <= 1e-12 * np.max(np.abs(b[0, :3]))
    Ls = sla.cholesky(P.M, lower=True)
    Xw = sla.solve_triangular(Ls, P.XL.T, lower=True)
    yw = sla.solve_triangular(Ls, P.y, lower=True)
    bT = np.linalg.lstsq(Xw, yw, rcond=None)[0]
    np.testing.assert_allclose(b[0, :3], bT, rtol=1e-11, atol=1e-12)


def test_whitening_invariance():
    """(M; X, y) and (I; L^-1 X, L^-1 y) give the same b; L from LAPACK."""
    n = 110
    P = gen.make_problem(n, 3, 1, seed=24)
    XR = gen.make_XR(24, n, 0, 12)
    b1, _ = oracle.solve(P.M, P.XL, P.y, XR, 1)
    Ls = sla.cholesky(P.M, lower=True)
    W = lambda A: np.ascontiguousarray(sla.solve_triangular(Ls, A.T, lower=True).T)
    b2, _ = oracle.solve(np.eye(n), W(P.XL), sla.solve_triangular(Ls, P.y, lower=True), W(XR), 1)
    np.testing.assert_allclose(b1, b2, rtol=1e-11, atol=1e-12)


def test_lapack_cross_check_config0_shape():
    """Alg. 1 route with LAPACK (scipy cholesky, trsm, gelsd) on a config-0-shaped problem."""
    cfg = gen.CONFIGS[0]
    P = gen.config_problem(cfg)
    sel = np.arange(0, cfg.m, 97)
    XR = gen.make_XR(gen.DEFAULT_SEED, cfg.n, 0, cfg.m)
    b, st = oracle.solve(P.M, P.XL, P.y, XR, 1, sel=sel)
    Ls = sla.cholesky(P.M, lower=True)
    yw = sla.solve_triangular(Ls, P.y, lower=True)
    XLw = sla.solve_triangular(Ls, P.XL.T, lower=True)
    for t, i in enumerate(sel):
        xw = sla.solve_triangular(Ls, XR[i], lower=True)
        ref = np.linalg.lstsq(np.column_stack([XLw, xw]), yw, rcond=None)[0]
        assert np.linalg.norm(b[t] - ref) <= 1e-12 * np.linalg.norm(ref)


def test_rank_deficient_isolation():
    """All-zero SNP and SNP = 2*sex are RankDeficient (NaN row, status 1); others unaffected."""
    n = 100
    P = gen.make_problem(n, 3, 1, with_sex=True, seed=25)
    XR = gen.make_XR(25, n, 0, 6)
    ref, st_ref = oracle.solve(P.M, P.XL, P.y, XR, 1)
    XR2 = XR.copy()
    XR2[1] = 0.0
    XR2[4] = 2.0 * P.XL[2]          # collinear with the sex column
    b, st = oracle.solve(P.M, P.XL, P.y, XR2, 1)
    assert list(st) == [0, 1, 0, 0, 1, 0]
    assert np.all(np.isnan(b[1])) and np.all(np.isnan(b[4]))
    for i in (0, 2, 3, 5):
        np.testing.assert_array_equal(b[i], ref[i])


def test_selection_and_packing_agree():
    P = gen.make_problem(80, 2, 2, with_sex=False, seed=26)
    XR = gen.make_XR(26, 80, 0, 20)
    ball, _ = oracle.solve(P.M, P.XL, P.y, XR, 2)
    sel = np.array([7, 2, 9])
    bsel, _ = oracle.solve(P.M, P.XL, P.y, XR, 2, sel=sel)
    packed = np.concatenate([XR[2 * i:2 * i + 2] for i in sel])
    bpk, _ = oracle.solve(P.M, P.XL, P.y, packed, 2, sel=sel, xr_is_selected=True)
    np.testing.assert_array_equal(bsel, ball[sel])
    np.testing.assert_array_equal(bpk, ball[sel])


# ----------------------------------------------------------------------------- p = 20 (config 3)
@pytest.mark.parametrize("pL,pR", [(16, 4), (0, 20), (19, 1)])
def test_p20_against_lapack(pL, pR):
    """p = 20, the config-3 width (pL = 16 covariates + pR = 4 genotype columns) and the two extreme
    splits: the oracle's 20-stride S / G arrays against the Alg. 1 route done by LAPACK (scipy
    cholesky, solve_triangular, then gelsd least squares on the whitened X_i)."""
    n, m = 260, 12
    P = gen.make_problem(n, pL, pR, with_sex=False, seed=60 + pL)
    XR = gen.make_XR(60 + pL, n, 0, m * pR)
    b, st = oracle.solve(P.M, P.XL, P.y, XR, pR)
    assert np.all(st == 0)
    Ls = sla.cholesky(P.M, lower=True)
    yw = sla.solve_triangular(Ls, P.y, lower=True)
    XLw = sla.solve_triangular(Ls, P.XL.T, lower=True) if pL else np.zeros((n, 0))
    for i in range(m):
        xw = sla.solve_triangular(Ls, XR[i * pR:(i + 1) * pR].T, lower=True)
        ref = np.linalg.lstsq(np.column_stack([XLw, xw]), yw, rcond=None)[0]
        assert np.linalg.norm(b[i] - ref) <= 1e-12 * np.linalg.norm(ref), (i, b[i], ref)


@pytest.mark.parametrize("n,pL,pR,m,seed", [(22, 16, 4, 2, 7), (23, 0, 20, 1, 8)])
def test_exact_rational_brute_force_p20(n, pL, pR, m, seed):
    """Eq. (1) in exact rationals at p = 20 (every index of the 20 x 20 S_i and of the b record)."""
    rng = np.random.default_rng(200 + seed)
    A = rng.integers(-2, 3, size=(n, n))
    Mi = (A @ A.T + n * np.eye(n, dtype=np.int64)).astype(np.int64)
    XLi = rng.integers(-2, 3, size=(pL, n))
    if pL:
        XLi[0] = 1
    XRi = rng.integers(0, 3, size=(m * pR, n))
    yi = rng.integers(-5, 6, size=n)
    b_or, st = oracle.solve(Mi.astype(float), XLi.astype(float), yi.astype(float), XRi.astype(float), pR)
    Mf = [[Fraction(int(v)) for v in row] for row in Mi]
    for i in range(m):
        cols = [XLi[k] for k in range(pL)] + [XRi[i * pR + k] for k in range(pR)]
        assert np.linalg.matrix_rank(np.array(cols, dtype=float).T) == pL + pR
        X = [[Fraction(int(c[r])) for c in cols] for r in range(n)]
        b_ex = np.array([float(v) for v in exact_gls(Mf, X, [Fraction(int(v)) for v in yi])])
        assert st[i] == 0
        err = np.linalg.norm(b_or[i] - b_ex) / np.linalg.norm(b_ex)
        assert err <= 1e-12, (i, err)


def test_planted_beta_p20():
    """Config-3 shape (pL = 16, pR = 4), noise-free y = X_L beta => b_i = (beta, 0, 0, 0, 0)."""
    n = 200
    P = gen.make_problem(n, 16, 4, with_sex=False, seed=61, noise=0.0)
    XR = gen.make_XR(61, n, 0, 10 * 4)
    b, st = oracle.solve(P.M, P.XL, P.y, XR, 4)
    assert np.all(st == 0)
    ref = np.concatenate([P.beta_L, np.zeros(4)])
    assert np.max(np.abs(b - ref)) / np.max(np.abs(P.beta_L)) <= 1e-11
