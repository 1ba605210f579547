"""Pins that tie the CPU oracle to what the paper and mathematics fix.

None of these re-types an oracle formula: each compares the oracle against a
hand-evaluated worked example (tests/golden), a closed form, an invariant, a
textbook generator, brute force on tiny inputs, or a library solver with the
paper's exact objective (scikit-learn, scipy).
"""
import itertools
import math
import os

import numpy as np
import pytest

import oracle as O
import synth

GOLD = os.path.join(os.path.dirname(__file__), "golden")


def _load(name):
    return np.loadtxt(os.path.join(GOLD, name), comments="#")


# ----------------------------------------------------------------------------- P1 / P2
def test_P1_lasso_worked_example():
    """P:758 objective, P:852 gap, P:848 B on A = I2, b = (1,1), lambda = 0.25."""
    A = np.eye(2, dtype=np.float32)
    b = np.ones(2)
    lam = 0.25
    B = O.lasso_B(b, lam)
    assert B == 2.0
    for a1, a2, g1, g2, tot, obj in _load("lasso_identity_2x2.txt"):
        alpha = np.array([a1, a2])
        v = O.matvec(A, alpha)
        w = O.primal_dual_w(O.LASSO, v, b, 2, lam)
        st, s, g = O.coord_gaps(O.LASSO, A, alpha, None, w, lam, B)
        assert st == O.OK
        np.testing.assert_allclose(g, [g1, g2], atol=1e-15)
        st, G, Ob, D = O.duality_gap(O.LASSO, A, alpha, b, lam, B)
        assert st == O.OK and abs(G - tot) < 1e-15 and abs(Ob - obj) < 1e-15
        assert abs((Ob - D) - tot) < 1e-14


def test_P2_svm_worked_example():
    """P:773 dual, P:862 primal, P:867 gap on A = I2, y = (+1,-1)."""
    A = np.eye(2, dtype=np.float32)
    y = np.array([1.0, -1.0])
    for lam, a1, a2, g1, g2, tot, dual_obj, primal in _load("svm_identity_2x2.txt"):
        alpha = np.array([a1, a2])
        v = O.matvec(A, alpha)
        w = O.primal_dual_w(O.SVM, v, None, 2, lam)
        st, s, g = O.coord_gaps(O.SVM, A, alpha, y, w, lam)
        assert st == O.OK
        np.testing.assert_allclose(g, [g1, g2], atol=1e-15)
        st, G, Ob, D = O.duality_gap(O.SVM, A, alpha, y, lam)
        assert abs(G - tot) < 1e-15 and abs(Ob - dual_obj) < 1e-15 and abs(-D - primal) < 1e-15


def test_P2_svm_zero_state_gap_is_one():
    """alpha = 0 => gap_i = 1/n exactly, total 1."""
    A, y = synth.svm_dense(37, 301, seed=5)
    n = A.shape[0]
    w = O.primal_dual_w(O.SVM, np.zeros(37), None, n, 0.01)
    st, s, g = O.coord_gaps(O.SVM, A, np.zeros(n), y, w, 0.01)
    assert np.all(g == 1.0 / n)
    st, G, Ob, D = O.duality_gap(O.SVM, A, np.zeros(n), y, 0.01)
    assert abs(G - 1.0) < 1e-13 and Ob == 0.0


# ----------------------------------------------------------------------------- P3 / P4
def _numpy_objectives(model, A, alpha, b_or_y, lam):
    """O and D from the paper's objective and conjugate definitions, in numpy.

    Lasso: f(v) = ||v - b||^2/(2d), g_i = lam |.| on |alpha_i| <= B;
      f*(u) = u^T b + (d/2)||u||^2, g_i*(x) = B [|x| - lam]_+,  u = grad f(A alpha).
    SVM: dual objective P:773 and primal P:862."""
    A64 = A.astype(np.float64)
    n, d = A64.shape
    v = A64.T @ alpha
    if model == O.LASSO:
        b = b_or_y
        B = (b @ b) / (2 * lam * d)
        Ob = ((v - b) @ (v - b)) / (2 * d) + lam * np.abs(alpha).sum()
        u = (v - b) / d
        D = -(u @ b + 0.5 * d * (u @ u)) - B * np.maximum(np.abs(A64 @ u) - lam, 0).sum()
        return Ob, D
    y = b_or_y
    Ob = -(y @ alpha) / n + (v @ v) / (2 * lam * n * n)
    w = v / (lam * n)
    P = np.maximum(0, 1 - y * (A64 @ w)).sum() / n + 0.5 * lam * (w @ w)
    return Ob, -P


@pytest.mark.parametrize("model", [O.LASSO, O.SVM])
def test_P3_gap_identity_and_nonnegativity(model):
    """sum_i gap_i = O(alpha) - D(w) (Eq. 2 / Eq. 4), gap_i >= 0."""
    rng = np.random.default_rng(3)
    if model == O.LASSO:
        A, b = synth.lasso_dense(60, 90, seed=11)
        lab, lam = b, 0.05
    else:
        A, y = synth.svm_dense(40, 120, seed=12)
        lab, lam = y, 0.02
    n = A.shape[0]
    for trial in range(5):
        if model == O.LASSO:
            alpha = rng.standard_normal(n) * (rng.random(n) < 0.3) * 0.1
        else:
            alpha = y * rng.random(n) * (rng.random(n) < 0.5)
        B = O.lasso_B(lab, lam) if model == O.LASSO else 0.0
        st, G, Ob, D = O.duality_gap(model, A, alpha, lab, lam, B)
        On, Dn = _numpy_objectives(model, A, alpha, lab, lam)
        assert abs(Ob - On) <= 1e-12 * max(1, abs(On))
        assert abs(D - Dn) <= 1e-11 * max(1, abs(Dn))
        assert abs(G - (On - Dn)) <= 1e-11 * max(1, abs(On) + abs(Dn))
        v = O.matvec(A, alpha)
        w = O.primal_dual_w(model, v, lab if model == O.LASSO else None, n, lam)
        st, s, g = O.coord_gaps(model, A, alpha, None if model == O.LASSO else lab, w, lam, B)
        assert st == O.OK and np.all(g >= 0)
        np.testing.assert_allclose(s, A.astype(np.float64) @ w, rtol=1e-12, atol=1e-12)


def test_P4_gap_vanishes_at_lasso_kkt_point():
    """Lasso KKT: |a_i^T w| <= lam d, with equality where alpha_i != 0 => gap_i = 0."""
    A, b = synth.lasso_dense(80, 40, seed=21)
    lam = 0.05
    st, alpha, gap, ep = O.solve_scd(O.LASSO, A, b, lam, 1e-13, 5000, seed=1)
    assert st == O.OK and gap <= 1e-13
    w = A.astype(np.float64).T @ alpha - b
    s = A.astype(np.float64) @ w
    d = A.shape[1]
    assert np.all(np.abs(s) <= lam * d * (1 + 1e-6))
    on = alpha != 0
    np.testing.assert_allclose(s[on], -np.sign(alpha[on]) * lam * d, rtol=1e-6)


# ----------------------------------------------------------------------------- P5 / P6
def test_P5_lasso_step_hand_examples():
    """SPEC S:221-222 (App. D.1, eta=0): tau=0.5, gamma=1 => 0.5; lambda=0.5 => 0."""
    # a_j = (1,0), ||a_j||^2 = 1, alpha_j = 0, v~ = (-1, 0) => s = -1, d = 2
    assert O.coord_update(O.LASSO, 0.0, -1.0, 1.0, 0.0, 0.25, 2, 2) == 0.5
    assert O.coord_update(O.LASSO, 0.0, -1.0, 1.0, 0.0, 0.5, 2, 2) == 0.0


def test_P6_svm_step_hand_examples():
    """SPEC S:231-232 (App. D.2): alpha=0, ||a||^2=1, lambda=1, n=1 => +-1."""
    assert O.coord_update(O.SVM, 0.0, 0.0, 1.0, 1.0, 1.0, 1, 1) == 1.0
    assert O.coord_update(O.SVM, 0.0, 0.0, 1.0, -1.0, 1.0, 1, 1) == -1.0


def test_P5_P6_steps_minimise_1d_objective():
    """Each closed-form step is the exact 1-D minimiser of the true objective (scipy bounded)."""
    from scipy.optimize import minimize_scalar
    rng = np.random.default_rng(7)
    for _ in range(100):
        d, n = int(rng.integers(2, 50)), int(rng.integers(2, 50))
        nrm = float(rng.uniform(0.1, 5))
        aj = float(rng.normal())
        s = float(rng.normal() * 3)
        lam = float(rng.uniform(0.001, 0.5))
        # Lasso: phi(x) = (1/2d)||v~ + (x - a_j) a||^2 + lam|x| = (1/2d)[2 s (x-aj) + nrm (x-aj)^2] + lam|x|
        phi = lambda x: (2 * s * (x - aj) + nrm * (x - aj) ** 2) / (2 * d) + lam * abs(x)
        x = O.coord_update(O.LASSO, aj, s, nrm, 0.0, lam, d, n)
        r = minimize_scalar(phi, bounds=(-50, 50), method="bounded", options={"xatol": 1e-10})
        assert phi(x) <= r.fun + 1e-12
        assert abs(x - r.x) < 1e-6
        # SVM dual: psi(x) = -y x / n + (1/(2 lam n^2))[2 s (x - aj) + nrm (x - aj)^2], y x in [0, 1]
        y = float(rng.choice([-1.0, 1.0]))
        ajs = y * float(rng.uniform(0, 1))
        psi = lambda x: -y * x / n + (2 * s * (x - ajs) + nrm * (x - ajs) ** 2) / (2 * lam * n * n)
        x = O.coord_update(O.SVM, ajs, s, nrm, y, lam, d, n)
        lo, hi = (0.0, 1.0) if y > 0 else (-1.0, 0.0)
        r = minimize_scalar(psi, bounds=(lo, hi), method="bounded", options={"xatol": 1e-12})
        cand = min([r.x, lo, hi], key=psi)
        assert lo - 1e-15 <= x <= hi + 1e-15
        assert psi(x) <= psi(cand) + 1e-12 * max(1, abs(psi(cand)))


# ----------------------------------------------------------------------------- ridge (NEXT-2)
def test_R1_ridge_worked_example():
    """A = I_2, b = (1, 1), lambda = 1/4, d = 2.  alpha* = b/(1 + lambda d) = 2/3;
    at alpha = 0: s = a_i^T (A 0 - b) = -1, gap_i = (1/d)(s^2/(2 lambda d)) = 1/2, O = 1/2;
    at alpha*: O* = (1/4)(2/9) + (1/8)(8/9) = 1/6 and every gap vanishes (s = -lambda d alpha)."""
    A = np.eye(2, dtype=np.float32)
    b = np.array([1.0, 1.0])
    lam = 0.25
    w0 = -b
    g0 = O.coord_gaps(O.RIDGE, A, np.zeros(2), None, w0, lam)[2]
    np.testing.assert_allclose(g0, [0.5, 0.5], rtol=0, atol=1e-15)
    st, G, Ob, Db = O.duality_gap(O.RIDGE, A, np.zeros(2), b, lam)
    assert st == O.OK and abs(G - 1.0) < 1e-15 and abs(Ob - 0.5) < 1e-15 and abs(G - (Ob - Db)) < 1e-15
    astar = np.full(2, 2.0 / 3.0)
    st, G, Ob, Db = O.duality_gap(O.RIDGE, A, astar, b, lam)
    assert abs(Ob - 1.0 / 6.0) < 1e-15 and G < 1e-15
    # one exact step from 0 reaches the minimiser (orthonormal design)
    assert abs(O.coord_update(O.RIDGE, 0.0, -1.0, 1.0, 0.0, lam, 2, 2) - 2.0 / 3.0) < 1e-16


def test_R2_ridge_closed_form_optimum_and_gap_identity():
    """Textbook normal equations (A^T A + lambda d I) alpha* = A^T b; plain SCD reaches the
    certified gap and alpha* (strongly convex: unique); sum gap_i = O - D and gap_i >= 0 at
    random states; sklearn Ridge(alpha = lambda d) minimises the same objective."""
    from sklearn.linear_model import Ridge
    d, n, lam = 120, 80, 0.03
    A, b = synth.lasso_dense(d, n, seed=17)
    A64 = A.astype(np.float64).T                     # d x n
    astar = np.linalg.solve(A64.T @ A64 + lam * d * np.eye(n), A64.T @ b)
    st, alpha, gap, ep = O.solve_scd(O.RIDGE, A, b, lam, 1e-13, 5000, seed=2)
    assert st == O.OK and gap <= 1e-13
    np.testing.assert_allclose(alpha, astar, atol=1e-6 * np.abs(astar).max())
    st, G, Ob, Db = O.duality_gap(O.RIDGE, A, astar, b, lam)
    assert G < 1e-12
    sk = Ridge(alpha=lam * d, fit_intercept=False, tol=1e-14, solver="cholesky").fit(A64, b).coef_
    r = A64 @ sk - b
    O_sk = r @ r / (2 * d) + 0.5 * lam * sk @ sk
    assert abs(O_sk - Ob) <= 1e-12 * abs(Ob)
    rng = np.random.default_rng(3)
    for _ in range(5):
        a = rng.standard_normal(n) * 0.3
        st, G, Ob, Db = O.duality_gap(O.RIDGE, A, a, b, lam)
        w = A64 @ a - b
        g = O.coord_gaps(O.RIDGE, A, a, None, w, lam)[2]
        assert np.all(g >= 0) and abs(g.sum() - G) <= 1e-12 * G
        assert abs(G - (Ob - Db)) <= 1e-10 * max(1.0, abs(Ob))
        # closed form of P:841: gap_i = (s_i + lambda d a_i)^2 / (2 lambda d^2)
        s_ = A64.T @ w
        np.testing.assert_allclose(g, (s_ + lam * d * a) ** 2 / (2 * lam * d * d), rtol=1e-9, atol=1e-300)


def test_R3_ridge_step_minimises_1d_objective():
    from scipy.optimize import minimize_scalar
    rng = np.random.default_rng(8)
    for _ in range(100):
        d, n = int(rng.integers(2, 50)), int(rng.integers(2, 50))
        nrm, aj, s_ = float(rng.uniform(0.0, 5)), float(rng.normal()), float(rng.normal() * 3)
        lam = float(rng.uniform(0.001, 0.5))
        phi = lambda x: (2 * s_ * (x - aj) + nrm * (x - aj) ** 2) / (2 * d) + 0.5 * lam * x * x
        x = O.coord_update(O.RIDGE, aj, s_, nrm, 0.0, lam, d, n)
        r = minimize_scalar(phi, bounds=(-100, 100), method="bounded", options={"xatol": 1e-10})
        assert phi(x) <= r.fun + 1e-12 and abs(x - r.x) < 1e-6


@pytest.mark.parametrize("policy", [O.SEL_GAP, O.SEL_UNIFORM])
def test_R4_ridge_duhl_reaches_the_normal_equations(policy):
    d, n, lam = 200, 400, 0.02
    A, b = synth.lasso_dense(d, n, seed=23)
    A64 = A.astype(np.float64).T
    astar = np.linalg.solve(A64.T @ A64 + lam * d * np.eye(n), A64.T @ b)
    r = O.duhl_solve(O.RIDGE, A, b, lam, m=100, passes=2, policy=policy, refresh_count=40,
                     eps=1e-10, max_rounds=3000, cert_every=1, seed=4)
    assert r["status"] == O.OK and r["gap"] <= 1e-10
    np.testing.assert_allclose(r["alpha"], astar, atol=1e-4 * np.abs(astar).max())


# ----------------------------------------------------------------------------- elastic net
def test_E1_elastic_net_worked_example_and_limits():
    """A = I_2, b = (1, 1), lambda = 1/4, eta = 1/2: per coordinate
    (1/4)(a - 1)^2 + lambda (eta/2 a^2 + (1 - eta)|a|) is minimised at
    a* = (1 - 2 lambda (1 - eta)) / (1 + 2 lambda eta) = 0.6, where every gap vanishes; one step from
    0 reaches it.  eta = 1 reproduces the ridge gaps exactly."""
    A = np.eye(2, dtype=np.float32)
    b = np.array([1.0, 1.0])
    lam = 0.25
    O.set_eta(0.5)
    assert abs(O.coord_update(O.ELASTIC, 0.0, -1.0, 1.0, 0.0, lam, 2, 2) - 0.6) < 1e-15
    st, G, Ob, Db = O.duality_gap(O.ELASTIC, A, np.full(2, 0.6), b, lam)
    assert st == O.OK and G < 1e-15 and abs(G - (Ob - Db)) < 1e-15
    # O* = (1/4)(2 * 0.16) + 0.25 (0.25 * 0.72 + 0.5 * 1.2) = 0.08 + 0.195 = 0.275
    assert abs(Ob - 0.275) < 1e-15
    rng = np.random.default_rng(4)
    A2, b2 = synth.lasso_dense(60, 40, seed=8)
    a = rng.standard_normal(40) * 0.2
    w = A2.astype(np.float64).T @ a - b2
    O.set_eta(1.0)
    ge = O.coord_gaps(O.ELASTIC, A2, a, None, w, 0.03)[2]
    gr = O.coord_gaps(O.RIDGE, A2, a, None, w, 0.03)[2]
    np.testing.assert_allclose(ge, gr, rtol=1e-12, atol=1e-300)
    O.set_eta(0.5)


@pytest.mark.parametrize("eta", [0.2, 0.7])
def test_E2_elastic_net_matches_sklearn_and_gap_identity(eta):
    """sklearn ElasticNet(alpha = lambda, l1_ratio = 1 - eta, fit_intercept = False) minimises the
    same objective (its 1/(2 n_samples) is our 1/(2d)); plain SCD reaches a certified gap and the
    same objective; sum gap_i = O - D with gap_i >= 0 at random states."""
    from sklearn.linear_model import ElasticNet
    O.set_eta(eta)
    d, n, lam = 150, 90, 0.02
    A, b = synth.lasso_dense(d, n, seed=29)
    A64 = A.astype(np.float64).T
    st, alpha, gap, ep = O.solve_scd(O.ELASTIC, A, b, lam, 1e-12, 20000, seed=1)
    assert st == O.OK and gap <= 1e-12
    sk = ElasticNet(alpha=lam, l1_ratio=1 - eta, fit_intercept=False, tol=1e-14, max_iter=200000).fit(A64, b).coef_
    r = A64 @ sk - b
    O_sk = r @ r / (2 * d) + lam * (0.5 * eta * sk @ sk + (1 - eta) * np.abs(sk).sum())
    st, G, Ob, Db = O.duality_gap(O.ELASTIC, A, alpha, b, lam)
    assert Ob <= O_sk + 1e-12 and O_sk - Ob <= 1e-9 * abs(Ob)
    rng = np.random.default_rng(5)
    for _ in range(4):
        a = rng.standard_normal(n) * (rng.random(n) < 0.5) * 0.3
        st, G, Ob, Db = O.duality_gap(O.ELASTIC, A, a, b, lam)
        g = O.coord_gaps(O.ELASTIC, A, a, None, A64 @ a - b, lam)[2]
        assert np.all(g >= 0) and abs(g.sum() - G) <= 1e-12 * G and abs(G - (Ob - Db)) <= 1e-10 * max(1, abs(Ob))
    O.set_eta(0.5)


def test_E3_elastic_step_minimises_1d_objective():
    from scipy.optimize import minimize_scalar
    rng = np.random.default_rng(9)
    for _ in range(100):
        eta = float(rng.uniform(0.05, 0.95))
        O.set_eta(eta)
        d, n = int(rng.integers(2, 50)), int(rng.integers(2, 50))
        nrm, aj, s_ = float(rng.uniform(0.0, 5)), float(rng.normal()), float(rng.normal() * 3)
        lam = float(rng.uniform(0.001, 0.5))
        phi = lambda x: (2 * s_ * (x - aj) + nrm * (x - aj) ** 2) / (2 * d) + lam * (0.5 * eta * x * x + (1 - eta) * abs(x))
        x = O.coord_update(O.ELASTIC, aj, s_, nrm, 0.0, lam, d, n)
        r = minimize_scalar(phi, bounds=(-100, 100), method="bounded", options={"xatol": 1e-10})
        assert phi(x) <= r.fun + 1e-12 and abs(x - r.x) < 1e-6
    O.set_eta(0.5)


# ----------------------------------------------------------------------------- P7 / P8
def test_P7_hadamard_lasso_closed_form_one_epoch():
    """Orthogonal design A^T A = d I: alpha* = soft(A^T b, lam d)/d (north_star pin).
    One sequential epoch in any order reaches it; the gap then vanishes."""
    d, n = 256, 128
    A = synth.hadamard_columns(d, n)
    rng = np.random.default_rng(0)
    b = rng.integers(-3, 4, size=d).astype(np.float64)
    lam = 0.1
    c = A.astype(np.float64) @ b
    astar = np.sign(c) * np.maximum(np.abs(c) - lam * d, 0) / d
    assert np.count_nonzero(astar) > 5
    norms = O.col_norms(A)
    assert np.all(norms == d)
    alpha = np.zeros(n)
    vt = -b.copy()
    O.scd_pass(O.LASSO, A, norms, None, lam, alpha, vt, synth.permutation(np.arange(n), 3))
    np.testing.assert_allclose(alpha, astar, atol=1e-14)
    st, G, Ob, D = O.duality_gap(O.LASSO, A, alpha, b, lam, O.lasso_B(b, lam))
    assert G < 1e-12


def test_P8_orthogonal_sample_svm_closed_form():
    """Orthogonal samples: y_i alpha_i* = clip(lam n/||a_i||^2, 0, 1), one epoch from 0."""
    d, n = 64, 32
    rng = np.random.default_rng(1)
    scales = rng.uniform(0.5, 2.0, n)
    A = synth.hadamard_columns(d, n, scales)
    y = np.where(rng.random(n) < 0.5, -1.0, 1.0)
    for lam in (0.01, 1.0):
        norms = O.col_norms(A)
        beta = np.clip(lam * n / norms, 0, 1)
        alpha = np.zeros(n)
        vt = np.zeros(d)
        O.scd_pass(O.SVM, A, norms, y, lam, alpha, vt, synth.permutation(np.arange(n), 4))
        np.testing.assert_allclose(y * alpha, beta, atol=1e-14)
        st, G, Ob, D = O.duality_gap(O.SVM, A, alpha, y, lam)
        assert G < 1e-13


@pytest.mark.parametrize("model", [O.LASSO, O.SVM])
def test_P7s_P8s_disjoint_support_closed_forms(model):
    """Sparse orthogonal designs (columns on disjoint row sets, a_i^T a_j = 0): the objective
    separates per coordinate, so Lasso alpha_i* = soft(a_i^T b, lam d)/||a_i||^2 and
    SVM y_i alpha_i* = clip(lam n/||a_i||^2, 0, 1), reached by one sequential epoch
    in any order (the pins the asynchronous GPU epochs are held to)."""
    d, n, k = 3000, 500, 6
    cp, rows, vals = synth.disjoint_support_csc(d, n, k, seed=5, scales=np.linspace(0.3, 3.0, n))
    A = synth.csc_to_dense(cp, rows, vals, d)
    A64 = A.astype(np.float64)
    assert np.count_nonzero(np.triu(A64 @ A64.T, 1)) == 0
    norms = O.col_norms(A)
    rng = np.random.default_rng(3)
    if model == O.LASSO:
        b = rng.standard_normal(d)
        lam = 0.2 * np.abs(A64 @ b).max() / d
        c = A64 @ b
        want = np.sign(c) * np.maximum(np.abs(c) - lam * d, 0) / (A64 ** 2).sum(1)
        assert 0 < np.count_nonzero(want) < n
        alpha, vt, lab = np.zeros(n), -b.copy(), b
        O.scd_pass(O.LASSO, A, norms, None, lam, alpha, vt, synth.permutation(np.arange(n), 8))
        np.testing.assert_allclose(alpha, want, rtol=1e-12, atol=1e-15)
    else:
        y = np.where(rng.random(n) < 0.5, -1.0, 1.0)
        lam = 1.0 / n
        beta = np.clip(lam * n / (A64 ** 2).sum(1), 0, 1)
        assert 0 < np.count_nonzero(beta < 1) < n
        alpha, vt, lab = np.zeros(n), np.zeros(d), y
        O.scd_pass(O.SVM, A, norms, y, lam, alpha, vt, synth.permutation(np.arange(n), 8))
        np.testing.assert_allclose(y * alpha, beta, rtol=1e-12, atol=1e-15)
    st, G, Ob, D = O.duality_gap(model, A, alpha, lab, lam, O.lasso_B(lab, lam) if model == O.LASSO else 0.0)
    assert st == O.OK and G < 1e-12


# ----------------------------------------------------------------------------- P9 / P10
def _svm_bruteforce(A64, y, lam):
    """Enumerate beta_i = y_i alpha_i in {0, 1, free}; solve free block stationarity."""
    n = A64.shape[0]
    K = (A64 @ A64.T) * np.outer(y, y)
    best = None
    for pat in itertools.product((0, 1, 2), repeat=n):
        beta = np.array([0.0 if p == 0 else 1.0 for p in pat])
        F = [i for i in range(n) if pat[i] == 2]
        if F:
            NF = [i for i in range(n) if pat[i] != 2]
            rhs = lam * n * np.ones(len(F)) - K[np.ix_(F, NF)] @ beta[NF]
            sol, *_ = np.linalg.lstsq(K[np.ix_(F, F)], rhs, rcond=None)
            if np.linalg.norm(K[np.ix_(F, F)] @ sol - rhs) > 1e-9:
                continue
            if np.any(sol < -1e-12) or np.any(sol > 1 + 1e-12):
                continue
            beta[F] = np.clip(sol, 0, 1)
        alpha = y * beta
        v = A64.T @ alpha
        obj = -(y @ alpha) / n + (v @ v) / (2 * lam * n * n)
        if best is None or obj < best[0]:
            best = (obj, v / (lam * n))
    return best


def test_P9_tiny_svm_bruteforce_optimum():
    rng = np.random.default_rng(9)
    for trial in range(8):
        d, n = int(rng.integers(2, 5)), int(rng.integers(3, 7))
        A = rng.standard_normal((n, d)).astype(np.float32)
        y = np.where(rng.random(n) < 0.5, -1.0, 1.0)
        lam = float(rng.uniform(0.05, 1.0))
        obj_bf, w_bf = _svm_bruteforce(A.astype(np.float64), y, lam)
        st, alpha, gap, ep = O.solve_scd(O.SVM, A, y, lam, 1e-12, 200000, seed=trial)
        assert st == O.OK
        st, G, Ob, D = O.duality_gap(O.SVM, A, alpha, y, lam)
        assert Ob - obj_bf <= 1e-11 and obj_bf - Ob <= G + 1e-12
        w = A.astype(np.float64).T @ alpha / (lam * n)
        np.testing.assert_allclose(w, w_bf, atol=1e-5)


def test_P10_lasso_matches_sklearn_objective():
    """sklearn Lasso(alpha=lam, fit_intercept=False) minimises exactly P:758."""
    from sklearn.linear_model import Lasso
    A, b = synth.lasso_dense(300, 150, seed=31)
    lam = 0.05
    st, alpha, gap, ep = O.solve_scd(O.LASSO, A, b, lam, 1e-10, 5000, seed=2)
    assert st == O.OK
    X = A.astype(np.float64).T
    sk = Lasso(alpha=lam, fit_intercept=False, tol=1e-14, max_iter=200000).fit(X, b)
    obj = lambda a: ((X @ a - b) @ (X @ a - b)) / (2 * len(b)) + lam * np.abs(a).sum()
    assert abs(obj(alpha) - obj(sk.coef_)) <= 1e-9 * obj(sk.coef_)
    # certificate dominates suboptimality: gap >= O(alpha) - O*
    assert gap >= obj(alpha) - obj(sk.coef_) - 1e-12


def test_P10_lambda_max_gives_zero_solution():
    """lam >= ||A^T b||_inf / d => alpha* = 0 and gap(0) = 0."""
    A, b = synth.lasso_dense(50, 30, seed=32)
    lam = np.abs(A.astype(np.float64) @ b).max() / 50 * 1.0001
    st, G, Ob, D = O.duality_gap(O.LASSO, A, np.zeros(30), b, lam, O.lasso_B(b, lam))
    assert G <= 1e-15


# ----------------------------------------------------------------------------- P11
def test_P11_topm_exhaustive_and_ties():
    rng = np.random.default_rng(4)
    for _ in range(60):
        n = int(rng.integers(1, 9))
        m = int(rng.integers(1, n + 1))
        z = rng.integers(0, 4, n).astype(np.float64) * 0.25  # many ties
        P = O.select_topm(z, m)
        best = max(sum(z[list(c)]) for c in itertools.combinations(range(n), m))
        assert abs(z[P].sum() - best) < 1e-15 and len(set(P)) == m
        # tie rule: among optimal sets, the lexicographically lowest indices
        thr = np.sort(z)[::-1][m - 1]
        expect = [i for i in range(n) if z[i] > thr]
        expect += [i for i in range(n) if z[i] == thr][: m - len(expect)]
        assert sorted(P.tolist()) == sorted(expect)
    assert O.select_topm(np.array([3.0, 1, 1, 1]), 2).tolist() == [0, 1]
    # rho >= 1
    g = rng.random(1000)
    P = O.select_topm(g, 100)
    assert g[P].mean() / g.mean() >= 1


def test_baseline_policies():
    """Sequential blocks (P:401, S:318 example) and uniform sampling without replacement."""
    seq = [O.select_policy(O.SEL_SEQUENTIAL, 10, 4, r, 0).tolist() for r in range(4)]
    assert seq == [[0, 1, 2, 3], [4, 5, 6, 7], [8, 9], [0, 1, 2, 3]]
    u = O.select_policy(O.SEL_UNIFORM, 1000, 100, 3, 5)
    assert len(set(u.tolist())) == 100 and u.min() >= 0 and u.max() < 1000
    counts = np.zeros(50)
    for r in range(2000):
        counts[O.select_policy(O.SEL_UNIFORM, 50, 5, r, 9)] += 1
    assert abs(counts.mean() - 200) < 1e-9 and counts.std() < 3 * math.sqrt(200)


def test_importance_sampling_policy():
    """IS baseline: m draws without replacement, the next one with
    probability proportional to ||a_j||^2 among the remaining columns.  Pinned by exact
    successive-sampling inclusion probabilities (enumerated here) against frequencies over
    many rounds, a single nonzero column, and equal norms == uniform inclusion m/n."""
    # one nonzero column is always in the set; zero columns follow by index
    w = np.zeros(10)
    w[5] = 2.0
    for r in range(5):
        assert O.select_policy(O.SEL_IMPORTANCE, 10, 1, r, 3, w).tolist() == [5]
        assert sorted(O.select_policy(O.SEL_IMPORTANCE, 10, 3, r, 3, w).tolist()) == [0, 1, 5]
    # exact inclusion probabilities of successive sampling (m = 1 and m = 2)
    w = np.array([1.0, 2.0, 3.0, 4.0, 10.0])
    Wt = w.sum()
    p1 = w / Wt
    p2 = p1 + np.array([sum(w[k] / Wt * w[i] / (Wt - w[k]) for k in range(5) if k != i) for i in range(5)])
    R = 20000
    for m, p in ((1, p1), (2, p2)):
        cnt = np.zeros(5)
        for r in range(R):
            cnt[O.select_policy(O.SEL_IMPORTANCE, 5, m, r, 11, w)] += 1
        f = cnt / R
        sd = np.sqrt(p * (1 - p) / R)
        assert np.all(np.abs(f - p) < 5 * sd + 1e-12), (m, f, p)
    # a plausible mistake (probabilities proportional to ||a||, or top-m of u * w) fails this:
    assert np.abs(p2 - 2 * np.sqrt(w) / np.sqrt(w).sum()).max() > 0.02
    # equal norms: uniform inclusion m / n
    cnt = np.zeros(40)
    for r in range(2000):
        cnt[O.select_policy(O.SEL_IMPORTANCE, 40, 8, r, 4, np.full(40, 0.7))] += 1
    assert abs(cnt.mean() - 400) < 1e-9 and cnt.std() < 4 * math.sqrt(400 * 0.8)


# ----------------------------------------------------------------------------- generator
def test_counter_generator_is_splitmix64():
    """or_mix64(x) is one splitmix64 step from state x; splitmix64(seed=0) first output."""
    assert O.lib().or_mix64(0) == 0xE220A8397B1DCDAF
    # second output of the splitmix64 stream from 0 = mix(0x9E37..) step
    assert O.lib().or_mix64(0x9E3779B97F4A7C15) == 0x6E789E6AA1B965F4


def test_pass_permutation_is_a_uniform_bijection():
    """Feistel + cycle walking: a bijection of P for every m,
    and positions are uniform over many keys (chi-square), so passes are randomized."""
    for m in (1, 2, 3, 5, 16, 17, 100, 1000, 4097):
        P = np.arange(7, 7 + m) * 3
        p = O.make_perm(P, 5, 1, 2)
        assert sorted(p.tolist()) == P.tolist()
    m = 10
    counts = np.zeros((m, m))
    for r in range(3000):
        p = O.make_perm(np.arange(m), 42, r, 0)
        counts[np.arange(m), p] += 1
    chi2 = ((counts - 300) ** 2 / 300).sum()
    assert chi2 < 81 + 5 * np.sqrt(2 * 81)   # dof (m-1)^2 = 81
    # different passes give different orders
    assert O.make_perm(np.arange(50), 1, 0, 0).tolist() != O.make_perm(np.arange(50), 1, 0, 1).tolist()


# ----------------------------------------------------------------------------- DuHL loop
def test_duhl_full_block_equals_plain_scd():
    """m = n: every round selects [n]; the permutation key matches the plain-SCD epoch."""
    A, b = synth.lasso_dense(100, 60, seed=41)
    lam = 0.05
    r = O.duhl_solve(O.LASSO, A, b, lam, m=60, passes=1, eps=1e-9, max_rounds=200, seed=4)
    st, alpha, gap, ep = O.solve_scd(O.LASSO, A, b, lam, 1e-9, 200, seed=4)
    assert r["status"] == O.OK and st == O.OK and r["rounds"] == ep
    assert np.array_equal(r["alpha"], alpha)


@pytest.mark.parametrize("model", [O.LASSO, O.SVM])
def test_duhl_converges_to_certified_optimum(model):
    if model == O.LASSO:
        A, lab = synth.lasso_dense(200, 400, seed=51)
        lam = 0.05
    else:
        A, lab = synth.svm_dense(30, 400, seed=52)
        lam = 1.0 / 400
    n = A.shape[0]
    res = {}
    for pol in (O.SEL_GAP, O.SEL_SEQUENTIAL, O.SEL_UNIFORM):
        r = O.duhl_solve(model, A, lab, lam, m=n // 4, passes=2, policy=pol,
                         refresh_count=n // 10, eps=1e-6, max_rounds=5000, seed=1)
        assert r["status"] == O.OK and r["gap"] <= 1e-6, (pol, r["gap"])
        st, G, Ob, D = O.duality_gap(model, A, r["alpha"], lab, lam,
                                     O.lasso_B(lab, lam) if model == O.LASSO else 0.0)
        res[pol] = (r["rounds"], Ob, r["swaps"])
        assert r["swaps"][0] == n // 4
    obs = [v[1] for v in res.values()]
    assert max(obs) - min(obs) <= 2e-6
    # gap-based selection needs fewer rounds than the sequential scheme (P:433-435 shape)
    assert res[O.SEL_GAP][0] < res[O.SEL_SEQUENTIAL][0]


def test_rho_definition_pins():
    """rho_{t,P} (Eq. 6): the whole index set gives 1; a uniform gap vector gives 1 for
    every P; averaged over all m-subsets rho is exactly 1 (each j lies in C(n-1,m-1) of the
    C(n,m) subsets); top-m maximises it (Eq. 9) and the complement of top-m minimises it."""
    z = np.array([4.0, 0.0, 1.0, 3.0, 2.0])
    assert O.rho(z, np.arange(5)) == 1.0
    assert abs(O.rho(z, [0]) - 4.0 / 2.0) < 1e-15          # worked: (4/1) / (10/5)
    assert abs(O.rho(z, [0, 3]) - 3.5 / 2.0) < 1e-15
    assert O.rho(np.full(7, 0.3), [2, 5]) == 1.0
    assert O.rho(np.zeros(4), [1]) == 1.0                    # zero gap: no block is preferred
    rng = np.random.default_rng(11)
    for n, m in [(6, 2), (7, 3), (5, 5)]:
        g = rng.random(n)
        vals = [O.rho(g, list(c)) for c in itertools.combinations(range(n), m)]
        assert abs(np.mean(vals) - 1.0) < 1e-13
        assert abs(max(vals) - O.rho(g, O.select_topm(g, m))) < 1e-15
        assert max(vals) >= 1.0 >= min(vals)
