"""The asynchronous TPA-SCD-style dense epoch (cfg.scd_async, csrc/scd_tpa.cu; App. D
P:790-830) against the oracle.

Its order of updates is not fixed (up to scd_block coordinates in flight, atomic fp32 updates
of a shadow of v), so element-wise epoch parity holds only where every interleaving is the
sequential epoch: the P7s/P8s disjoint-support designs (tests/test_oracle_pins.py).  Beyond
them: the exact fp64 resync makes v = A alpha (- b) to rounding after any epoch, and DuHL
with the asynchronous epoch reaches a certified gap and the oracle's optimum."""
import numpy as np
import pytest

import oracle as O
import synth

pytestmark = pytest.mark.gpu


@pytest.fixture(scope="module")
def D():
    import paper_1708_05357_b200 as D
    return D


def _disjoint_dense(d, n, k, seed):
    cp, rows, vals = synth.disjoint_support_csc(d, n, k, seed=seed, scales=np.linspace(0.3, 3.0, n))
    return synth.csc_to_dense(cp, rows, vals, d)


@pytest.mark.parametrize("model", [O.LASSO, O.SVM])
@pytest.mark.parametrize("W", [8, 32, 128])
def test_P7s_P8s_async_dense_epoch(D, model, W):
    """One asynchronous epoch with W coordinates in flight on a disjoint-support design reaches
    the closed forms (fp32 shadow of v: 1e-6 relative, the north_star's fp32-mode bound is 1e-4)
    and the resynced v is exactly A alpha (- b)."""
    d, n, k = 40000, 2000, 20
    A = _disjoint_dense(d, n, k, seed=3 + W)
    A64 = A.astype(np.float64)
    nrm = (A64 ** 2).sum(1)
    rng = np.random.default_rng(W)
    if model == O.LASSO:
        lab = rng.standard_normal(d)
        lam = 0.2 * np.abs(A64 @ lab).max() / d
        c = A64 @ lab
        want = np.sign(c) * np.maximum(np.abs(c) - lam * d, 0) / nrm
    else:
        lab = np.where(rng.random(n) < 0.5, -1.0, 1.0)
        lam = 1.0 / n
        want = lab * np.clip(lam * n / nrm, 0, 1)
    with D.create(A, lab, lam, model, m=n, scd_async=True, scd_block=W) as P:
        name, Wd, G, R = P.scd_shape()   # W is capped by the SMs: W x cluster size <= the grid
        assert name == "k_scd_tpa" and 0 < Wd <= W and G == Wd * ((d + R - 1) // R)
        P.select(D.SEL_GAP, m=n)
        P.scd_epoch(passes=1, seed=2)
        a, v, _ = P.get_state()
    # the step reads s_j = a_j^T v~ with the epoch's own updates in fp32: |s err| <= 1e-6 sum|a v~|
    v0 = -lab if model == O.LASSO else np.zeros(d)
    tol = 1e-6 * (np.abs(A64) @ np.abs(v0)) / nrm + 1e-12 * np.abs(want).max()
    assert np.all(np.abs(a - want) <= tol), np.max(np.abs(a - want) / tol)
    v_exact = O.matvec(A, a) - (lab if model == O.LASSO else 0.0)
    np.testing.assert_allclose(v, v_exact, rtol=0, atol=1e-11 * max(1.0, np.abs(v_exact).max()))


@pytest.mark.parametrize("model", [O.LASSO, O.SVM])
def test_async_epoch_resync_is_exact_on_correlated_data(D, model):
    """After asynchronous epochs on generic data (many interleavings), the state is consistent:
    v = A alpha (- b) to fp64 rounding, SVM box constraints hold."""
    d, n = (3000, 2000) if model == O.LASSO else (4000, 1500)
    A, lab = (synth.lasso_dense(d, n, seed=8) if model == O.LASSO else synth.svm_dense(d, n, seed=8))
    lam = 0.05 if model == O.LASSO else 1.0 / n
    with D.create(A, lab, lam, model, m=n, scd_async=True, scd_block=32) as P:
        P.select(D.SEL_GAP, m=n)
        P.scd_epoch(passes=3, seed=4)
        a, v, _ = P.get_state()
    v_exact = O.matvec(A, a) - (lab if model == O.LASSO else 0.0)
    np.testing.assert_allclose(v, v_exact, rtol=0, atol=1e-10 * max(1.0, np.abs(v_exact).max()))
    if model == O.SVM:
        assert (lab * a).min() >= 0.0 and (lab * a).max() <= 1.0


@pytest.mark.parametrize("model,budget_cols", [(O.LASSO, 0), (O.SVM, 0), (O.LASSO, 300), (O.SVM, 260)])
def test_async_duhl_solve_reaches_the_oracle_optimum(D, model, budget_cols):
    """DuHL rounds with the asynchronous epoch (gamma line search on): certified gap <= eps, the
    oracle certifies the returned alpha, and the objective matches the oracle's optimum to 1e-4."""
    d, n = (400, 1000) if model == O.LASSO else (120, 1000)
    A, lab = (synth.lasso_dense(d, n, seed=21) if model == O.LASSO else synth.svm_dense(d, n, seed=21))
    lam = 0.05 if model == O.LASSO else 1.0 / n
    eps = 1e-6
    with D.create(A, lab, lam, model, hbm_budget_bytes=budget_cols * d * 4, m=250, refresh_fraction=0.05,
                  cert_every=1, seed=5, scd_async=True, scd_block=16) as P:
        r = P.solve(eps, 3000, passes=2)
        a, v, _ = P.get_state()
        g, Ob, Db = P.duality_gap()
    assert r["status"] == 0 and g <= eps
    B = O.lasso_B(lab, lam) if model == O.LASSO else 0.0
    st, G_o, O_o, _ = O.duality_gap(model, A, a, lab, lam, B)
    assert G_o <= 1.01 * eps and abs(O_o - Ob) <= 1e-9 * max(1.0, abs(O_o))
    ref = O.solve_scd(model, A, lab, lam, 1e-9, 20000)
    _, _, O_ref, _ = O.duality_gap(model, A, ref[1], lab, lam, B)
    assert abs(Ob - O_ref) <= 1e-4 * abs(O_ref)


@pytest.mark.parametrize("W", [16, 128])
def test_P7_hadamard_async_converges_to_closed_form(D, W):
    """Hadamard design (A^T A = d I: the Lasso optimum alpha* = soft(A^T b, lambda d)/d is unique,
    P7): the asynchronous epoch is not exact in one pass here (partial column updates are visible
    to the other coordinates), but repeated epochs must reach alpha* (strongly convex problem);
    one pass per epoch, so each reads v~0 exact + only its own pass's fp32 updates."""
    d, n = 2048, 1024
    A = synth.hadamard_columns(d, n)
    rng = np.random.default_rng(0)
    b = rng.integers(-3, 4, size=d).astype(np.float64)
    lam = 0.1
    c = A.astype(np.float64) @ b
    astar = np.sign(c) * np.maximum(np.abs(c) - lam * d, 0) / d
    with D.create(A, b, lam, D.LASSO, m=n, scd_async=True, scd_block=W) as P:
        P.select(D.SEL_GAP, m=n)
        for e in range(25):   # one pass per epoch: each starts from the exactly resynced v
            P.scd_epoch(passes=1, seed=1, round=e)
        a, v, _ = P.get_state()
        g, _, _ = P.duality_gap()
    np.testing.assert_allclose(a, astar, rtol=0, atol=1e-11)
    assert g < 1e-10
