"""GPU edge and degenerate cases of the hot path (empty / ragged inputs,
maximum sizes, the degenerate cases the method has), CUDA path through the C ABI against
the CPU oracle on the same seeded inputs, plus the ABI's documented error behaviour
(include/duhl.h status codes).

Degenerate cases and where the paper fixes their answer:
  * Lasso with lambda >= lambda_max = max_i |a_i^T b| / d: every gap at alpha = 0 is
    (B/d)[|a_i^T b| - lambda d]_+ = 0, so alpha = 0 is certified optimal at once.
  * Lasso with b = 0: B = ||b||^2 / (2 lambda d) = 0 and alpha = 0 is optimal.
  * d = 1 (one row: every column is a scalar, the data maximally collinear), n = 1 (one
    coordinate: a working set of the whole problem), m = n with a budget of exactly m columns.
"""
import numpy as np
import pytest

import oracle as O
import synth

pytestmark = pytest.mark.gpu


@pytest.fixture(scope="module")
def D():
    import paper_1708_05357_b200 as D
    O.set_eta(0.5)
    return D


def _lasso_lmax(A, b, d):
    return np.abs(A[:, :d].astype(np.float64) @ b).max() / d


@pytest.mark.parametrize("factor", [1.0001, 3.0])
def test_lasso_lambda_above_lambda_max_is_optimal_at_zero(D, factor):
    d, n = 3001, 700
    A, b = synth.lasso_dense(d, n, seed=41)
    lam = factor * _lasso_lmax(A, b, d)
    ref = O.duhl_solve(O.LASSO, A, b, lam, m=100, passes=1, refresh_count=10, eps=1e-12,
                       max_rounds=5, cert_every=1, seed=1)
    assert ref["status"] == O.OK and np.all(ref["alpha"] == 0)
    with D.create(A, b, lam, D.LASSO, m=100, cert_every=1, seed=1) as P:
        z0 = P.get_state()[2]
        assert np.all(z0 == 0.0)                   # exact gaps at alpha = 0 (reading: SPEC S:422)
        r = P.solve(1e-12, 5, passes=1)
        a, v, z = P.get_state()
        g, Ob, Db = P.duality_gap()
    assert r["status"] == 0 and r["rounds"] <= ref["rounds"]
    assert np.all(a == 0.0) and g == 0.0
    np.testing.assert_allclose(v, -b, rtol=0, atol=0)                 # v~ = A alpha - b
    assert abs(Ob - (b @ b) / (2 * d)) <= 1e-12 * (b @ b) / (2 * d)   # O(0) = ||b||^2 / 2d


def test_lasso_zero_labels(D):
    d, n = 517, 300
    A, _ = synth.lasso_dense(d, n, seed=42)
    b = np.zeros(d)
    with D.create(A, b, 0.1, D.LASSO, m=64, cert_every=1, seed=1) as P:
        g, s = P.gaps(want_s=True)
        assert np.all(s == 0.0) and np.all(g == 0.0)
        r = P.solve(1e-12, 3, passes=1)
        a, v, z = P.get_state()
    assert r["status"] == 0 and np.all(a == 0.0) and np.all(v == 0.0)


@pytest.mark.parametrize("model", [O.LASSO, O.SVM, O.RIDGE])
def test_single_row_gaps_and_epoch(D, model):
    """d = 1: one row (d % 4 = 1, a single row tile with a ragged tail)."""
    d, n, m = 1, 333, 300
    if model == O.SVM:
        A, lab = synth.svm_dense(d, n, seed=43)
        lam = 1.0 / n
    else:
        A, lab = synth.lasso_dense(d, n, seed=43)
        lam = 0.01
    y = lab if model == O.SVM else None
    order = synth.permutation(np.arange(m), 3)
    with D.create(A, lab, lam, model, m=m) as P:
        g0, s0 = P.gaps(want_s=True)
        P.select(D.SEL_SEQUENTIAL, m=m, round=0)
        P.scd_epoch(perm=order)
        a_gpu, v_gpu, _ = P.get_state()
        g1, s1 = P.gaps(want_s=True)
    alpha = np.zeros(n)
    vt = -lab.copy() if model != O.SVM else np.zeros(d)
    # oracle gaps at alpha = 0
    w0 = O.primal_dual_w(model, np.zeros(d), lab if model != O.SVM else None, n, lam)   # v = A 0
    B = O.lasso_B(lab, lam) if model == O.LASSO else 0.0
    st, s_or, g_or = (O.coord_gaps(model, A, alpha, None, w0, lam, B, d=d) if model != O.SVM
                      else O.coord_gaps(O.SVM, A, alpha, lab, w0, lam, d=d))
    np.testing.assert_allclose(s0, s_or, rtol=1e-12, atol=1e-300)
    np.testing.assert_allclose(g0, g_or, rtol=1e-12, atol=1e-300)
    O.scd_pass(model, A, O.col_norms(A), y, lam, alpha, vt, order)
    assert np.abs(a_gpu - alpha).max() <= 1e-11 * max(1e-300, np.abs(alpha).max())
    assert np.abs(v_gpu - vt).max() <= 1e-11 * max(1.0, np.abs(vt).max())
    # gaps at the post-epoch state: oracle from its own v
    v_or = O.matvec(A, alpha, d=d)
    w = O.primal_dual_w(model, v_or, lab if model != O.SVM else None, n, lam)
    st, s_or, g_or = (O.coord_gaps(model, A, alpha, None, w, lam, B, d=d) if model != O.SVM
                      else O.coord_gaps(O.SVM, A, alpha, lab, w, lam, d=d))
    # conditioning floor: |a_i| times the scale of w, here w at alpha = 0 (the ridge
    # residual after one pass on one row is ~1e-83 on both sides)
    sc = np.abs(A[:, 0]).astype(np.float64) * max(np.abs(w).max(), np.abs(w0).max())
    assert np.all(np.abs(s1 - s_or) <= 1e-9 * np.maximum(np.abs(s_or), sc) + 1e-300)


def test_single_row_svm_solve(D):
    d, n = 1, 60
    A, y = synth.svm_dense(d, n, seed=4)
    lam = 1.0 / n
    ref = O.duhl_solve(O.SVM, A, y, lam, m=10, passes=2, refresh_count=5, eps=1e-8,
                       max_rounds=2000, cert_every=1, seed=1)
    assert ref["status"] == O.OK
    with D.create(A, y, lam, D.SVM_DUAL, m=10, refresh_fraction=5 / n, cert_every=1, seed=1) as P:
        r = P.solve(1e-8, 2000, passes=2)
        g, Ob, Db = P.duality_gap()
    assert r["status"] == 0 and g <= 1e-8
    st, G_ref, O_ref, _ = O.duality_gap(O.SVM, A, ref["alpha"], y, lam, 0.0)
    assert abs(Ob - O_ref) <= 1e-4 * abs(O_ref)


@pytest.mark.parametrize("model", [O.LASSO, O.SVM])
def test_single_column(D, model):
    """n = 1, m = 1: one coordinate; one exact step reaches the 1-D minimiser (App. D)."""
    d, n = 1003, 1
    if model == O.SVM:
        A, lab = synth.svm_dense(d, n, seed=44)
        lam = 0.5
    else:
        A, lab = synth.lasso_dense(d, n, seed=44)
        lam = 0.01
    ref = O.duhl_solve(model, A, lab, lam, m=1, passes=1, refresh_count=1, eps=1e-12,
                       max_rounds=20, cert_every=1, seed=1)
    with D.create(A, lab, lam, model, m=1, cert_every=1, seed=1) as P:
        r = P.solve(1e-12, 20, passes=1)
        a, v, z = P.get_state()
        g, Ob, Db = P.duality_gap()
    assert r["status"] == ref["status"] == 0
    np.testing.assert_allclose(a, ref["alpha"], rtol=1e-12, atol=1e-300)
    assert g <= 1e-12


@pytest.mark.parametrize("model", [O.LASSO, O.SVM])
def test_working_set_is_everything_under_an_exact_budget(D, model):
    """m = n with an HBM budget of exactly n columns: the maximum working set (no swaps
    after the cold fill)."""
    d, n = 257, 400
    if model == O.SVM:
        A, lab = synth.svm_dense(d, n, seed=45)
        lam = 1.0 / n
    else:
        A, lab = synth.lasso_dense(d, n, seed=45)
        lam = 0.05
    col_bytes = ((d + 3) // 4) * 16
    ref = O.duhl_solve(model, A, lab, lam, m=n, passes=1, refresh_count=0, eps=1e-7,
                       max_rounds=500, cert_every=1, seed=2)
    with D.create(A, lab, lam, model, hbm_budget_bytes=n * col_bytes, m=n, refresh_fraction=0.0,
                  cert_every=1, seed=2) as P:
        r = P.solve(1e-7, 500, passes=1)
    assert r["status"] == 0 and ref["status"] == O.OK
    sw = [t.swaps for t in r["trace"]]
    assert sw[0] == n and all(s == 0 for s in sw[1:])
    k = min(5, len(r["trace"]), len(ref["gaps"]))
    np.testing.assert_allclose([t.cert_gap for t in r["trace"]][:k], ref["gaps"][:k], rtol=1e-8)


# ------------------------------------------------------------ documented error behaviour
def test_invalid_arguments_are_rejected(D):
    d, n = 64, 50
    A, b = synth.lasso_dense(d, n, seed=46)
    Ay, y = synth.svm_dense(d, n, seed=46)
    bad = A.copy()
    bad[3, 5] = np.nan
    cases = [
        lambda: D.create(A, b, 0.0, D.LASSO),                      # lambda <= 0
        lambda: D.create(A, b, -1.0, D.LASSO),
        lambda: D.create(bad, b, 0.1, D.LASSO),                    # non-finite data
        lambda: D.create(Ay, y * 2.0, 1.0 / n, D.SVM_DUAL),             # y not +-1
        lambda: D.create(A, b, 0.1, D.LASSO, m=n + 1),             # m > n
        lambda: D.create(A, b, 0.1, D.LASSO, hbm_budget_bytes=16, m=10),  # budget < m columns
    ]
    for c in cases:
        with pytest.raises(D.DuhlError) as e:
            P = c()
            P.close()
        assert e.value.status == 2, (e.value.status, str(e.value))   # DUHL_E_INVALID
    with D.create(A, b, 0.1, D.LASSO, m=10) as P:
        with pytest.raises(D.DuhlError) as e:
            P.select(D.SEL_GAP, m=n + 1)
        assert e.value.status == 2
        with pytest.raises(D.DuhlError) as e:
            P.gaps(np.array([0, n]))                                 # index out of range
        assert e.value.status == 2
        P.gaps()                                                     # the handle is still usable


def test_c_program_solves_P1(tmp_path):
    """tests/c/abi_check.c, a plain C caller of include/duhl.h: solves the P1 worked example
    (alpha* = (1/2, 1/2), O* = 0.375) through duhl_solve with a trace callback."""
    import subprocess
    from test_abi import _build_abi_check
    exe = _build_abi_check(tmp_path)
    r = subprocess.run([exe, "1"], capture_output=True, text=True, timeout=300)
    assert r.returncode == 0, r.stdout + r.stderr
