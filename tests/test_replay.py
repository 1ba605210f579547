"""The oracle replay (oracle/replay.py) composes the oracle's primitives in the order of
or_duhl_solve / or_duhl_solve_cocoa: fed the oracle's own selections it must reproduce those
loops exactly, and its band check must accept every valid top-m and reject invalid ones."""
import numpy as np
import pytest

import oracle as O
import synth
from oracle.replay import Alg2


def _data(model, d, n, seed):
    if model == O.SVM:
        return synth.svm_dense(d, n, seed=seed)
    return synth.lasso_dense(d, n, seed=seed)


def _own_sets(R, policy, t):
    out = []
    for k in range(R.K):
        lo, hi = R.shard(k)
        zk = R.norms[lo:hi] if policy == O.SEL_IMPORTANCE else R.z[lo:hi]
        out.append(np.sort(O.select_policy(policy, hi - lo, R.m, t, R.seed, zk)) + lo)
    return out


@pytest.mark.parametrize("model,policy", [(O.LASSO, O.SEL_GAP), (O.SVM, O.SEL_GAP), (O.RIDGE, O.SEL_GAP),
                                          (O.SVM, O.SEL_SEQUENTIAL), (O.LASSO, O.SEL_UNIFORM)])
def test_replay_reproduces_or_duhl_solve(model, policy):
    d, n, m = (150, 400, 100) if model != O.SVM else (60, 400, 100)
    A, lab = _data(model, d, n, 31)
    lam = 0.05 if model == O.LASSO else (0.02 if model == O.RIDGE else 1.0 / n)
    R0 = 12
    ref = O.duhl_solve(model, A, lab, lam, m=m, passes=2, policy=policy, refresh_count=30, eps=0.0,
                       max_rounds=R0, cert_every=1, seed=5)
    R = Alg2(model, A, lab, lam, m, 2, 30, 5)
    for t in range(R0):
        P = _own_sets(R, policy, t)
        R.check_selection(P, policy, t)
        r = R.round(t, P)
        assert r["gap"] == ref["gaps"][t] and r["swaps"] == ref["swaps"][t]
    np.testing.assert_array_equal(R.alpha, ref["alpha"])
    np.testing.assert_array_equal(R.z, ref["z"])


@pytest.mark.parametrize("model,K", [(O.LASSO, 1), (O.SVM, 2), (O.LASSO, 3), (O.ELASTIC, 2)])
def test_replay_reproduces_or_duhl_solve_cocoa(model, K):
    O.set_eta(0.5)
    d, n, m = (120, 600, 60) if model != O.SVM else (50, 600, 60)
    A, lab = _data(model, d, n, 32)
    lam = 0.05 if model == O.LASSO else (0.03 if model == O.ELASTIC else 1.0 / n)
    R0 = 8
    ref = O.duhl_solve_cocoa(model, A, lab, lam, m=m, K=K, linesearch=True, passes=2, refresh_count=20,
                             eps=0.0, max_rounds=R0, cert_every=1, seed=9)
    R = Alg2(model, A, lab, lam, m, 2, 20, 9, K=K, linesearch=True)
    for t in range(R0):
        P = _own_sets(R, O.SEL_GAP, t)
        R.check_selection(P, O.SEL_GAP, t)
        r = R.round(t, P)
        assert r["gap"] == ref["gaps"][t] and r["gamma"] == ref["gammas"][t]
    np.testing.assert_array_equal(R.alpha, ref["alpha"])


def test_band_check_accepts_ties_and_rejects_violations():
    """Near-ties inside the band may go either way; a coordinate clearly above the m-th
    largest gap must be in P, one clearly below must not."""
    d, n, m = 80, 300, 50
    A, b = synth.lasso_dense(d, n, seed=3)
    R = Alg2(O.LASSO, A, b, 0.05, m, 1, 0, 1)
    for t in range(3):
        R.round(t, _own_sets(R, O.SEL_GAP, t))
    order = np.lexsort((np.arange(n), -R.z))
    P = np.sort(order[:m])
    R.check_selection([P], O.SEL_GAP, 3)
    # perturb z within the band at the boundary: either order is accepted
    tau = R._tau(np.arange(n))
    z0 = R.z.copy()
    i_in, i_out = order[m - 1], order[m]
    if abs(z0[i_in] - z0[i_out]) <= min(tau[i_in], tau[i_out]):
        P2 = np.sort(np.r_[order[:m - 1], i_out])
        R.check_selection([P2], O.SEL_GAP, 3)
    # a clear violation: swap the largest gap for the smallest
    if z0[order[0]] > z0[order[-1]] + tau[order[0]] + tau[order[-1]]:
        P3 = np.sort(np.r_[order[1:m], order[-1]])
        with pytest.raises(AssertionError):
            R.check_selection([P3], O.SEL_GAP, 3)
    # wrong size
    with pytest.raises(AssertionError):
        R.check_selection([P[:-1]], O.SEL_GAP, 3)
