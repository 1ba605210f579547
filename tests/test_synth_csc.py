"""The sparse (C5) input generator: counter-based, shard-consistent, Bernoulli pattern
(nnz_i ~ Binomial(d, 0.01), rows uniform without replacement, sorted)."""
import numpy as np

import synth


def test_csc_pattern_is_bernoulli_and_sorted():
    d, n, p = 20000, 4000, 0.01
    cp, rows, vals = synth.csc_lasso(d, n, seed=11, density=p)
    cnt = np.diff(cp)
    assert cp[0] == 0 and cp[-1] == rows.size == vals.size
    mean, var = d * p, d * p * (1 - p)
    assert abs(cnt.mean() - mean) < 4 * np.sqrt(var / n)
    assert 0.85 * var < cnt.var() < 1.15 * var
    for i in range(0, n, 97):
        r = rows[cp[i]:cp[i + 1]]
        assert np.all(np.diff(r) > 0) and (r.size == 0 or (r[0] >= 0 and r[-1] < d))
    # rows uniform: chi-square over 20 row bins
    h = np.bincount(rows * 20 // d, minlength=20)
    e = rows.size / 20
    assert ((h - e) ** 2 / e).sum() < 45.3  # chi2(19) 0.999 quantile
    assert abs(vals.astype(np.float64).mean()) < 0.01 and abs(vals.astype(np.float64).std() - 1) < 0.01


def test_csc_shards_regenerate_independently():
    d, n = 5000, 3000
    cp, rows, vals = synth.csc_lasso(d, n, seed=3)
    for lo, hi in [(0, 256), (100, 900), (2999, 3000), (700, 3000)]:
        c2, r2, v2 = synth.csc_lasso(d, n, seed=3, col_lo=lo, col_hi=hi)
        assert np.array_equal(np.diff(cp[lo:hi + 1]), np.diff(c2))
        assert np.array_equal(rows[cp[lo]:cp[hi]], r2) and np.array_equal(vals[cp[lo]:cp[hi]], v2)


def test_csc_to_dense_and_signal():
    d, n = 300, 200
    cp, rows, vals = synth.csc_lasso(d, n, seed=9, density=0.05)
    A = synth.csc_to_dense(cp, rows, vals, d)
    assert A.shape == (n, d) and np.count_nonzero(A) == rows.size
    sig = synth.csc_lasso_signal(cp, rows, vals, d, seed=9, support=0.1)
    at = synth.lasso_truth(n, 9, 0.1)
    np.testing.assert_allclose(sig, A.astype(np.float64).T @ at, rtol=1e-12, atol=1e-12)
