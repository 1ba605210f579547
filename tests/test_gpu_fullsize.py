"""Parity at BASELINE.json's full sizes, in the launch configuration bench.py times.

test_bench_launch_rounds_replay_oracle: the bench's own options (bench.parse_args +
bench.launch_kwargs: fast-mode SCD, k_scd_ser W = 12 on 140 CTAs at C4 / k_scd_pipe W = 32
with tensor-core Gram tiles at C3, 8 unit-A refresh CTAs, host unit-A threads, passes per
round) for the first rounds from alpha = 0, each round replayed by the oracle on the device's
(band-verified) working set (oracle/replay.py): alpha and v element-wise, the certificate.

C4 (hinge-SVM dual, 200,704 x 40,000 fp32 = 32.1 GB in pinned host memory) and C3 (Lasso,
40,000 x 200,704) under the 8.03 GB HBM budget, m, passes, refresh and SCD mode of the bench
(fast mode: fp32 Gram products inside a warp).  After a few DuHL rounds (Alg. 2)
the device state is checked against the oracle on what it can compute at this size:

* v = A alpha (- b): the oracle's matvec over the columns alpha touches (exact definition);
* a2 gap pass: gap_i and s_i = a_i^T w of sampled columns (ragged tail included) against the
  oracle's coord_gaps at the same alpha (Eq. 4, P:852 / P:867), north_star tolerance;
* a7 certificate: the total duality gap and the objective against the oracle's;
* properties that hold at any size: SVM box y_i alpha_i in [0, 1], z >= 0, rho >= 1 for the
  gap-selected sets (Eq. 9), swaps(first round) = m, the objective decreases from alpha = 0.
"""
import gc

import numpy as np
import pytest

import bench
import oracle as O
from oracle.replay import Alg2

pytestmark = pytest.mark.gpu

TOL = 1e-6


@pytest.fixture(scope="module")
def D():
    import paper_1708_05357_b200 as D
    return D


@pytest.mark.parametrize("name", ["c4", "c3"])
def test_full_size_rounds_against_oracle(D, name):
    cfg = bench.CONFIGS[name]
    d, n, model = cfg["d"], cfg["n"], cfg["model"]
    A, lab = bench.make_data(cfg, 170805357 + 3)
    lam = bench.lam_of(cfg, A, lab)
    col_bytes = ((d + 3) // 4) * 16
    budget = int(cfg["budget_frac"] * n * col_bytes)
    m = cfg["m"]
    args, _ = bench.parse_args(["--config", name])
    kw = bench.launch_kwargs(args, cfg)   # the bench's launch (C3: the asynchronous epoch)
    with D.create(A, lab, lam, model, cert_every=1 << 40, scd_exact=False, **kw) as P:
        recs = [P.round(t, passes=cfg["passes"]) for t in range(3)]
        a, v, z = P.get_state()
        rng = np.random.default_rng(5)
        idx = np.unique(np.concatenate([rng.choice(n, 62, replace=False), [0, n - 1]]))
        g_gpu, s_gpu = P.gaps(idx, want_s=True)
        G, Ob, Db = P.duality_gap()
    assert recs[0].swaps == m and all(r.rho >= 1.0 - 1e-12 for r in recs)
    assert np.all(z >= 0) and np.all(np.isfinite(a))
    if model == O.SVM:
        ya = lab * a
        assert ya.min() >= 0.0 and ya.max() <= 1.0
    assert np.count_nonzero(a) > 0
    # v = A alpha (- b): the oracle's matvec (skips alpha_i = 0)
    v_or = O.matvec(A, a)
    if model == O.LASSO:
        v_or = v_or - lab
    scale = np.abs(A[np.flatnonzero(a)]).max() * np.abs(a).sum()
    assert np.max(np.abs(v - v_or)) <= 1e-9 * scale
    # sampled gap pass
    w = O.primal_dual_w(model, v_or + (lab if model == O.LASSO else 0.0),
                        lab if model == O.LASSO else None, n, lam)
    B = O.lasso_B(lab, lam) if model == O.LASSO else 0.0
    st, s_or, g_or = O.coord_gaps(model, A, a, lab if model == O.SVM else None, w, lam, B, idx=idx)
    An = np.linalg.norm(A[idx].astype(np.float64), axis=1)
    floor = 1e-3 * An * np.linalg.norm(w)
    assert np.all(np.abs(s_gpu - s_or) <= TOL * np.maximum(np.abs(s_or), floor))
    c = (np.abs(a[idx]) + B) / d if model == O.LASSO else (np.abs(a[idx]) + 1) / n
    assert np.all(np.abs(g_gpu - g_or) <= TOL * np.maximum(np.abs(g_or), 1e-3 * c * An * np.linalg.norm(w)))
    # certificate (a7) against the oracle's full pass
    st, G_or, O_or, D_or = O.duality_gap(model, A, a, lab, lam, B)
    assert st == O.OK
    assert abs(Ob - O_or) <= 1e-9 * max(1.0, abs(O_or))
    assert abs(G - G_or) <= TOL * max(G_or, 1e-12)
    O0 = 0.0 if model == O.SVM else float(lab @ lab) / (2 * d)   # objective at alpha = 0
    assert Ob < O0
    del A
    gc.collect()


@pytest.mark.parametrize("name,rounds", [("c4", 3), ("c3", 2)])
def test_bench_launch_rounds_replay_oracle(D, name, rounds):
    """C4: the bench's exact launch.  C3's bench launch is the asynchronous epoch, whose order is
    not reproducible; its exact kernel (k_scd_pipe, W = 32, tensor-core Gram tiles, fast mode) is
    replayed here and the asynchronous launch is held to the invariants of
    test_full_size_rounds_against_oracle."""
    args, cfg = bench.parse_args(["--config", name])
    kw = dict(bench.launch_kwargs(args, cfg), scd_async=False)
    d, n, model = cfg["d"], cfg["n"], cfg["model"]
    A, lab = bench.make_data(cfg, kw["seed"])
    lam = bench.lam_of(cfg, A, lab)
    m, passes = kw["m"], args.passes
    R = Alg2(model, A, lab, lam, m, passes, int(np.ceil(args.refresh * n - 1e-9)), kw["seed"])
    with D.create(A, lab, lam, model, cert_every=1 << 40, scd_exact=args.exact, **kw) as P:
        shape = P.scd_shape()
        assert shape[0] == ("k_scd_ser" if name == "c4" else "k_scd_pipe")
        for t in range(rounds):
            rec = P.round(t, passes=passes, certify=(t == rounds - 1))
            Pd = P.working_set()
            R.check_selection([Pd], O.SEL_GAP, t, tol=1e-4)   # fast mode: the fp32-mode tolerance
            rr = R.round(t, [Pd], certify=(t == rounds - 1))
            assert rec.swaps == rr["swaps"], (t, rec.swaps, rr["swaps"])
        a, v, _ = P.get_state()
        cols, share = P.unit_a_host()
    if args.unit_a_host > 0:
        assert cols > 0                                  # the host threads took part of unit A
    sa = np.abs(R.alpha).max()
    assert np.abs(a - R.alpha).max() <= 1e-6 * sa, np.abs(a - R.alpha).max() / sa
    assert np.abs(v - R.vt).max() <= 1e-6 * max(1.0, np.abs(R.vt).max())
    assert abs(rec.cert_gap - rr["gap"]) <= 1e-6 * rr["gap"], (rec.cert_gap, rr["gap"])
    del A
    gc.collect()


@pytest.mark.parametrize("name", ["c1", "c2"])
def test_c1_c2_bench_launch_replay_to_eps(D, name):
    """C1 (Lasso 2000 x 1000, lambda = 0.1, m = 25 %) and C2 (SVM dual 500 x 20,000, m = 10 %) at
    their full shapes in the bench's launch configuration: every round until the certified gap
    <= 1e-5 is replayed by the oracle on the device's band-verified working set; certificates
    to 1e-8, the final alpha to 1e-9 of its largest entry (exact SCD kernels, fp64)."""
    args, cfg = bench.parse_args(["--config", name, "--exact"])
    kw = bench.launch_kwargs(args, cfg)
    A, lab = bench.make_data(cfg, kw["seed"])
    lam = bench.lam_of(cfg, A, lab)
    n = cfg["n"]
    R = Alg2(cfg["model"], A, lab, lam, kw["m"], args.passes, int(np.ceil(args.refresh * n - 1e-9)), kw["seed"])
    with D.create(A, lab, lam, cfg["model"], cert_every=1, scd_exact=True, **kw) as P:
        for t in range(400):
            rec = P.round(t, passes=args.passes, certify=True)
            Pd = P.working_set()
            R.check_selection([Pd], O.SEL_GAP, t)
            rr = R.round(t, [Pd])
            assert abs(rec.cert_gap - rr["gap"]) <= 1e-8 * rr["gap"] + 1e-13, (t, rec.cert_gap, rr["gap"])
            if rec.cert_gap <= 1e-5:
                break
        a, _, _ = P.get_state()
    assert rec.cert_gap <= 1e-5, (t, rec.cert_gap)
    assert np.abs(a - R.alpha).max() <= 1e-9 * max(1e-300, np.abs(R.alpha).max())
