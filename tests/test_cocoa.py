"""Multi-GPU aggregation (R16) on the CPU.

* the oracle's exact line search on gamma is pinned by brute force;
* K = 1 without line search reduces exactly to Algorithm 2 (or_duhl_solve);
* a world_size-2 gloo run -- two processes, each owning a column shard, composing
  the round from oracle primitives with a real torch.distributed all_reduce of
  dv -- reproduces the single-process K = 2 oracle (or_duhl_solve_cocoa) bit for
  bit.  That validates the sharded semantics the CUDA path implements with
  ncclAllReduce (one NCCL process per GPU).
"""
import os

import numpy as np
import pytest

import oracle as O
import synth


def _objective(model, A, lab, lam, alpha):
    A64 = A.astype(np.float64)
    n, d = A64.shape
    v = A64.T @ alpha
    if model == O.LASSO:
        return ((v - lab) @ (v - lab)) / (2 * d) + lam * np.abs(alpha).sum()
    if model == O.RIDGE:
        return ((v - lab) @ (v - lab)) / (2 * d) + 0.5 * lam * (alpha @ alpha)
    if model == O.ELASTIC:  # P:796-800 with eta = 0.5 (O.set_eta)
        return ((v - lab) @ (v - lab)) / (2 * d) + lam * (0.25 * (alpha @ alpha) + 0.5 * np.abs(alpha).sum())
    return -(lab @ alpha) / n + (v @ v) / (2 * lam * n * n)


@pytest.mark.parametrize("model", [O.LASSO, O.SVM, O.RIDGE, O.ELASTIC])
def test_linesearch_is_the_exact_minimiser(model):
    O.set_eta(0.5)
    rng = np.random.default_rng(5)
    for trial in range(20):
        if model in (O.LASSO, O.RIDGE, O.ELASTIC):
            A, lab = synth.lasso_dense(40, 30, seed=trial)
            lam = 0.05
            a0 = rng.standard_normal(30) * (rng.random(30) < 0.5) * 0.2
            a1 = rng.standard_normal(30) * (rng.random(30) < 0.5) * 0.2
        else:
            A, lab = synth.svm_dense(20, 30, seed=trial)
            lam = 0.02
            a0 = lab * rng.random(30)
            a1 = lab * rng.random(30)
        A64 = A.astype(np.float64)
        v0 = A64.T @ a0 - (lab if model != O.SVM else 0)
        dv = A64.T @ (a1 - a0)
        idx = np.arange(30)
        g = O.linesearch(model, v0, dv, a0[idx], (a1 - a0)[idx],
                         lab if model == O.SVM else None, lam, 30)
        assert 0.0 <= g <= 1.0
        grid = np.linspace(0, 1, 2001)
        f = [_objective(model, A, lab, lam, a0 + t * (a1 - a0)) for t in grid]
        fg = _objective(model, A, lab, lam, a0 + g * (a1 - a0))
        assert fg <= min(f) + 1e-12 * max(1, abs(min(f)))


def test_cocoa_k1_without_linesearch_is_algorithm_2():
    A, b = synth.lasso_dense(150, 300, seed=61)
    r1 = O.duhl_solve(O.LASSO, A, b, 0.05, m=75, passes=2, refresh_count=30, eps=1e-6,
                      max_rounds=500, seed=3)
    r2 = O.duhl_solve_cocoa(O.LASSO, A, b, 0.05, m=75, K=1, linesearch=False, passes=2,
                            refresh_count=30, eps=1e-6, max_rounds=500, seed=3)
    assert r1["rounds"] == r2["rounds"] and np.array_equal(r1["alpha"], r2["alpha"])


@pytest.mark.parametrize("model", [O.LASSO, O.SVM])
def test_cocoa_shards_converge_with_linesearch(model):
    if model == O.LASSO:
        A, lab = synth.lasso_dense(200, 400, seed=62)
        lam = 0.05
    else:
        A, lab = synth.svm_dense(30, 400, seed=63)
        lam = 1 / 400
    for K in (2, 4):
        r = O.duhl_solve_cocoa(model, A, lab, lam, m=100 // K, K=K, linesearch=True, passes=2,
                               refresh_count=40 // K, eps=1e-6, max_rounds=5000, seed=1)
        assert r["status"] == O.OK and r["gap"] <= 1e-6
        assert np.all((r["gammas"] >= 0) & (r["gammas"] <= 1))


# ------------------------------------------------------------------ world_size-2 gloo run
def _shard_round_worker(rank, world, port, model, A, lab, lam, m, passes, refresh, rounds, seed, out):
    """One rank: the K-shard DuHL round of or_duhl_solve_cocoa composed from oracle
    primitives; dv is summed with torch.distributed (gloo) and the line-search
    inputs are all-gathered."""
    import torch
    import torch.distributed as dist
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    n, d = A.shape
    lo, hi = rank * n // world, (rank + 1) * n // world
    nk = hi - lo
    y = lab if model == O.SVM else None
    b = lab if model == O.LASSO else None
    B = O.lasso_B(b, lam) if model == O.LASSO else 0.0
    norms = O.col_norms(A)
    alpha = np.zeros(n)                     # only columns [lo, hi) are ever written here
    vt = -b.copy() if model == O.LASSO else np.zeros(d)
    w = O.primal_dual_w(model, vt + (b if b is not None else 0), b, n, lam)
    z = O.coord_gaps(model, A, alpha, y, w, lam, B)[2]
    cursor = 0
    for t in range(rounds):
        P = np.sort(O.select_topm(z[lo:hi], m)) + lo
        w = vt if model == O.LASSO else vt / (lam * n)
        kr = min(refresh, nk)
        idx = lo + (cursor + np.arange(kr)) % nk
        cursor = (cursor + kr) % nk
        if kr:
            z[idx] = O.coord_gaps(model, A, alpha, y, w, lam, B, idx=idx)[2]
        v0 = vt.copy()
        aold = alpha[P].copy()
        vk = v0.copy()
        for p in range(passes):
            O.scd_pass(model, A, norms, y, lam, alpha, vk, O.make_perm(P, seed, t, p))
        dv_t = torch.from_numpy(vk - v0)
        dist.all_reduce(dv_t)
        dv = dv_t.numpy()
        parts = [None] * world
        dist.all_gather_object(parts, (aold, alpha[P] - aold, lab[P] if model == O.SVM else None))
        a_all = np.concatenate([p[0] for p in parts])
        da_all = np.concatenate([p[1] for p in parts])
        y_all = np.concatenate([p[2] for p in parts]) if model == O.SVM else None
        g = O.linesearch(model, v0, dv, a_all, da_all, y_all, lam, n)
        vt = v0 + g * dv
        alpha[P] = aold + g * (alpha[P] - aold)
        w = vt if model == O.LASSO else vt / (lam * n)
        z[P] = O.coord_gaps(model, A, alpha, y, w, lam, B, idx=P)[2]
    out[rank] = alpha[lo:hi].copy()
    dist.destroy_process_group()


@pytest.mark.parametrize("model", [O.LASSO, O.SVM])
def test_gloo_two_ranks_match_oracle_cocoa(model):
    import multiprocessing as mp
    import socket
    if model == O.LASSO:
        A, lab = synth.lasso_dense(120, 240, seed=64)
        lam = 0.05
    else:
        A, lab = synth.svm_dense(24, 240, seed=65)
        lam = 1 / 240
    m, passes, refresh, rounds, seed = 30, 2, 12, 6, 4
    ref = O.duhl_solve_cocoa(model, A, lab, lam, m=m, K=2, linesearch=True, passes=passes,
                             refresh_count=refresh, eps=0.0, max_rounds=rounds, cert_every=0,
                             seed=seed)   # no certificates: they would refresh z (R25)
    with socket.socket() as s:
        s.bind(("127.0.0.1", 0))
        port = s.getsockname()[1]
    ctx = mp.get_context("spawn")
    with ctx.Manager() as man:
        out = man.dict()
        procs = [ctx.Process(target=_shard_round_worker,
                             args=(r, 2, port, model, A, lab, lam, m, passes, refresh, rounds, seed, out))
                 for r in range(2)]
        for p in procs:
            p.start()
        for p in procs:
            p.join(timeout=120)
            assert p.exitcode == 0
        alpha = np.concatenate([out[0], out[1]])
    np.testing.assert_array_equal(alpha, ref["alpha"])
