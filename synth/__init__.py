"""Seeded synthetic inputs shared by the oracle tests and the CUDA path.

This module holds NONE of DuHL's arithmetic (no gaps, updates, selection or
objectives): it only draws data matrices, labels and permutations, with the
shapes and value distributions of the paper's workloads (DESIGN.md "Input
recipe").

Randomness is counter-based: column block ``k`` (``BLOCK`` columns) of a matrix
is drawn from ``numpy.random.Philox(key=[seed, k])``, so any block regenerates
independently of the others -- a rank of a sharded run draws only its own
columns, and a bounded oracle sample can redraw a handful of columns.

Layout convention everywhere: a d x n column-major float32 matrix is stored as a
C-contiguous numpy array of shape (n, ld), ld >= d; row i is column a_i.
"""
from __future__ import annotations

import math
import os
from concurrent.futures import ThreadPoolExecutor

import numpy as np

BLOCK = 256          # columns per counter-based RNG block
SEED0 = 170805357    # seed 170805357 + config index


def _rng(seed: int, block: int, stream: int = 0) -> np.random.Generator:
    return np.random.Generator(np.random.Philox(key=[(seed + (stream << 40)) & ((1 << 64) - 1),
                                                     block & ((1 << 64) - 1)]))


def _normal_into(r: np.random.Generator, X: np.ndarray) -> None:
    if X.flags.c_contiguous:
        r.standard_normal(out=X, dtype=np.float32)
    else:
        for q in range(X.shape[0]):
            X[q] = r.standard_normal(X.shape[1], dtype=np.float32)


def _threads(nblocks: int) -> int:
    return max(1, min(nblocks, os.cpu_count() or 1, 64))


def _unit_vector(seed: int, d: int) -> np.ndarray:
    u = _rng(seed, 0, stream=7).standard_normal(d)
    return u / np.linalg.norm(u)


# --------------------------------------------------------------------------- SVM
def svm_labels(n: int, seed: int, flip: float = 0.02, col_lo: int = 0, col_hi: int | None = None):
    """y_i in {-1,+1}: class label (sign of a uniform draw) and the flipped observed label."""
    col_hi = n if col_hi is None else col_hi
    y_true = np.empty(col_hi - col_lo)
    y_obs = np.empty(col_hi - col_lo)
    for blk in range(col_lo // BLOCK, (col_hi + BLOCK - 1) // BLOCK):
        lo, hi = blk * BLOCK, min((blk + 1) * BLOCK, n)
        r = _rng(seed, blk, stream=1)
        yt = np.where(r.random(hi - lo) < 0.5, -1.0, 1.0)
        fl = r.random(hi - lo) < flip
        yo = np.where(fl, -yt, yt)
        a, b = max(lo, col_lo), min(hi, col_hi)
        if a < b:
            y_true[a - col_lo:b - col_lo] = yt[a - lo:b - lo]
            y_obs[a - col_lo:b - col_lo] = yo[a - lo:b - lo]
    return y_true, y_obs


def svm_fill(out: np.ndarray, d: int, n: int, seed: int, mu: float = 0.3, flip: float = 0.02,
             col_lo: int = 0, normalize: bool = True) -> np.ndarray:
    """Fill out[(i - col_lo), :d] with sample x_i, i in [col_lo, col_lo + len(out)).

    x_i = N(0, I_d)/sqrt(d) + mu * ytrue_i * u_hat, then ||x_i|| = 1.
    Returns the observed labels y (2% flipped) for these columns."""
    col_hi = col_lo + out.shape[0]
    assert col_lo % BLOCK == 0 or col_lo == 0
    u = _unit_vector(seed, d).astype(np.float32)
    y_true, y_obs = svm_labels(n, seed, flip, col_lo, col_hi)
    blocks = list(range(col_lo // BLOCK, (col_hi + BLOCK - 1) // BLOCK))
    inv = np.float32(1.0 / math.sqrt(d))

    def work(blk):
        lo, hi = blk * BLOCK, min((blk + 1) * BLOCK, col_hi)
        r = _rng(seed, blk, stream=0)
        X = out[lo - col_lo:hi - col_lo, :d]
        _normal_into(r, X)
        X *= inv
        coef = np.float32(mu) * y_true[lo - col_lo:hi - col_lo].astype(np.float32)
        for q in range(hi - lo):
            X[q] += coef[q] * u
        if normalize:
            nr = np.sqrt(np.einsum("ij,ij->i", X, X, dtype=np.float64))
            nr[nr == 0] = 1.0
            X *= (1.0 / nr).astype(np.float32)[:, None]
        if out.shape[1] > d:
            out[lo - col_lo:hi - col_lo, d:] = 0

    with ThreadPoolExecutor(_threads(len(blocks))) as ex:
        list(ex.map(work, blocks))
    return y_obs


def svm_dense(d: int, n: int, seed: int = SEED0 + 1, mu: float = 0.3, flip: float = 0.02,
              ld: int | None = None):
    """Dense SVM-dual data (columns = samples), unit-norm samples.  Returns (A, y)."""
    ld = d if ld is None else ld
    A = np.empty((n, ld), dtype=np.float32)
    y = svm_fill(A, d, n, seed, mu, flip)
    return A, y


# --------------------------------------------------------------------------- Lasso
def lasso_fill(out: np.ndarray, d: int, n: int, seed: int, corr: float = 0.0, rank: int = 8,
               col_lo: int = 0) -> None:
    """A_ki = sqrt(1-corr) N(0,1) + sqrt(corr) (F l_i)_k, F: d x rank shared factors."""
    col_hi = col_lo + out.shape[0]
    F = None
    if corr > 0:
        F = (_rng(seed, 0, stream=5).standard_normal((rank, d)) / math.sqrt(rank)).astype(np.float32)
    blocks = list(range(col_lo // BLOCK, (col_hi + BLOCK - 1) // BLOCK))
    a = np.float32(math.sqrt(1.0 - corr))
    c = np.float32(math.sqrt(corr))

    def work(blk):
        lo, hi = blk * BLOCK, min((blk + 1) * BLOCK, col_hi)
        r = _rng(seed, blk, stream=0)
        X = out[lo - col_lo:hi - col_lo, :d]
        _normal_into(r, X)
        if F is not None:
            L = r.standard_normal((hi - lo, rank)).astype(np.float32)
            X *= a
            X += c * (L @ F)
        if out.shape[1] > d:
            out[lo - col_lo:hi - col_lo, d:] = 0

    with ThreadPoolExecutor(_threads(len(blocks))) as ex:
        list(ex.map(work, blocks))


def lasso_truth(n: int, seed: int, support: float = 0.1):
    """alpha_true: `support` fraction nonzero, N(0,1) values (per-block counter RNG)."""
    at = np.zeros(n)
    for blk in range((n + BLOCK - 1) // BLOCK):
        lo, hi = blk * BLOCK, min((blk + 1) * BLOCK, n)
        r = _rng(seed, blk, stream=2)
        on = r.random(hi - lo) < support
        val = r.standard_normal(hi - lo)
        at[lo:hi] = np.where(on, val, 0.0)
    return at


def lasso_signal(A: np.ndarray, d: int, seed: int, support: float = 0.1, col_lo: int = 0,
                 n_total: int | None = None) -> np.ndarray:
    """A_shard alpha_true[shard] for the columns [col_lo, col_lo + len(A)) of an
    n_total-column problem (fp64 accumulation in column order)."""
    n_total = A.shape[0] + col_lo if n_total is None else n_total
    at = lasso_truth(n_total, seed, support)[col_lo:col_lo + A.shape[0]]
    b = np.zeros(d)
    for i in np.nonzero(at)[0]:
        b += at[i] * A[i, :d].astype(np.float64)
    return b


def lasso_finish(signal: np.ndarray, d: int, seed: int, noise: float = 0.1) -> np.ndarray:
    """b = signal + noise N(0,1), rescaled to ||b||^2 = d (normalised data, reading R12)."""
    b = signal + noise * _rng(seed, 0, stream=3).standard_normal(d)
    b *= math.sqrt(d) / np.linalg.norm(b)
    return b


def lasso_labels(A: np.ndarray, d: int, seed: int, support: float = 0.1, noise: float = 0.1):
    """b = A alpha_true + noise N(0,1), rescaled to ||b||^2 = d (normalised data, reading R12)."""
    return lasso_finish(lasso_signal(A, d, seed, support), d, seed, noise)


def lasso_dense(d: int, n: int, seed: int = SEED0, corr: float = 0.0, support: float = 0.1,
                noise: float = 0.1, ld: int | None = None):
    """Dense Lasso data (columns = features).  Returns (A, b)."""
    ld = d if ld is None else ld
    A = np.empty((n, ld), dtype=np.float32)
    lasso_fill(A, d, n, seed, corr)
    b = lasso_labels(A, d, seed, support, noise)
    return A, b


# --------------------------------------------------------------------------- sparse (CSC)
def _csc_block(d: int, density: float, seed: int, blk: int, lo: int, hi: int):
    """Columns [lo, hi) of counter block blk: each row is a nonzero independently
    with probability `density` (so nnz_i ~ Binomial(d, density) and, given the
    count, the rows are uniform without replacement), drawn as geometric gaps;
    values N(0, 1).  Returns (counts, rows, vals) of the block's columns."""
    r = _rng(seed, blk, stream=5)
    nb = hi - lo
    mean = d * density
    g = int(mean + 8.0 * math.sqrt(max(mean, 1.0)) + 16)
    gaps = r.geometric(density, size=(nb, g)).astype(np.int64)
    pos = np.cumsum(gaps, axis=1) - 1            # row positions, ascending per column
    counts = (pos < d).sum(axis=1)
    short = np.nonzero(counts == g)[0]           # (vanishingly rare) ran out of draws: extend
    rows_list = None
    if short.size:
        rows_list = [pos[q, :counts[q]] for q in range(nb)]
        for q in short:
            ext = [pos[q]]
            last = pos[q, -1]
            while last < d:
                more = np.cumsum(r.geometric(density, size=g).astype(np.int64)) + last
                ext.append(more)
                last = more[-1]
            allp = np.concatenate(ext)
            rows_list[q] = allp[allp < d]
        counts = np.array([x.size for x in rows_list], dtype=np.int64)
        rows = np.concatenate(rows_list).astype(np.int32)
    else:
        rows = pos[pos < d].astype(np.int32)     # row-major mask keeps column order
    vals = r.standard_normal(rows.size, dtype=np.float32)
    return counts, rows, vals


def csc_lasso(d: int, n: int, seed: int = SEED0 + 5, density: float = 0.01, col_lo: int = 0,
              col_hi: int | None = None):
    """Sparse Lasso design (C5): columns [col_lo, col_hi) of a d x n matrix, CSC
    (col_ptr int64 [k+1], rows int32 ascending per column, values float32)."""
    col_hi = n if col_hi is None else col_hi
    b0, b1 = col_lo // BLOCK, (col_hi - 1) // BLOCK
    jobs = [(blk, max(col_lo, blk * BLOCK), min(col_hi, (blk + 1) * BLOCK)) for blk in range(b0, b1 + 1)]

    def one(job):
        blk, lo, hi = job
        c, r_, v = _csc_block(d, density, seed, blk, blk * BLOCK, min(n, (blk + 1) * BLOCK))
        skip = lo - blk * BLOCK
        take = hi - lo
        starts = np.concatenate([[0], np.cumsum(c)])
        return c[skip:skip + take], r_[starts[skip]:starts[skip + take]], v[starts[skip]:starts[skip + take]]

    with ThreadPoolExecutor(_threads(len(jobs))) as ex:
        parts = list(ex.map(one, jobs))
    counts = np.concatenate([p[0] for p in parts])
    col_ptr = np.zeros(counts.size + 1, dtype=np.int64)
    np.cumsum(counts, out=col_ptr[1:])
    rows = np.concatenate([p[1] for p in parts]) if parts else np.zeros(0, np.int32)
    vals = np.concatenate([p[2] for p in parts]) if parts else np.zeros(0, np.float32)
    return col_ptr, rows, vals


def csc_lasso_signal(col_ptr, rows, vals, d: int, seed: int, support: float = 0.002, col_lo: int = 0,
                     n_total: int | None = None) -> np.ndarray:
    """A_shard alpha_true[shard] (fp64) for CSC columns [col_lo, col_lo + k)."""
    k = col_ptr.size - 1
    n_total = k + col_lo if n_total is None else n_total
    at = lasso_truth(n_total, seed, support)[col_lo:col_lo + k]
    b = np.zeros(d)
    for i in np.nonzero(at)[0]:
        sl = slice(col_ptr[i], col_ptr[i + 1])
        np.add.at(b, rows[sl], at[i] * vals[sl].astype(np.float64))
    return b


def csc_to_dense(col_ptr, rows, vals, d: int, ld: int | None = None) -> np.ndarray:
    """The (n, ld) float32 dense layout of a CSC matrix (test helper)."""
    ld = d if ld is None else ld
    n = col_ptr.size - 1
    A = np.zeros((n, ld), dtype=np.float32)
    cols = np.repeat(np.arange(n), np.diff(col_ptr))
    A[cols, rows] = vals
    return A


# --------------------------------------------------------------------------- structured
def hadamard(d: int) -> np.ndarray:
    """Sylvester Hadamard matrix H_d (d a power of two), entries +-1, H^T H = d I."""
    assert d > 0 and d & (d - 1) == 0
    H = np.ones((1, 1))
    while H.shape[0] < d:
        H = np.block([[H, H], [H, -H]])
    return H


def hadamard_columns(d: int, n: int, scales=None) -> np.ndarray:
    """n <= d distinct Hadamard columns (optionally scaled), as an (n, d) float32 array."""
    H = hadamard(d)
    A = H[:, :n].T.copy()
    if scales is not None:
        A *= np.asarray(scales)[:, None]
    return A.astype(np.float32)


def disjoint_support_csc(d: int, n: int, k: int, seed: int, scales=None):
    """CSC matrix whose n columns have k nonzeros each on pairwise DISJOINT row sets (n k <= d):
    a_i^T a_j = 0 for i != j exactly, whatever subset of their entries is summed, so every
    interleaving of concurrent coordinate updates is the sequential one (the P7/P8 pins of the
    asynchronous epoch).  Rows drawn as a seeded permutation, sorted per column; values N(0,1)
    times an optional per-column scale.  Returns (col_ptr int64, rows int32, vals float32)."""
    assert n * k <= d
    r = np.random.Generator(np.random.Philox(key=[seed, 77]))
    perm = r.permutation(d)[:n * k].reshape(n, k)
    rows = np.sort(perm, axis=1).astype(np.int32).ravel()
    vals = r.standard_normal((n, k))
    if scales is not None:
        vals *= np.asarray(scales, dtype=np.float64)[:, None]
    col_ptr = np.arange(n + 1, dtype=np.int64) * k
    return col_ptr, rows, vals.astype(np.float32).ravel()


def permutation(P, seed: int) -> np.ndarray:
    """A seeded permutation of the index list P (explicit-order parity tests)."""
    P = np.asarray(P, dtype=np.int64)
    return P[np.random.Generator(np.random.Philox(key=[seed, 99])).permutation(P.size)]
