"""CPU oracle for the DuHL hot path (arXiv 1708.05357) -- TEST INFRASTRUCTURE.

Only ``tests/``, ``__graft_entry__.smoke()`` and ``bench.py``'s cpu_baseline /
``--impl reference`` legs may import this package.  The product path
(``paper_1708_05357_b200``) never imports it and shares no code with it.

The arithmetic lives in ``oracle/duhl_oracle.c`` (plain C, fp64 accumulation,
single thread; each function cites the PAPER.md passage it follows).  This
module only compiles it with gcc and marshals numpy arrays through ctypes.

Pins that tie the oracle to the paper (not to itself) are in
``tests/test_oracle_pins.py``; DESIGN.md lists them.
"""
from __future__ import annotations

import ctypes as C
import os
import subprocess

import numpy as np

_HERE = os.path.dirname(os.path.abspath(__file__))
_SRC = os.path.join(_HERE, "duhl_oracle.c")
_LIB = os.path.join(_HERE, "liboracle.so")

LASSO, SVM, RIDGE, ELASTIC = 0, 1, 2, 3
SEL_GAP, SEL_SEQUENTIAL, SEL_UNIFORM, SEL_IMPORTANCE = 0, 1, 2, 3
OK, E_INVALID, E_NUMERIC, E_NOT_CONVERGED = 0, 2, 4, 9


def build(force: bool = False) -> str:
    """Compile the oracle with gcc (plain -O2, no fast-math: IEEE semantics)."""
    if force or not os.path.exists(_LIB) or os.path.getmtime(_LIB) < os.path.getmtime(_SRC):
        tmp = _LIB + f".tmp{os.getpid()}"
        subprocess.check_call(["gcc", "-O2", "-fPIC", "-shared", "-std=c11", "-fno-fast-math",
                               "-ffp-contract=off", "-o", tmp, _SRC, "-lm"])
        os.replace(tmp, _LIB)
    return _LIB


_lib = None
_P = C.c_void_p
_I = C.c_int64


def lib():
    global _lib
    if _lib is None:
        L = C.CDLL(build())
        L.or_mix64.restype = C.c_uint64
        L.or_mix64.argtypes = [C.c_uint64]
        L.or_perm_key.restype = C.c_uint64
        L.or_perm_key.argtypes = [C.c_uint64, _I, _I, _I]
        L.or_col_norms.argtypes = [_P, _I, _I, _I, _P]
        L.or_lasso_B.restype = C.c_double
        L.or_lasso_B.argtypes = [_P, _I, C.c_double]
        L.or_set_eta.restype = None
        L.or_set_eta.argtypes = [C.c_double]
        L.or_matvec.argtypes = [_P, _I, _I, _I, _P, _P]
        L.or_primal_dual_w.argtypes = [C.c_int, _P, _P, _I, _I, C.c_double, _P]
        L.or_coord_gaps.restype = C.c_int
        L.or_coord_gaps.argtypes = [C.c_int, _P, _I, _I, _I, _P, _P, _P, C.c_double, C.c_double,
                                    _P, _I, _P, _P]
        L.or_select_topm.argtypes = [_P, _I, _I, _P]
        L.or_rho.restype = C.c_double
        L.or_rho.argtypes = [_P, _I, _P, _I]
        L.or_select_policy.restype = _I
        L.or_select_policy.argtypes = [C.c_int, _I, _I, _I, C.c_uint64, _P, _P]
        L.or_make_perm.argtypes = [_P, _I, C.c_uint64, _I, _I, _P]
        L.or_perm_index.restype = C.c_int64
        L.or_perm_index.argtypes = [C.c_uint64, _I, _I, _I, _I]
        L.or_coord_update.restype = C.c_double
        L.or_coord_update.argtypes = [C.c_int, C.c_double, C.c_double, C.c_double, C.c_double,
                                      C.c_double, _I, _I]
        L.or_scd_pass.argtypes = [C.c_int, _P, _I, _I, _I, _P, _P, C.c_double, _P, _P, _P, _I]
        L.or_duality_gap.restype = C.c_int
        L.or_duality_gap.argtypes = [C.c_int, _P, _I, _I, _I, _P, _P, C.c_double, C.c_double,
                                     _P, _P, _P]
        L.or_solve_scd.restype = C.c_int
        L.or_solve_scd.argtypes = [C.c_int, _P, _I, _I, _I, _P, C.c_double, C.c_double, _I,
                                   C.c_uint64, _P, _P, _P]
        L.or_linesearch.restype = C.c_double
        L.or_linesearch.argtypes = [C.c_int, _P, _P, _I, _P, _P, _P, _I, C.c_double, _I]
        L.or_duhl_solve_cocoa.restype = C.c_int
        L.or_duhl_solve_cocoa.argtypes = [_P, C.c_int, C.c_int, _P, _I, _I, _I, _P, C.c_double, _P, _P,
                                          _P, _P, _P, _P]
        L.or_duhl_solve.restype = C.c_int
        L.or_duhl_solve.argtypes = [_P, _P, _I, _I, _I, _P, C.c_double, _P, _P, _P, _P, _P, _P]
        _lib = L
    return _lib


class DuhlCfg(C.Structure):
    _fields_ = [("model", C.c_int), ("policy", C.c_int), ("m", C.c_int64), ("passes", C.c_int),
                ("refresh_count", C.c_int64), ("eps", C.c_double), ("max_rounds", C.c_int64),
                ("cert_every", C.c_int64), ("seed", C.c_uint64)]


def _p(a):
    return None if a is None else a.ctypes.data_as(C.c_void_p)


def _f32A(A):
    """A as (n, ld) C-contiguous float32: row i is column a_i (column-major d x n)."""
    A = np.asarray(A)
    assert A.dtype == np.float32 and A.ndim == 2 and A.flags.c_contiguous
    return A


def _f64(x):
    return np.ascontiguousarray(x, dtype=np.float64)


def col_norms(A, d=None):
    A = _f32A(A)
    n, ld = A.shape
    d = ld if d is None else d
    out = np.empty(n)
    lib().or_col_norms(_p(A), d, n, ld, _p(out))
    return out


def set_eta(eta):
    """eta of the elastic-net model (OR_ELASTIC), global in the oracle library."""
    lib().or_set_eta(float(eta))


def lasso_B(b, lam):
    b = _f64(b)
    return lib().or_lasso_B(_p(b), b.size, lam)


def matvec(A, alpha, d=None):
    A = _f32A(A)
    n, ld = A.shape
    d = ld if d is None else d
    alpha = _f64(alpha)
    v = np.empty(d)
    lib().or_matvec(_p(A), d, n, ld, _p(alpha), _p(v))
    return v


def primal_dual_w(model, v, b, n, lam):
    v = _f64(v)
    w = np.empty_like(v)
    bb = _f64(b) if b is not None else None
    lib().or_primal_dual_w(model, _p(v), _p(bb), v.size, n, lam, _p(w))
    return w


def coord_gaps(model, A, alpha, y, w, lam, B=0.0, idx=None, d=None):
    """Returns (status, s, gap) for columns idx (all if None)."""
    A = _f32A(A)
    n, ld = A.shape
    d = ld if d is None else d
    alpha = _f64(alpha)
    yy = _f64(y) if y is not None else None
    w = _f64(w)
    ii = None if idx is None else np.ascontiguousarray(idx, dtype=np.int64)
    k = n if ii is None else ii.size
    s = np.empty(k)
    g = np.empty(k)
    st = lib().or_coord_gaps(model, _p(A), d, n, ld, _p(alpha), _p(yy), _p(w), lam, B, _p(ii), k,
                             _p(s), _p(g))
    return st, s, g


def select_topm(z, m):
    z = _f64(z)
    out = np.empty(m, dtype=np.int64)
    lib().or_select_topm(_p(z), z.size, m, _p(out))
    return out


def rho(z, P):
    """rho_{t,P} (Eq. 6) of the index set P on the gap vector z."""
    z = _f64(z)
    PP = np.ascontiguousarray(P, dtype=np.int64)
    return lib().or_rho(_p(z), z.size, _p(PP), PP.size)


def select_policy(policy, n, m, rnd, seed, z=None):
    """z: the gap memory (SEL_GAP) or ||a_j||^2 (SEL_IMPORTANCE); unused otherwise."""
    zz = _f64(z) if z is not None else np.zeros(n)
    out = np.empty(m, dtype=np.int64)
    k = lib().or_select_policy(policy, n, m, rnd, seed, _p(zz), _p(out))
    return out[:k]


def perm_key(seed, rnd, pas, j):
    return lib().or_perm_key(seed, rnd, pas, j)


def perm_index(seed, rnd, pas, m, t):
    return lib().or_perm_index(seed, rnd, pas, m, t)


def make_perm(P, seed, rnd, pas):
    P = np.ascontiguousarray(P, dtype=np.int64)
    out = np.empty_like(P)
    lib().or_make_perm(_p(P), P.size, seed, rnd, pas, _p(out))
    return out


def coord_update(model, alpha_j, s, norm, y_j, lam, d, n):
    return lib().or_coord_update(model, alpha_j, s, norm, y_j, lam, d, n)


def scd_pass(model, A, norms, y, lam, alpha, vt, order, d=None):
    """In place on alpha (n,) and vt (d,) float64 arrays."""
    A = _f32A(A)
    n, ld = A.shape
    d = ld if d is None else d
    assert alpha.dtype == np.float64 and vt.dtype == np.float64
    order = np.ascontiguousarray(order, dtype=np.int64)
    yy = _f64(y) if y is not None else None
    lib().or_scd_pass(model, _p(A), d, n, ld, _p(_f64(norms)), _p(yy), lam, _p(alpha), _p(vt),
                      _p(order), order.size)


def duality_gap(model, A, alpha, b_or_y, lam, B=0.0, d=None):
    """Returns (status, gap, primal O, dual D)."""
    A = _f32A(A)
    n, ld = A.shape
    d = ld if d is None else d
    g, O, D = C.c_double(), C.c_double(), C.c_double()
    st = lib().or_duality_gap(model, _p(A), d, n, ld, _p(_f64(alpha)), _p(_f64(b_or_y)), lam, B,
                              C.byref(g), C.byref(O), C.byref(D))
    return st, g.value, O.value, D.value


def solve_scd(model, A, b_or_y, lam, eps, max_epochs, seed=0, alpha0=None, d=None):
    """Plain sequential SCD to certified gap <= eps. Returns (status, alpha, gap, epochs)."""
    A = _f32A(A)
    n, ld = A.shape
    d = ld if d is None else d
    alpha = np.zeros(n) if alpha0 is None else _f64(alpha0).copy()
    g = C.c_double()
    e = C.c_int64()
    st = lib().or_solve_scd(model, _p(A), d, n, ld, _p(_f64(b_or_y)), lam, eps, max_epochs, seed,
                            _p(alpha), C.byref(g), C.byref(e))
    return st, alpha, g.value, e.value


def duhl_solve(model, A, b_or_y, lam, m, passes=1, policy=SEL_GAP, refresh_count=None, eps=1e-5,
               max_rounds=100, cert_every=1, seed=0, alpha0=None, d=None):
    """DuHL Algorithm 2 in the deterministic semantics of duhl_oracle.c.

    Returns dict(status, alpha, z, rounds, gap, swaps[rounds], gaps[rounds])."""
    A = _f32A(A)
    n, ld = A.shape
    d = ld if d is None else d
    cfg = DuhlCfg(model, policy, m, passes, n if refresh_count is None else refresh_count, eps,
                  max_rounds, cert_every, seed)
    alpha = np.zeros(n) if alpha0 is None else _f64(alpha0).copy()
    z = np.empty(n)
    rounds = C.c_int64()
    gap = C.c_double()
    sw = np.zeros(max_rounds, dtype=np.int64)
    tg = np.zeros(max_rounds)
    st = lib().or_duhl_solve(C.byref(cfg), _p(A), d, n, ld, _p(_f64(b_or_y)), lam, _p(alpha),
                             _p(z), C.byref(rounds), C.byref(gap), _p(sw), _p(tg))
    r = rounds.value
    return dict(status=st, alpha=alpha, z=z, rounds=r, gap=gap.value, swaps=sw[:r], gaps=tg[:r])


def linesearch(model, v0, dv, a_old, da, y, lam, n):
    """Exact line search on the aggregation weight gamma in [0, 1] (or_linesearch)."""
    v0, dv = _f64(v0), _f64(dv)
    a_old, da = _f64(a_old), _f64(da)
    yy = _f64(y) if y is not None else np.zeros_like(da)
    return lib().or_linesearch(model, _p(v0), _p(dv), v0.size, _p(a_old), _p(da), _p(yy), da.size,
                               lam, n)


def duhl_solve_cocoa(model, A, b_or_y, lam, m, K, linesearch=True, passes=1, policy=SEL_GAP,
                     refresh_count=0, eps=1e-5, max_rounds=100, cert_every=1, seed=0, d=None):
    """DuHL on K column shards with CoCoA-style aggregation (or_duhl_solve_cocoa).
    m and refresh_count are per shard.  Returns dict(status, alpha, z, rounds, gap, gaps, gammas)."""
    A = _f32A(A)
    n, ld = A.shape
    d = ld if d is None else d
    cfg = DuhlCfg(model, policy, m, passes, refresh_count, eps, max_rounds, cert_every, seed)
    alpha = np.zeros(n)
    z = np.empty(n)
    rounds = C.c_int64()
    gap = C.c_double()
    tg = np.zeros(max_rounds)
    gm = np.zeros(max_rounds)
    st = lib().or_duhl_solve_cocoa(C.byref(cfg), K, int(bool(linesearch)), _p(A), d, n, ld,
                                   _p(_f64(b_or_y)), lam, _p(alpha), _p(z), C.byref(rounds),
                                   C.byref(gap), _p(tg), _p(gm))
    r = rounds.value
    return dict(status=st, alpha=alpha, z=z, rounds=r, gap=gap.value, gaps=tg[:r], gammas=gm[:r])
