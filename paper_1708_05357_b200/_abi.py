"""ctypes binding of include/duhl.h (marshalling only; no arithmetic of the method here)."""
from __future__ import annotations

import ctypes as C
import os

import numpy as np

from . import build as _build

LASSO, SVM_DUAL, RIDGE, ELASTIC_NET = 0, 1, 2, 3
SEL_GAP, SEL_SEQUENTIAL, SEL_UNIFORM, SEL_IMPORTANCE = 0, 1, 2, 3
STATUS = {0: "OK", 2: "E_INVALID", 3: "E_IO", 4: "E_NUMERIC", 5: "E_BOUND", 6: "E_NOMEM",
          7: "E_CUDA", 8: "E_NCCL", 9: "E_NOT_CONVERGED"}

FUNCTIONS = ["duhl_default_config", "duhl_create", "duhl_create_csc", "duhl_destroy", "duhl_gaps", "duhl_select",
             "duhl_scd_epoch", "duhl_duality_gap", "duhl_round", "duhl_solve", "duhl_get_state",
             "duhl_set_state", "duhl_comm_unique_id", "duhl_comm_init", "duhl_get_stream",
             "duhl_get_kernel_stats", "duhl_get_counters", "duhl_get_scd_shape", "duhl_get_unit_a_host",
             "duhl_group_create", "duhl_group_destroy", "duhl_comm_init_group", "duhl_get_working_set",
             "duhl_set_trace_callback", "duhl_last_error"]
KIND_SCD, KIND_GAP, KIND_TOPM, KIND_STAGE = 0, 1, 2, 3


class DuhlError(RuntimeError):
    def __init__(self, status, msg):
        super().__init__(f"duhl {STATUS.get(status, status)}: {msg}")
        self.status = status


class Matrix(C.Structure):
    _fields_ = [("d", C.c_int64), ("n", C.c_int64), ("values", C.c_void_p), ("ld", C.c_int64)]


class Csc(C.Structure):
    _fields_ = [("d", C.c_int64), ("n", C.c_int64), ("col_ptr", C.c_void_p), ("row_idx", C.c_void_p),
                ("values", C.c_void_p)]


class Config(C.Structure):
    _fields_ = [("hbm_budget_bytes", C.c_size_t), ("m", C.c_int64), ("device", C.c_int),
                ("scd_block", C.c_int), ("scd_ctas", C.c_int), ("refresh_fraction", C.c_double),
                ("cert_every", C.c_int64), ("seed", C.c_uint64), ("borrow_host", C.c_int),
                ("cert_adaptive", C.c_int), ("profile", C.c_int), ("scd_exact", C.c_int),
                ("n_global", C.c_int64), ("col_offset", C.c_int64), ("linesearch", C.c_int),
                ("unit_a_ctas", C.c_int), ("scd_kernel", C.c_int), ("eta", C.c_double),
                ("unit_a_host_threads", C.c_int), ("unit_a_host_share", C.c_double), ("scd_async", C.c_int)]


class RoundRecord(C.Structure):
    _fields_ = [("round", C.c_int64), ("swaps", C.c_int64), ("refreshed", C.c_int64),
                ("cert_gap", C.c_double), ("z_sum", C.c_double), ("gamma", C.c_double),
                ("time_s", C.c_double), ("rho", C.c_double), ("gap_est", C.c_double)]


TRACE_CB = C.CFUNCTYPE(None, C.POINTER(RoundRecord), C.c_void_p)

_lib = None
_P = C.c_void_p
_I = C.c_int64


def lib_path() -> str:
    return _build.LIB


def lib():
    """Load libduhl.so (building it in-tree first if the sources are newer)."""
    global _lib
    if _lib is None:
        path = os.environ.get("DUHL_LIB") or (
            _build.build() if os.environ.get("DUHL_NO_BUILD") != "1" else _build.LIB)
        L = C.CDLL(path)
        L.duhl_default_config.argtypes = [C.POINTER(Config)]
        L.duhl_default_config.restype = None
        L.duhl_create.argtypes = [C.POINTER(Matrix), _P, C.c_double, C.c_int, C.POINTER(Config),
                                  C.POINTER(C.c_void_p)]
        L.duhl_create_csc.argtypes = [C.POINTER(Csc), _P, C.c_double, C.c_int, C.POINTER(Config),
                                      C.POINTER(C.c_void_p)]
        L.duhl_destroy.argtypes = [_P]
        L.duhl_gaps.argtypes = [_P, _P, _I, _P, _P]
        L.duhl_select.argtypes = [_P, C.c_int, _I, _I, _P, _P]
        L.duhl_scd_epoch.argtypes = [_P, C.c_int, C.c_uint64, _I, _P, _I]
        L.duhl_duality_gap.argtypes = [_P, _P, _P, _P]
        L.duhl_round.argtypes = [_P, _I, C.c_int, C.c_int, C.c_int, _P]
        L.duhl_solve.argtypes = [_P, C.c_double, _I, C.c_int, C.c_int, _P, _I, _P, _P]
        L.duhl_get_kernel_stats.argtypes = [_P, C.c_int, _P, _P, _P]
        L.duhl_comm_unique_id.argtypes = [_P]
        L.duhl_comm_init.argtypes = [_P, _P, C.c_int, C.c_int]
        L.duhl_get_state.argtypes = [_P, _P, _P, _P]
        L.duhl_set_state.argtypes = [_P, _P]
        L.duhl_get_stream.argtypes = [_P, C.POINTER(C.c_void_p)]
        L.duhl_get_counters.argtypes = [_P, _P, _P, _P, _P, _P]
        L.duhl_get_unit_a_host.argtypes = [_P, _P, _P]
        L.duhl_get_scd_shape.argtypes = [_P, _P, _P, _P, _P]
        L.duhl_group_create.argtypes = [C.c_int, C.POINTER(C.c_void_p)]
        L.duhl_group_destroy.argtypes = [_P]
        L.duhl_comm_init_group.argtypes = [_P, _P, C.c_int]
        L.duhl_get_working_set.argtypes = [_P, _P, _I, _P]
        L.duhl_set_trace_callback.argtypes = [_P, TRACE_CB, _P]
        L.duhl_last_error.argtypes = [_P]
        L.duhl_last_error.restype = C.c_char_p
        for f in FUNCTIONS:
            if f not in ("duhl_default_config", "duhl_last_error"):
                getattr(L, f).restype = C.c_int
        _lib = L
    return _lib


def exported_symbols():
    L = lib()
    return {f: hasattr(L, f) for f in FUNCTIONS}


def _p(a):
    return None if a is None else C.c_void_p(a.ctypes.data)


def default_config(**kw) -> Config:
    cfg = Config()
    lib().duhl_default_config(C.byref(cfg))
    for k, v in kw.items():
        if v is not None:
            setattr(cfg, k, v)
    return cfg


class Problem:
    """One duhl_ctx.  Arrays in/out are numpy (host); the library owns device state."""

    def __init__(self, handle, d, n, keepalive=None):
        self._h = handle
        self.d, self.n = d, n
        self._keep = keepalive

    def _check(self, st):
        if st != 0:
            msg = lib().duhl_last_error(self._h).decode()
            raise DuhlError(st, msg)

    def close(self):
        if self._h:
            lib().duhl_destroy(self._h)
            self._h = None

    def __del__(self):
        try:
            self.close()
        except Exception:
            pass

    def __enter__(self):
        return self

    def __exit__(self, *a):
        self.close()

    # ---- ABI calls
    def gaps(self, idx=None, want_s=False):
        """duhl_gaps: returns (gap, s) for columns idx (all if None); z is updated."""
        ii = None if idx is None else np.ascontiguousarray(idx, dtype=np.int64)
        k = self.n if ii is None else ii.size
        z = np.empty(k)
        s = np.empty(k) if want_s else None
        self._check(lib().duhl_gaps(self._h, _p(ii), k, _p(z), _p(s)))
        return (z, s) if want_s else z

    def select(self, policy=SEL_GAP, m=0, round=0):
        """duhl_select: returns (P ascending, swaps)."""
        mm = m if m > 0 else self.m
        P = np.empty(mm, dtype=np.int64)
        sw = C.c_int64()
        self._check(lib().duhl_select(self._h, policy, m, round, _p(P), C.byref(sw)))
        return P, sw.value

    def scd_epoch(self, passes=1, seed=0, round=0, perm=None):
        pp = None if perm is None else np.ascontiguousarray(perm, dtype=np.int64)
        self._check(lib().duhl_scd_epoch(self._h, passes, seed, round, _p(pp),
                                         0 if pp is None else pp.size))

    def duality_gap(self):
        g, O, D = C.c_double(), C.c_double(), C.c_double()
        self._check(lib().duhl_duality_gap(self._h, C.byref(g), C.byref(O), C.byref(D)))
        return g.value, O.value, D.value

    def round(self, t, passes=1, policy=SEL_GAP, certify=False):
        """duhl_round: one DuHL round; returns its RoundRecord."""
        rec = RoundRecord()
        self._check(lib().duhl_round(self._h, t, passes, policy, int(bool(certify)), C.byref(rec)))
        return rec

    def kernel_stats(self, kind):
        """duhl_get_kernel_stats: (timed launches, total ms, total algorithmic bytes)."""
        n, ms, by = C.c_int64(), C.c_double(), C.c_double()
        self._check(lib().duhl_get_kernel_stats(self._h, kind, C.byref(n), C.byref(ms), C.byref(by)))
        return n.value, ms.value, by.value

    def solve(self, eps, max_rounds, passes=1, policy=SEL_GAP, trace_cap=None, check=True):
        cap = max_rounds if trace_cap is None else trace_cap
        tr = (RoundRecord * max(cap, 1))()
        r, g = C.c_int64(), C.c_double()
        st = lib().duhl_solve(self._h, eps, max_rounds, passes, policy, C.cast(tr, C.c_void_p), cap,
                              C.byref(r), C.byref(g))
        if check and st not in (0, 9):
            self._check(st)
        recs = [tr[i] for i in range(min(r.value, cap))]
        return dict(status=st, rounds=r.value, gap=g.value, trace=recs)

    def get_state(self):
        a, v, z = np.empty(self.n), np.empty(self.d), np.empty(self.n)
        self._check(lib().duhl_get_state(self._h, _p(a), _p(v), _p(z)))
        return a, v, z

    def set_state(self, alpha):
        a = np.ascontiguousarray(alpha, dtype=np.float64)
        self._check(lib().duhl_set_state(self._h, _p(a)))

    def working_set(self):
        """duhl_get_working_set: the current P (ascending local column indices)."""
        m = C.c_int64()
        self._check(lib().duhl_get_working_set(self._h, None, 0, C.byref(m)))
        P = np.empty(m.value, dtype=np.int64)
        self._check(lib().duhl_get_working_set(self._h, _p(P), P.size, C.byref(m)))
        return P

    def set_trace_callback(self, fn):
        """duhl_set_trace_callback: fn(RoundRecord) after every duhl_solve round (None removes it)."""
        self._cb = None if fn is None else TRACE_CB(lambda rec, user: fn(rec.contents))
        self._check(lib().duhl_set_trace_callback(self._h, self._cb if self._cb else TRACE_CB(), None))

    def comm_init_group(self, group, rank: int):
        """duhl_comm_init_group: join an in-process Group (contexts driven by host threads)."""
        self._check(lib().duhl_comm_init_group(self._h, group._h, rank))

    def comm_init(self, unique_id: bytes, nranks: int, rank: int):
        """duhl_comm_init: join the NCCL group identified by the 128-byte id."""
        buf = C.create_string_buffer(bytes(unique_id), 128)
        self._check(lib().duhl_comm_init(self._h, buf, nranks, rank))

    def stream(self):
        s = C.c_void_p()
        self._check(lib().duhl_get_stream(self._h, C.byref(s)))
        return s.value

    def unit_a_host(self):
        """duhl_get_unit_a_host: (host-refreshed columns so far, current host share)."""
        c, sh = C.c_int64(), C.c_double()
        self._check(lib().duhl_get_unit_a_host(self._h, C.byref(c), C.byref(sh)))
        return c.value, sh.value

    def scd_shape(self):
        """(kernel name, W, G, R) of the exact SCD epoch chosen at create."""
        k, w, g, r = C.c_int(), C.c_int(), C.c_int(), C.c_int()
        self._check(lib().duhl_get_scd_shape(self._h, C.byref(k), C.byref(w), C.byref(g), C.byref(r)))
        return ["k_csc_scd", "k_scd_gram", "k_scd_pipe", "k_scd_tpa", "k_scd_ser"][k.value], w.value, g.value, r.value

    def counters(self):
        a, b, z, c, e = C.c_int64(), C.c_int64(), C.c_int64(), C.c_int64(), C.c_int64()
        self._check(lib().duhl_get_counters(self._h, C.byref(a), C.byref(b), C.byref(z), C.byref(c),
                                            C.byref(e)))
        return dict(launches=a.value, h2d_bytes=b.value, zc_bytes=z.value, updates=c.value, d2h_bytes=e.value)


def create(A, b_or_y, lam, model, hbm_budget_bytes=0, m=0, device=0, scd_block=0, scd_ctas=0,
           refresh_fraction=0.05, cert_every=10, seed=170805357, borrow_host=False, d=None,
           cert_adaptive=True, profile=False, scd_exact=True, n_global=0, col_offset=0,
           linesearch=False, unit_a_ctas=0, scd_kernel=0, eta=0.0, unit_a_host_threads=0,
           unit_a_host_share=-1.0, scd_async=False):
    """duhl_create.  eta: the elastic-net mix (model ELASTIC_NET only).  A: (n, ld) C-contiguous float32 (row i = column a_i of the d x n matrix)."""
    A = np.asarray(A)
    if A.dtype != np.float32 or A.ndim != 2 or not A.flags.c_contiguous:
        raise ValueError("A must be a C-contiguous (n, ld) float32 array")
    n, ld = A.shape
    d = ld if d is None else d
    lab = np.ascontiguousarray(b_or_y, dtype=np.float64)
    mat = Matrix(d, n, A.ctypes.data, ld)
    cfg = default_config(hbm_budget_bytes=hbm_budget_bytes, m=m, device=device,
                         scd_block=scd_block, scd_ctas=scd_ctas,
                         refresh_fraction=refresh_fraction, cert_every=cert_every, seed=seed,
                         borrow_host=int(bool(borrow_host)), cert_adaptive=int(bool(cert_adaptive)),
                         profile=int(bool(profile)), scd_exact=int(bool(scd_exact)),
                         n_global=n_global, col_offset=col_offset, linesearch=int(bool(linesearch)),
                         unit_a_ctas=unit_a_ctas, scd_kernel=scd_kernel, eta=float(eta),
                         unit_a_host_threads=int(unit_a_host_threads),
                         unit_a_host_share=float(unit_a_host_share), scd_async=int(bool(scd_async)))
    h = C.c_void_p()
    st = lib().duhl_create(C.byref(mat), _p(lab), lam, model, C.byref(cfg), C.byref(h))
    if st != 0:
        raise DuhlError(st, "duhl_create failed (a B200 / sm_100 device is required)")
    prob = Problem(h, d, n, keepalive=A if borrow_host else None)
    prob.m = cfg.m if cfg.m > 0 else (n if hbm_budget_bytes == 0 else
                                      min(n, hbm_budget_bytes // (((d + 3) // 4) * 16)))
    return prob


def create_csc(col_ptr, row_idx, values, d, b_or_y, lam, model, m=0, device=0, refresh_fraction=0.05,
               cert_every=10, seed=170805357, cert_adaptive=True, profile=False, scd_exact=True,
               n_global=0, col_offset=0, linesearch=False, scd_ctas=0, eta=0.0):
    """duhl_create_csc.  CSC arrays: col_ptr int64 [n+1], row_idx int32 [nnz] (ascending per
    column), values float32 [nnz]; the matrix is copied to HBM."""
    cp = np.ascontiguousarray(col_ptr, dtype=np.int64)
    ri = np.ascontiguousarray(row_idx, dtype=np.int32)
    va = np.ascontiguousarray(values, dtype=np.float32)
    n = cp.shape[0] - 1
    lab = np.ascontiguousarray(b_or_y, dtype=np.float64)
    mat = Csc(d, n, cp.ctypes.data, ri.ctypes.data, va.ctypes.data)
    cfg = default_config(m=m, device=device, refresh_fraction=refresh_fraction, cert_every=cert_every,
                         seed=seed, cert_adaptive=int(bool(cert_adaptive)), profile=int(bool(profile)),
                         scd_exact=int(bool(scd_exact)), n_global=n_global, col_offset=col_offset,
                         linesearch=int(bool(linesearch)), scd_ctas=scd_ctas, eta=float(eta))
    h = C.c_void_p()
    st = lib().duhl_create_csc(C.byref(mat), _p(lab), lam, model, C.byref(cfg), C.byref(h))
    if st != 0:
        raise DuhlError(st, "duhl_create_csc failed (a B200 / sm_100 device is required)")
    prob = Problem(h, d, n)
    prob.m = cfg.m if cfg.m > 0 else n
    return prob


class Group:
    """duhl_group_create / duhl_group_destroy: an in-process communicator for nranks contexts,
    each driven by its own host thread; collectives reduce through host memory in rank order."""

    def __init__(self, nranks: int):
        h = C.c_void_p()
        st = lib().duhl_group_create(nranks, C.byref(h))
        if st != 0:
            raise DuhlError(st, "duhl_group_create failed")
        self._h, self.nranks = h, nranks

    def close(self):
        if self._h:
            lib().duhl_group_destroy(self._h)
            self._h = None

    def __enter__(self):
        return self

    def __exit__(self, *a):
        self.close()


def comm_unique_id() -> bytes:
    """duhl_comm_unique_id: a fresh 128-byte NCCL id (call on one rank, broadcast it)."""
    buf = C.create_string_buffer(128)
    st = lib().duhl_comm_unique_id(buf)
    if st != 0:
        raise DuhlError(st, "duhl_comm_unique_id failed")
    return buf.raw
