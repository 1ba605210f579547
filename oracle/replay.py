"""Algorithm 2 round by round on the CPU oracle, following the
device's working sets -- TEST INFRASTRUCTURE (only tests/ and smoke() use it).

Eq. 11's argmax is set-valued: gap-memory entries that agree to rounding
(converged coordinates whose gap is 0 in exact arithmetic, but ~1e-17 after
rounding) may be ordered either way, and the oracle's ``max(gap, +0.0)`` clamp (reading
R17) keeps that noise while the kernels read it as +0.0.  SURVEY 8(c) therefore requires
selection parity only outside a tolerance band.  Each round ``check_selection`` verifies
the device's P against the ORACLE's own gap memory -- |P| = m, every coordinate above
t + tau_i in, every one below t - tau_i out (t = the m-th largest z, tau_i the gap
tolerance) -- and exact equality for the gap-independent policies; ``round`` then runs
the oracle's round on that (verified) set.  Every number is the oracle's arithmetic
(``oracle/duhl_oracle.c``: gaps, permutations, SCD passes, line search, certificate),
composed in the order of ``or_duhl_solve`` / ``or_duhl_solve_cocoa``; no value is taken
from the device except the choice among equally valid working sets.
"""
from __future__ import annotations

import numpy as np

import oracle as O

TOL = 1e-6     # north_star gap tolerance (fp64-accumulated mode)
KAPPA = 1e-3   # SURVEY 8(c) conditioning floor


class Alg2:
    """The oracle's DuHL state (alpha, shared vector, gap memory) on K column shards.

    K = 1 without line search is or_duhl_solve; otherwise or_duhl_solve_cocoa (sigma' = 1
    local passes from the common v, dv summed in shard order, gamma by or_linesearch)."""

    def __init__(self, model, A, lab, lam, m, passes, refresh_count, seed, K=1, linesearch=False,
                 d=None):
        self.A = A
        self.n, ld = A.shape
        self.d = ld if d is None else d
        self.model, self.lab, self.lam = model, np.asarray(lab, dtype=np.float64), lam
        self.y = self.lab if model == O.SVM else None
        self.b = None if model == O.SVM else self.lab
        self.norms = O.col_norms(A, d=self.d)
        self.B = O.lasso_B(self.lab, lam) if model == O.LASSO else 0.0
        self.m, self.passes, self.rc, self.seed = m, passes, refresh_count, seed
        self.K, self.ls = K, linesearch
        self.cursor = [0] * K
        self.prev = set()
        self.alpha = np.zeros(self.n)
        self.vt = -self.b.copy() if self.b is not None else np.zeros(self.d)  # alpha = 0
        st, _, self.z = O.coord_gaps(model, A, self.alpha, self.y, self.w(), lam, self.B, d=self.d)
        assert st == O.OK
        self.eta = None

    def shard(self, k):
        return k * self.n // self.K, (k + 1) * self.n // self.K

    def w(self):
        """App. E: w = v~ (regression models) or v^/(lambda n) (SVM)."""
        if self.model == O.SVM:
            return O.primal_dual_w(O.SVM, self.vt, None, self.n, self.lam)
        return self.vt.copy()

    def _tau(self, idx, eta=0.5, tol=TOL):
        """Gap tolerance of SURVEY 8(c): tol * max(|z_i|, kappa c_i ||a_i|| ||w||), c_i a bound
        on |d gap_i / d s_i| at the current state."""
        a = np.abs(self.alpha[idx])
        an = np.sqrt(self.norms[idx])
        wn = np.linalg.norm(self.w())
        d, n, lam = self.d, self.n, self.lam
        if self.model == O.LASSO:
            c = (a + self.B) / d
        elif self.model == O.SVM:
            c = (a + 1.0) / n
        elif self.model == O.RIDGE:
            c = (an * wn + lam * d * a) / (lam * d * d) + 1.0 / d
        else:
            c = a / d + an * wn / (lam * eta * d * d) + 1.0 / d
        return tol * np.maximum(np.abs(self.z[idx]), KAPPA * c * an * wn)

    def check_selection(self, P_list, policy, t, tol=TOL):
        """P_list[k]: shard k's working set (global indices, ascending) from the device.
        tol: the gap tolerance (north_star: 1e-6 fp64-accumulated, 1e-4 fp32 mode)."""
        for k, Pk in enumerate(P_list):
            lo, hi = self.shard(k)
            Pk = np.asarray(Pk, dtype=np.int64)
            nk = hi - lo
            assert np.all(np.diff(Pk) > 0) and (Pk.size == 0 or (Pk[0] >= lo and Pk[-1] < hi))
            if policy != O.SEL_GAP:   # gap-independent: one valid answer
                ref = O.select_policy(policy, nk, self.m, t, self.seed,
                                      self.norms[lo:hi] if policy == O.SEL_IMPORTANCE else None)
                assert Pk.tolist() == (np.sort(ref) + lo).tolist(), (k, t)
                continue
            mk = min(self.m, nk)
            assert Pk.size == mk, (k, t, Pk.size, mk)
            zk = self.z[lo:hi]
            thr = np.sort(zk)[::-1][mk - 1]
            tau = self._tau(np.arange(lo, hi), tol=tol)
            sel = np.zeros(nk, dtype=bool)
            sel[Pk - lo] = True
            must_in = zk > thr + tau
            must_out = zk < thr - tau
            assert np.all(sel[must_in]), (k, t, np.nonzero(must_in & ~sel)[0][:5])
            assert not np.any(sel[must_out]), (k, t, np.nonzero(must_out & sel)[0][:5])

    def round(self, t, P_list, certify=True):
        """One Alg. 2 round on the given per-shard sets; returns dict(gap, gamma, swaps)."""
        A, model, lam, d = self.A, self.model, self.lam, self.d
        P_list = [np.asarray(Pk, dtype=np.int64) for Pk in P_list]
        P_all = np.concatenate(P_list) if P_list else np.zeros(0, dtype=np.int64)
        cur = set(P_all.tolist())
        swaps = len(cur - self.prev)
        self.prev = cur
        # unit A (l.7-10): rotating-cursor refresh of each shard at the round-start state (R8)
        w = self.w()
        for k in range(self.K):
            lo, hi = self.shard(k)
            nk = hi - lo
            kr = min(self.rc, nk)
            if kr > 0:
                idx = lo + (self.cursor[k] + np.arange(kr)) % nk
                self.cursor[k] = (self.cursor[k] + kr) % nk
                st, _, g = O.coord_gaps(model, A, self.alpha, self.y, w, lam, self.B, idx=idx, d=d)
                assert st == O.OK
                self.z[idx] = g
        # unit B (l.6, l.11): randomized passes (R10), aggregation (R16)
        gamma = 1.0
        if self.K == 1 and not self.ls:
            for p in range(self.passes):
                O.scd_pass(model, A, self.norms, self.y, lam, self.alpha, self.vt,
                           O.make_perm(P_all, self.seed, t, p), d=d)
        else:
            v0 = self.vt.copy()
            aold = self.alpha[P_all].copy()
            dv = np.zeros(d)
            for Pk in P_list:
                vk = v0.copy()
                for p in range(self.passes):
                    O.scd_pass(model, A, self.norms, self.y, lam, self.alpha, vk,
                               O.make_perm(Pk, self.seed, t, p), d=d)
                dv += vk - v0
            da = self.alpha[P_all] - aold
            if self.ls:
                gamma = O.linesearch(model, v0, dv, aold, da, None if self.y is None else self.y[P_all],
                                     lam, self.n)
            self.vt = v0 + gamma * dv
            self.alpha[P_all] = aold + gamma * da
        # z_P at the new state (R9)
        st, _, g = O.coord_gaps(model, A, self.alpha, self.y, self.w(), lam, self.B, idx=P_all, d=d)
        assert st == O.OK
        self.z[P_all] = g
        gap = None
        if certify:
            st, gap, _, _ = O.duality_gap(model, A, self.alpha, self.lab, lam, self.B, d=d)
            assert st == O.OK
            # R25: the certificate's gaps at the current state refresh the whole gap memory
            st, _, self.z = O.coord_gaps(model, A, self.alpha, self.y, self.w(), lam, self.B, d=d)
            assert st == O.OK
        return dict(gap=gap, gamma=gamma, swaps=swaps)
