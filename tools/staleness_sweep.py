"""NEXT-1 staleness study (Sec. 5.1, Fig. 4a "Effect of Gap-Approximation", P:387-388,
and Fig. 4b "Reduced I/O operations"), on the GPU path.

For proxies of the C3 (dense Lasso, d << n) and C4 (dense SVM dual, d >> n) aspects held 4x over
an HBM budget of 25 %, DuHL is run to a certified duality gap eps with the unit-A refresh of
a fraction f of the gap memory per round (rotating cursor, reading R8): f = 1 is o-DuHL (every
gap exact at selection time), smaller f = staler gaps.  Reported per f: rounds and wall time
to eps, total columns swapped, and the swaps-per-round trace (Fig. 4b), next to the
sequential [Yu 2012] / uniform batch baselines on the same data and budget.  Writes
profiles/r02_staleness_sweep.json."""
import json, os, sys, time
import numpy as np
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_1708_05357_b200 as D
import synth

EPS = 1e-5


def run(name, model, A, lab, lam, m, passes, policies):
    n, d = A.shape
    budget = m * ((d + 3) // 4) * 16
    rows = []
    for pol, f in policies:
        P = D.create(A, lab, lam, model, hbm_budget_bytes=budget, m=m, refresh_fraction=f, cert_every=1,
                     seed=11, scd_exact=False)
        t0 = time.perf_counter()
        r = P.solve(EPS, 3000, passes=passes, policy=pol)
        t = time.perf_counter() - t0
        P.close()
        sw = [x.swaps for x in r["trace"]]
        rows.append(dict(policy=["gap", "sequential", "uniform", "importance"][pol], refresh=f,
                         rounds=r["rounds"], converged=r["status"] == 0, gap=r["gap"], time_s=t,
                         swaps_total_over_m=sum(sw) / m, swaps_per_round=sw,
                         rho_mean=float(np.mean([x.rho for x in r["trace"]]))))
        print(name, json.dumps({k: v for k, v in rows[-1].items() if k != "swaps_per_round"}), flush=True)
    return dict(name=name, d=d, n=n, m=m, passes=passes, lam=lam, eps=EPS, runs=rows)


def main():
    out = []
    gap_f = [1.0, 0.2, 0.1, 0.05, 0.02, 0.01]
    pols = [(D.SEL_GAP, f) for f in gap_f] + [(D.SEL_SEQUENTIAL, 0.0), (D.SEL_UNIFORM, 0.0)]
    # C3 aspect (Lasso, d << n), 4x over budget
    d, n = 4000, 20000
    A, b = synth.lasso_dense(d, n, seed=5)
    lmax = np.abs(A.astype(np.float64) @ b).max() / d
    out.append(run("lasso_c3_aspect", D.LASSO, A, b, 0.07 * lmax, n // 4, 3, pols))
    # C4 aspect (SVM dual, d >> n), 4x over budget
    d, n = 20000, 4000
    A, y = synth.svm_dense(d, n, seed=6)
    out.append(run("svm_c4_aspect", D.SVM_DUAL, A, y, 1.0 / n, n // 4, 2, pols))
    os.makedirs("profiles", exist_ok=True)
    json.dump(out, open("profiles/r02_staleness_sweep.json", "w"), indent=1)


if __name__ == "__main__":
    main()
