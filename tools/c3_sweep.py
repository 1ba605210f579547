"""C3 time-to-eps sweep over (refresh fraction, passes) with adaptive certificates only.

    python tools/c3_sweep.py 0.1:3 0.05:2 ...
"""
import os, sys, time
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import bench, paper_1708_05357_b200 as D
cfg = bench.CONFIGS[os.environ.get("CONFIG", "c3")]
A, lab = bench.make_data(cfg, 170805360)
lam = bench.lam_of(cfg, A, lab)
n, d = A.shape
budget = int(0.25 * n * ((d + 3) // 4) * 16)
for spec in sys.argv[1:]:
    f, p = spec.split(":")
    P = D.create(A, lab, lam, cfg["model"], hbm_budget_bytes=budget, m=cfg["m"], refresh_fraction=float(f),
                 borrow_host=True, scd_exact=False, cert_every=100000, profile=False)
    t0 = time.perf_counter()
    r = P.solve(1e-5, 2000, passes=int(p))
    dt = time.perf_counter() - t0
    ncert = sum(1 for t in r["trace"] if t.cert_gap >= 0)
    print(f"refresh {f} passes {p}: {dt:.2f} s, {r['rounds']} rounds, {ncert} certificates, gap {r['gap']:.3e}", flush=True)
    P.close()
