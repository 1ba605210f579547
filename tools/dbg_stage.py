import os, sys, time
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np, synth, paper_1708_05357_b200 as D
for (d, n, m, exact, cert, f) in [(2000, 1000, 250, True, 1, 0.05), (2000, 1000, 250, True, 1, 0.0),
                                  (2000, 1000, 250, True, 1000, 0.05), (2000, 1000, 250, False, 1, 0.05),
                                  (256, 2000, 500, True, 1, 0.05)]:
    A, b = synth.lasso_dense(d, n)
    t0 = time.time()
    try:
        with D.create(A, b, 0.1, D.LASSO, hbm_budget_bytes=m * d * 4, m=m, refresh_fraction=f, cert_every=cert,
                      seed=1, scd_exact=exact) as P:
            r = P.solve(0.0, 3, passes=1)
            print(d, n, m, exact, cert, f, "ok", r["rounds"], round(time.time() - t0, 2), flush=True)
    except Exception as e:
        print(d, n, m, exact, cert, f, "FAIL", e, round(time.time() - t0, 2), flush=True)
