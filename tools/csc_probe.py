"""Sparse (CSC) DuHL: rounds/time to a certified gap vs the async epoch's concurrency.

    python tools/csc_probe.py [d n density model] [warps,...]
"""
import os, sys, time
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np
import paper_1708_05357_b200 as D
import synth

d, n, dens, model = 40000, 200000, 0.01, 0
if len(sys.argv) > 4:
    d, n, dens, model = int(sys.argv[1]), int(sys.argv[2]), float(sys.argv[3]), int(sys.argv[4])
warps = [int(x) for x in (sys.argv[5] if len(sys.argv) > 5 else "0,128,512,2048,8192").split(",")]
t0 = time.time()
cp, rows, vals = synth.csc_lasso(d, n, seed=77, density=dens)
if model == 0:
    lab = synth.lasso_finish(synth.csc_lasso_signal(cp, rows, vals, d, 77, support=0.002), d, 77)
    s = np.abs(np.add.reduceat(vals.astype(np.float64) * lab[rows], cp[:-1])) * (np.diff(cp) > 0)
    lam = 0.1 * s.max() / d
else:
    lab = synth.svm_labels(n, 77)[1]
    lam = 1.0 / n
print(f"gen {time.time() - t0:.1f}s nnz {cp[-1]} lam {lam:.3e}", flush=True)
for w in warps:
    for ls in (False, True):
        with D.create_csc(cp, rows, vals, d, lab, lam, model, m=n // 4, refresh_fraction=0.1, cert_every=10,
                          scd_exact=False, scd_ctas=w, linesearch=ls, profile=True) as P:
            t1 = time.time()
            r = P.solve(1e-5, 3000, passes=1)
            dt = time.time() - t1
            c, ms, by = P.kernel_stats(0)
            print(f"warps {w:6d} ls {int(ls)}: status {r['status']} rounds {r['rounds']} gap {r['gap']:.2e} "
                  f"solve {dt:.2f}s scd {ms / max(c, 1):.3f} ms/pass {by / max(ms, 1e-9) / 1e6:.0f} GB/s", flush=True)
