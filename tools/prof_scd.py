"""Profiling driver: C4-shaped SCD epoch + gap pass on an all-resident working set.

python tools/prof_scd.py [--d 200704] [--n 10000] [--passes 2] [--W 0]
"""
import argparse
import os
import sys
import time

import numpy as np

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_1708_05357_b200 as D  # noqa: E402
import synth  # noqa: E402

ap = argparse.ArgumentParser()
ap.add_argument("--d", type=int, default=200704)
ap.add_argument("--n", type=int, default=10000)
ap.add_argument("--passes", type=int, default=2)
ap.add_argument("--W", type=int, default=0)
ap.add_argument("--ctas", type=int, default=0)
ap.add_argument("--lasso", action="store_true")
ap.add_argument("--fast", action="store_true")
ap.add_argument("--kernel", type=int, default=0, help="0 auto, 1 warp-specialised, 2 pipelined")
ap.add_argument("--async_W", type=int, default=0, help="> 0: the asynchronous TPA-style epoch with W in flight")
a = ap.parse_args()
if a.lasso:
    A = np.empty((a.n, a.d), dtype=np.float32)
    synth.lasso_fill(A, a.d, a.n, 5)
    lab = synth.lasso_labels(A, a.d, 5)
    model, lam = D.LASSO, 0.05
else:
    A = np.empty((a.n, a.d), dtype=np.float32)
    lab = synth.svm_fill(A, a.d, a.n, 5)
    model, lam = D.SVM_DUAL, 1.0 / 40000
P = D.create(A, lab, lam, model, profile=True, scd_ctas=a.ctas, borrow_host=True,
             **({} if a.async_W else {"scd_block": a.W}),
             scd_exact=not a.fast, scd_kernel=a.kernel, scd_async=a.async_W > 0, **({"scd_block": a.async_W} if a.async_W else {}))
P.select(D.SEL_GAP, m=a.n)
t0 = time.perf_counter()
P.scd_epoch(passes=a.passes, seed=1)
t1 = time.perf_counter()
P.gaps()
for k, name in enumerate(["scd", "gap", "topm", "stage"]):
    n, ms, by = P.kernel_stats(k)
    if n:
        print(f"{name}: {n} launches, {ms / n:.3f} ms/launch, {by / ms / 1e6:.1f} GB/s algorithmic")
print(f"wall scd {1e3 * (t1 - t0) / a.passes:.2f} ms/pass")
