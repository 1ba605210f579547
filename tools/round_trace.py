"""Developer timing of C4 DuHL rounds (DUHL_ROUND_TRACE / DUHL_SCD_TRACE)."""
import os, sys, time
import numpy as np
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import bench, paper_1708_05357_b200 as D
cfg = bench.CONFIGS["c4"]
A, lab = bench.make_data(cfg, 170805360)
f = float(os.environ.get("REFRESH", "0.01"))
P = D.create(A, lab, 1.0 / cfg["n"], 1, hbm_budget_bytes=int(0.25 * cfg["n"] * cfg["d"] * 4), m=10000,
             refresh_fraction=f, borrow_host=True, profile=True, scd_exact=False)
for t in range(int(sys.argv[1]) if len(sys.argv) > 1 else 30):
    r = P.round(t)
    print(t, "swaps", r.swaps, "time_ms", round(1e3 * r.time_s, 2), file=sys.stderr)

for k, nm in enumerate(["scd", "gap", "topm", "stage", "refresh"]):
    n_, ms, by = P.kernel_stats(k)
    if n_: print(nm, n_, round(ms / n_, 3), "ms/launch", round(by / ms / 1e6, 1), "GB/s", file=sys.stderr)
