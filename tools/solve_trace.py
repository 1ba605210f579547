"""Round-by-round trace of a C4 duhl_solve (time, swaps, certificates)."""
import os, sys, time
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import bench, paper_1708_05357_b200 as D
cfg = bench.CONFIGS["c4"]
A, lab = bench.make_data(cfg, 170805360)
budget = int(0.25 * cfg["n"] * ((cfg["d"] + 3) // 4) * 16)
f = float(os.environ.get("REFRESH", "0.1"))
t0 = time.perf_counter()
P = D.create(A, lab, 1.0 / cfg["n"], 1, hbm_budget_bytes=budget, m=cfg["m"], refresh_fraction=f,
             borrow_host=True, scd_exact=False, cert_every=50, profile=True)
print("create", round(time.perf_counter() - t0, 2), file=sys.stderr)
r = P.solve(1e-5, 1000, passes=int(os.environ.get("PASSES", "1")))
prev = 0.0
for t in r["trace"]:
    print(t.round, "swaps", t.swaps, "dt_ms", round(1e3 * (t.time_s - prev), 1), "cert", t.cert_gap,
          "zsum", round(t.z_sum, 8), file=sys.stderr)
    prev = t.time_s
for k, nm in enumerate(["scd", "gap", "topm", "stage", "refresh"]):
    n_, ms, by = P.kernel_stats(k)
    if n_: print(nm, n_, "launches", round(ms, 1), "ms total", round(by / ms / 1e6, 1), "GB/s", file=sys.stderr)
print("solve", r["status"], r["rounds"], r["gap"], round(prev, 2), file=sys.stderr)
