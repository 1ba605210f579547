"""Where does a C4 round's time go?  Certificate (zero-copy gap pass alone), rounds
with/without refresh, per-kernel stats."""
import os, sys, time
import numpy as np
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch
import bench, paper_1708_05357_b200 as D
cfg = bench.CONFIGS["c4"]
A, lab = bench.make_data(cfg, 170805360)
n, d = A.shape
x = torch.empty(int(2e9) // 4, dtype=torch.float32).pin_memory()
g = torch.empty_like(x, device="cuda")
for _ in range(2): g.copy_(x, non_blocking=True)
torch.cuda.synchronize(); t = time.perf_counter()
for _ in range(5): g.copy_(x, non_blocking=True)
torch.cuda.synchronize(); print("DMA H2D alone %.1f GB/s" % (5 * 2e9 / (time.perf_counter() - t) / 1e9))
del x, g
for f in [float(v) for v in os.environ.get("REFRESH", "0.1,0.0").split(",")]:
    P = D.create(A, lab, 1.0 / n, 1, hbm_budget_bytes=int(0.25 * n * d * 4), m=cfg["m"], refresh_fraction=f,
                 borrow_host=True, profile=True)
    for t in range(5): P.round(t)
    base = [P.kernel_stats(k) for k in range(5)]
    t0 = time.perf_counter(); P.duality_gap(); tc = time.perf_counter() - t0
    gs = P.kernel_stats(1)
    print("refresh %.2f: certificate %.1f ms (%.1f GB/s over all columns); gap kernel %.1f ms" %
          (f, tc * 1e3, n * d * 4 / tc / 1e9, gs[1] - base[1][1]))
    base = [P.kernel_stats(k) for k in range(5)]
    t0 = time.perf_counter()
    R = 10
    for t in range(5, 5 + R): r = P.round(t)
    tr = (time.perf_counter() - t0) / R
    print("  round %.1f ms" % (tr * 1e3))
    for k, nm in enumerate(["scd", "gap", "topm", "stage", "refresh"]):
        c, ms, by = P.kernel_stats(k)
        c -= base[k][0]; ms -= base[k][1]; by -= base[k][2]
        if c: print("  %-8s %4d launches %8.2f ms/round %7.1f GB/s" % (nm, c, ms / R, by / ms / 1e6 if ms else 0))
    P.close()
