"""Developer timing of C3 rounds (DUHL_ROUND_TRACE host phases)."""
import os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import bench, paper_1708_05357_b200 as D
cfg = bench.CONFIGS[os.environ.get("CONFIG", "c3")]
A, lab = bench.make_data(cfg, 170805360)
lam = bench.lam_of(cfg, A, lab)
n, d = A.shape
budget = int(0.25 * n * ((d + 3) // 4) * 16)
P = D.create(A, lab, lam, cfg["model"], hbm_budget_bytes=budget, m=cfg["m"], refresh_fraction=0.1,
             borrow_host=True, scd_exact=False, profile=True, unit_a_ctas=int(os.environ.get("UNIT_A", "0")))
prev = [P.kernel_stats(k)[1] for k in range(5)]
for t in range(int(sys.argv[1]) if len(sys.argv) > 1 else 40):
    r = P.round(t, passes=cfg.get("passes", 1))
    cur = [P.kernel_stats(k)[1] for k in range(5)]
    dk = [round(c - p_, 2) for c, p_ in zip(cur, prev)]
    prev = cur
    print(t, "swaps", r.swaps, "time_ms", round(1e3 * r.time_s, 2), "kernel ms scd/gap/topm/stage/refresh", dk,
          file=sys.stderr)
