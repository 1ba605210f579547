"""Time-to-eps sweep on C4 over refresh fraction and passes (gap policy)."""
import json, os, sys, time
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import bench, paper_1708_05357_b200 as D
cfg = bench.CONFIGS["c4"]
A, lab = bench.make_data(cfg, 170805360)
budget = int(0.25 * cfg["n"] * ((cfg["d"] + 3) // 4) * 16)
out = []
for f, passes in [(0.01, 1), (0.02, 1), (0.05, 1), (0.02, 2), (0.05, 2), (0.1, 1)]:
    t0 = time.perf_counter()
    P = D.create(A, lab, 1.0 / cfg["n"], 1, hbm_budget_bytes=budget, m=cfg["m"], refresh_fraction=f,
                 borrow_host=True, scd_exact=False, cert_every=50)
    tc = time.perf_counter() - t0
    r = P.solve(1e-5, 1000, passes=passes)
    t = time.perf_counter() - t0
    c = P.counters()
    P.close()
    rec = dict(refresh=f, passes=passes, rounds=r["rounds"], status=r["status"], gap=r["gap"], time_s=t,
               create_s=tc, h2d_GB=c["h2d_bytes"] / 1e9)
    print(json.dumps(rec), flush=True)
    out.append(rec)
json.dump(out, open("gpurun_out/sweep_c4.json", "w"), indent=1)
