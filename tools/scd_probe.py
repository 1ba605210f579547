"""SCD kernel time per launch on a bench config for several (W, G) shapes.

    CONFIG=c3 SHAPES="0x0,16x74,16x37" EXACT=0 python tools/scd_probe.py
"""
import os, sys, time
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import bench, paper_1708_05357_b200 as D
cfg = bench.CONFIGS[os.environ.get("CONFIG", "c4")]
seed = 170805357 + 3
A, lab = bench.make_data(cfg, seed)
lam = bench.lam_of(cfg, A, lab)
n, d = A.shape
col_bytes = ((d + 3) // 4) * 16
exact = bool(int(os.environ.get("EXACT", "0")))
for shape in os.environ.get("SHAPES", "0x0").split(","):
    W, G = (int(x) for x in shape.split("x"))
    P = D.create(A, lab, lam, cfg["model"], hbm_budget_bytes=int(cfg["budget_frac"] * n * col_bytes),
                 m=cfg["m"], refresh_fraction=0.0, borrow_host=True, profile=True, scd_exact=exact,
                 scd_block=W, scd_ctas=G, seed=seed)
    for t in range(3):
        P.round(t)
    c0, ms0, by0 = P.kernel_stats(0)
    P.scd_epoch(passes=3, round=100)
    c1, ms1, by1 = P.kernel_stats(0)
    ms = (ms1 - ms0) / (c1 - c0)
    print("shape W=%d G=%d: scd %.3f ms/pass, %.1f GB/s" % (W, G, ms, (by1 - by0) / (c1 - c0) / ms / 1e6),
          flush=True)
    P.close()
