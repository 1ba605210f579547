"""SCD kernel time inside a C4 round vs back-to-back epochs on the same working set."""
import os, sys, time
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import bench, paper_1708_05357_b200 as D
cfg = bench.CONFIGS["c4"]
A, lab = bench.make_data(cfg, 170805360)
n, d = A.shape
f = float(os.environ.get("REFRESH", "0.1"))
P = D.create(A, lab, 1.0 / n, 1, hbm_budget_bytes=int(0.25 * n * d * 4), m=cfg["m"], refresh_fraction=f,
             borrow_host=True, profile=True)
def scd_delta(fn):
    c0, ms0, _ = P.kernel_stats(0)
    fn()
    c1, ms1, _ = P.kernel_stats(0)
    return (ms1 - ms0) / max(1, c1 - c0)
for t in range(8):
    print("round %d: scd %.2f ms/launch" % (t, scd_delta(lambda: P.round(t))), flush=True)
for k in range(3):
    print("epoch after round: scd %.2f ms/launch" % scd_delta(lambda: P.scd_epoch(passes=1, round=100 + k)), flush=True)
print("3-pass epoch: scd %.2f ms/launch" % scd_delta(lambda: P.scd_epoch(passes=3, round=200)), flush=True)
