timeout 900 python -m pytest tests -m gpu -x -q > gpurun_out/pytest_gpu.log 2>&1; echo rc=$? >> gpurun_out/pytest_gpu.log
PASSES=3 timeout 600 python - > gpurun_out/strace_c3.log 2>&1 <<'PY'
import os, sys, time
sys.path.insert(0, os.getcwd())
import bench, paper_1708_05357_b200 as D
cfg = bench.CONFIGS["c3"]
A, lab = bench.make_data(cfg, 170805360)
lam = bench.lam_of(cfg, A, lab)
n, d = A.shape
budget = int(0.25 * n * ((d + 3) // 4) * 16)
t0 = time.perf_counter()
P = D.create(A, lab, lam, 0, hbm_budget_bytes=budget, m=cfg["m"], refresh_fraction=0.1,
             borrow_host=True, scd_exact=False, cert_every=50, profile=True)
print("create", round(time.perf_counter() - t0, 2), P.scd_shape())
r = P.solve(1e-5, 1000, passes=3)
prev = 0.0
for t in r["trace"]:
    if t.cert_gap >= 0 or t.round % 10 == 0:
        print(t.round, "swaps", t.swaps, "dt_ms", round(1e3 * (t.time_s - prev), 1), "cert", t.cert_gap, "zsum", t.z_sum)
    prev = t.time_s
print("solve", r["status"], r["rounds"], r["gap"], round(prev, 2))
PY
timeout 900 compute-sanitizer --tool memcheck --error-exitcode 9 python -m pytest tests/test_gpu_parity.py -x -q -k "explicit_order and (2-0-300 or 2-1-300 or 2-2-40000 or 1-0-300)" > gpurun_out/memcheck.log 2>&1; echo rc=$? >> gpurun_out/memcheck.log
