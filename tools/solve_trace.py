"""Round-by-round trace of a duhl_solve in the bench's launch configuration (time, swaps,
certificates, gamma) plus per-kind kernel time.   python tools/solve_trace.py [c4|c3|c5|c5s]"""
import os, sys, time
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import bench, paper_1708_05357_b200 as D
name = sys.argv[1] if len(sys.argv) > 1 else "c4"
args, cfg = bench.parse_args(["--config", name] + sys.argv[2:])
kw = bench.launch_kwargs(args, cfg)
A, lab = bench.make_data(cfg, kw["seed"])
lam = bench.lam_of(cfg, A, lab)
if not cfg.get("sparse"):
    bench.pin_host(A)
t0 = time.perf_counter()
P = bench.create(D, A, lab, lam, cfg["model"], cert_every=args.cert_every, scd_exact=args.exact, profile=True, **kw)
print("create", round(time.perf_counter() - t0, 2), "shape", P.scd_shape(), file=sys.stderr)
t0 = time.perf_counter()
r = P.solve(1e-5, 1000, passes=args.passes)
wall = time.perf_counter() - t0
prev = 0.0
for t in r["trace"]:
    print(t.round, "swaps", t.swaps, "dt_ms", round(1e3 * (t.time_s - prev), 1), "cert", round(t.cert_gap, 9),
          "zsum", round(t.z_sum, 8), "gamma", round(t.gamma, 3), file=sys.stderr)
    prev = t.time_s
for k, nm in enumerate(["scd", "gap", "topm", "stage", "refresh", "scd_staged"]):
    n_, ms, by = P.kernel_stats(k)
    if n_: print(nm, n_, "launches", round(ms, 1), "ms total", round(by / ms / 1e6, 1), "GB/s", file=sys.stderr)
print("solve", r["status"], r["rounds"], r["gap"], "wall", round(wall, 3), file=sys.stderr)
