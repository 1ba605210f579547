"""Developer: wall time of repeated duhl_create calls in the bench's launch configuration.
python tools/create_timing.py [c2] [reps]"""
import os, sys, time
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import bench, paper_1708_05357_b200 as D
name = sys.argv[1] if len(sys.argv) > 1 else "c2"
reps = int(sys.argv[2]) if len(sys.argv) > 2 else 5
args, cfg = bench.parse_args(["--config", name])
kw = bench.launch_kwargs(args, cfg)
A, lab = bench.make_data(cfg, kw["seed"])
lam = bench.lam_of(cfg, A, lab)
bench.pin_host(A)
solve = len(sys.argv) > 3 and sys.argv[3] == "solve"
for r in range(reps):
    t0 = time.perf_counter()
    P = D.create(A, lab, lam, cfg["model"], scd_exact=args.exact, **kw)
    t1 = time.perf_counter()
    if solve:
        P.solve(1e-5, 1000, passes=args.passes)
    t2 = time.perf_counter()
    P.close()
    print(name, "create", round(t1 - t0, 4), "solve", round(t2 - t1, 4), "close", round(time.perf_counter() - t2, 4),
          flush=True)
