"""C3 time to 1e-5 with the asynchronous epoch over (W, passes) in the bench's launch."""
import json, os, sys, time
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import bench, paper_1708_05357_b200 as D
args, cfg = bench.parse_args(["--config", "c3"])
kw = bench.launch_kwargs(args, cfg)
A, lab = bench.make_data(cfg, kw["seed"])
lam = bench.lam_of(cfg, A, lab)
bench.pin_host(A)
out = []
for spec in (sys.argv[1:] or ["128:3", "140:3", "128:2", "128:4", "140:2"]):
    W, passes = (int(x) for x in spec.split(":"))
    P = D.create(A, lab, lam, cfg["model"], cert_every=1 << 30, scd_exact=False, **dict(kw, scd_block=W))
    t0 = time.perf_counter()
    r = P.solve(1e-5, 1000, passes=passes)
    t = time.perf_counter() - t0
    P.close()
    rec = dict(W=W, passes=passes, rounds=r["rounds"], status=r["status"], gap=r["gap"], time_s=t)
    print(json.dumps(rec), flush=True)
    out.append(rec)
json.dump(out, open("gpurun_out/c3_tpa_sweep.json", "w"), indent=1)
