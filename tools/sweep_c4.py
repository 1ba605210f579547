"""Time-to-eps sweep over refresh fraction and passes per round (gap policy), in the bench's
launch configuration (bench.parse_args + launch_kwargs: host unit-A threads, fast-mode SCD,
gather staging overlapping the epoch).
Usage: python tools/sweep_c4.py [--config c3] f:p [f:p ...]   (default config c4)"""
import json, os, sys, time
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import bench, paper_1708_05357_b200 as D
argv = sys.argv[1:]
cname = "c4"
if argv[:1] == ["--config"]:
    cname, argv = argv[1], argv[2:]
args, cfg = bench.parse_args(["--config", cname])
kw = bench.launch_kwargs(args, cfg)
A, lab = bench.make_data(cfg, kw["seed"])
lam = bench.lam_of(cfg, A, lab)
grid = [tuple(float(x) for x in a.split(":")) for a in argv] or [(0.05, 2), (0.1, 2)]
out = []
for f, passes in grid:
    kw2 = dict(kw, refresh_fraction=f)
    P = D.create(A, lab, lam, cfg["model"], cert_every=1 << 30, scd_exact=False, **kw2)
    t0 = time.perf_counter()
    r = P.solve(1e-5, 1000, passes=int(passes))
    t = time.perf_counter() - t0
    c = P.counters()
    P.close()
    rec = dict(config=cname, refresh=f, passes=int(passes), rounds=r["rounds"], status=r["status"], gap=r["gap"], time_s=t,
               ms_per_round=1e3 * t / max(1, r["rounds"]), h2d_GB=c["h2d_bytes"] / 1e9)
    print(json.dumps(rec), flush=True)
    out.append(rec)
os.makedirs("gpurun_out", exist_ok=True)
json.dump(out, open(f"gpurun_out/sweep_{cname}.json", "w"), indent=1)
