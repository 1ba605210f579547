"""Time to certified gap 1e-5 with the exact Gram-block epoch vs the asynchronous TPA-style epoch
(cfg.scd_async, W coordinates in flight) in the bench's launch configuration.
    python tools/tpa_vs_exact.py c4 [W ...]     (W = 0: the exact kernel)"""
import json, os, sys, time
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import bench, paper_1708_05357_b200 as D
name = sys.argv[1] if len(sys.argv) > 1 else "c4"
Ws = [int(x) for x in sys.argv[2:]] or [0, 8, 16, 32]
args, cfg = bench.parse_args(["--config", name])
kw = bench.launch_kwargs(args, cfg)
A, lab = bench.make_data(cfg, kw["seed"])
lam = bench.lam_of(cfg, A, lab)
bench.pin_host(A)
out = []
for W in Ws:
    kw2 = dict(kw, scd_async=W > 0, scd_block=W)
    P = D.create(A, lab, lam, cfg["model"], cert_every=1 << 30, scd_exact=False, profile=True, **kw2)
    shape = P.scd_shape()
    t0 = time.perf_counter()
    r = P.solve(1e-5, 1500, passes=args.passes)
    t = time.perf_counter() - t0
    n0, ms0, by0 = P.kernel_stats(0)
    n5, ms5, by5 = P.kernel_stats(5)
    P.close()
    rec = dict(config=name, kernel=shape[0], W=shape[1], G=shape[2], R=shape[3], passes=args.passes,
               rounds=r["rounds"], status=r["status"], gap=r["gap"], time_to_eps_s=t,
               scd_ms_per_pass=(ms0 + ms5) / max(1, n0 + n5))
    print(json.dumps(rec), flush=True)
    out.append(rec)
os.makedirs("gpurun_out", exist_ok=True)
json.dump(out, open(f"gpurun_out/tpa_vs_exact_{name}.json", "w"), indent=1)
