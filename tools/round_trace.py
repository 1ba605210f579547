"""Developer: DUHL_ROUND_TRACE phase timing of a few rounds in the bench's launch configuration.
python tools/round_trace.py [c5s] [rounds]"""
import os, sys
os.environ["DUHL_ROUND_TRACE"] = "1"
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import bench, paper_1708_05357_b200 as D
name = sys.argv[1] if len(sys.argv) > 1 else "c5s"
rounds = int(sys.argv[2]) if len(sys.argv) > 2 else 12
args, cfg = bench.parse_args(["--config", name])
kw = bench.launch_kwargs(args, cfg)
A, lab = bench.make_data(cfg, kw["seed"])
lam = bench.lam_of(cfg, A, lab)
P = bench.create(D, A, lab, lam, cfg["model"], cert_every=1 << 30, scd_exact=args.exact, **kw)
for t in range(rounds):
    P.round(t, passes=args.passes)
P.close()
