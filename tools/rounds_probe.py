"""Rounds / time to 1e-5 of repeated C4 solves (bench launch) under the current environment."""
import os, sys, time, json
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np
import bench, paper_1708_05357_b200 as D, oracle as O
args, cfg = bench.parse_args(["--config", os.environ.get("CFG", "c4")])
kw = bench.launch_kwargs(args, cfg)
A, lab = bench.make_data(cfg, kw["seed"])
lam = bench.lam_of(cfg, A, lab)
bench.pin_host(A)
for rep in range(int(os.environ.get("REPS", "2"))):
    P = D.create(A, lab, lam, cfg["model"], cert_every=1 << 30, scd_exact=False, **kw)
    t0 = time.perf_counter()
    r = P.solve(1e-5, 300, passes=args.passes)
    t = time.perf_counter() - t0
    a, v, _ = P.get_state()
    P.close()
    nz = np.flatnonzero(a)
    vv = O.matvec(np.ascontiguousarray(A[nz]), a[nz]) - (lab if cfg["model"] == 0 else 0.0) if len(nz) < 20000 else None
    err = None if vv is None else float(np.abs(v - vv).max())
    print(json.dumps(dict(env=os.environ.get("DUHL_STAGE_CE_SHARE"), rep=rep, rounds=r["rounds"], time_s=t, gap=r["gap"],
                          certs=sum(1 for x in r["trace"] if x.cert_gap >= 0), v_err=err)), flush=True)
