"""Developer check: after every DuHL round of the C4 bench launch, v (library) against A alpha
recomputed in fp64 with torch on the GPU; reports the first round where they disagree."""
import os, sys, json
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np
import torch
import bench, paper_1708_05357_b200 as D
args, cfg = bench.parse_args(["--config", os.environ.get("CFG", "c4")])
kw = bench.launch_kwargs(args, cfg)
A, lab = bench.make_data(cfg, kw["seed"])
lam = bench.lam_of(cfg, A, lab)
bench.pin_host(A)
At = torch.from_numpy(A)   # (n, d) pinned, float32


def v_ref(alpha):
    nz = np.flatnonzero(alpha)
    out = torch.zeros(A.shape[1], dtype=torch.float64, device="cuda")
    for k in range(0, len(nz), 2048):
        idx = torch.from_numpy(nz[k:k + 2048])
        blk = At.index_select(0, idx).cuda().double()
        out += blk.t() @ torch.from_numpy(alpha[nz[k:k + 2048]]).cuda()
    r = out.cpu().numpy()
    return r - lab if cfg["model"] == 0 else r


CERT_AT = {int(x) for x in os.environ.get("CERT_AT", "").split(",") if x}
for rep in range(int(os.environ.get("REPS", "2"))):
    P = D.create(A, lab, lam, cfg["model"], cert_every=1 << 30, scd_exact=False, **kw)
    bad = None
    for t in range(int(os.environ.get("ROUNDS", "24"))):
        certify = t in CERT_AT
        rec = P.round(t, passes=args.passes, certify=certify)
        if os.environ.get("NOSYNC") and t + 1 < int(os.environ.get("ROUNDS", "24")):
            continue
        a, v, _ = P.get_state()
        err = float(np.abs(v - v_ref(a)).max())
        print(json.dumps(dict(rep=rep, t=t, swaps=rec.swaps, cert=rec.cert_gap, err=err)), flush=True)
        if err > 1e-8:
            bad = t
            break
    P.close()
    print("REP", rep, "first bad round", bad, flush=True)
