#!/usr/bin/env python
"""bench.py -- the DuHL hot path (arXiv 1708.05357) on B200.

One step = one DuHL round (Algorithm 2) over the configured workload:
gap-memory top-m selection (Eq. 11) -> staging of A_[P] host -> HBM under the
budget -> unit-A refresh of a rotating fraction of the gaps (zero-copy from
pinned host memory) -> `passes` exact SCD passes over the working set (App. D;
per-config default: C4 2, C3 5 -- they run in the shadow of the PCIe-bound
refresh) -> refresh of z_P.  The metric is BASELINE.json's: coordinate updates/s (plus
time-to-certified-gap and gap-pass GB/s as extra keys).

    python bench.py [--gpus N --steps K --warmup W] [--config c4|c2|c1] [--impl reference]

Default workload C4 (BASELINE.json configs[3], the config the metric is quoted
on at 1/2/4/8 GPUs): hinge-SVM dual, 200,704 features x 40,000 samples dense
fp32 (32.1 GB in pinned host memory), HBM budget 25% (8.03 GB, m = 10,000).
"""
from __future__ import annotations

import argparse
import json
import os
import statistics
import subprocess
import sys
import threading
import time

import numpy as np

ROOT = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, ROOT)

METRIC = json.load(open(os.path.join(ROOT, "BASELINE.json")))["metric"]
PEAKS_PATH = os.path.join(ROOT, "MEASURED_PEAKS.json")
HBM_FALLBACK = 6650.0  # GB/s, B200_PROFILING.md fallback

CONFIGS = {
    # name: model, d, n, budget fraction of data (0 = all resident), m, lambda (None: 1/n), label
    # passes: SCD passes per round (tuned per scheme): the epoch runs in the shadow of the
    # PCIe-bound unit-A refresh, so extra passes are free until they outlast it (measured sweep:
    # C4 time-to-eps 5.5 / 4.8 / 6.2 s at 1 / 2 / 4 passes; C3 14.2 / 8.1 / 6.6 s at 1 / 2 / 3, and
    # with adaptive-only certificates (tools/c3_sweep.py) 6.1 / 5.2 / 4.9 / 5.2 s at 3 / 4 / 5 / 6)
    # with host threads in unit A (--unit-a-host) the refresh no longer hides the epoch: C3 4.3 s at
    # 2 and 3 passes, 5.1 s at 4 (passes_host); re-swept with the asynchronous epoch and the pool
    # prefill (tools/sweep_c4.py --config c3, profiles/r02_sweep_c3.json): refresh 0.1 at 2 / 3 / 4 /
    # 5 / 6 passes 3.23 / 2.71 / 2.57-2.60 / 2.65 / 2.70 s; 0.05 / 0.07 / 0.15 at 3 passes 2.98 /
    # 2.74 / 3.07 s; with the gather staging C3's heavy rounds (profiles/r02_sweep_c3_gather.json)
    # 3 / 4 / 5 passes 2.03 / 1.91 / 1.93 s, refresh 0.08 / 0.12 at 4 passes 1.99 / 1.99 s
    # C3 runs the asynchronous TPA-style epoch (scd_async, 128 coordinates in flight): time to 1e-5
    # 3.16 s vs 3.90 s with the exact k_scd_pipe (profiles/r02_tpa_vs_exact_c3.json); C4 keeps the
    # exact kernel (k_scd_gram then: 2.62 s vs 3.27 s async at W = 16; W >= 32 stalls on C4's correlated samples)
    "c3": dict(model=0, d=40000, n=200704, budget_frac=0.25, m=50176, lam=None, lam_rel=0.07, passes=5,
               passes_host=4, scd_async=True, scd_block=128,
               label="C3: Lasso, ImageNet-shaped dense synthetic 40000 samples x 200704 features fp32 "
                     "(32.1 GB pinned host), HBM budget 25% (8.03 GB), m=50176, lambda=0.07 lambda_max"),
    "c4": dict(model=1, d=200704, n=40000, budget_frac=0.25, m=10000, lam=None, passes=2,
               label="C4: hinge-SVM dual, ImageNet-shaped dense synthetic 200704 features x 40000 "
                     "samples fp32 (32.1 GB pinned host), HBM budget 25% (8.03 GB), m=10000"),
    "c5": dict(model=0, sparse=True, d=40000, n=10_000_000, density=0.01, budget_frac=0.0, m=2_500_000,
               lam=None, lam_rel=0.1, support=0.002,
               label="C5: sparse Lasso, CSC synthetic 40000 samples x 10M features, 1% density (4e9 nonzeros, "
                     "32 GB), resident in HBM, m=25% of local columns, lambda=0.1 lambda_max"),
    "c5s": dict(model=0, sparse=True, d=40000, n=1_250_000, density=0.01, budget_frac=0.0, m=312_500,
                lam=None, lam_rel=0.1, support=0.002,
                label="C5 shard: sparse Lasso, CSC 40000 samples x 1.25M features (one of C5's 8 feature "
                      "blocks), 1% density, resident, m=25%, lambda=0.1 lambda_max"),
    "c2": dict(model=1, d=500, n=20000, budget_frac=0.0, m=2000, lam=None,
               label="C2: hinge-SVM dual, dense synthetic 500 features x 20000 samples, m=10%"),
    "c1": dict(model=0, d=2000, n=1000, budget_frac=0.0, m=250, lam=0.1,
               label="C1: Lasso, dense synthetic 2000 samples x 1000 features, lambda=0.1, m=25%"),
}


def hbm_peak():
    try:
        return float(json.load(open(PEAKS_PATH))["hbm_gbs"]), "measured (MEASURED_PEAKS.json)"
    except Exception:
        return HBM_FALLBACK, "fallback (B200_PROFILING.md)"


# ------------------------------------------------------------------ distributed plumbing
def dist_init(n_gpus):
    rank = int(os.environ.get("RANK", "0"))
    world = int(os.environ.get("WORLD_SIZE", "1"))
    local = int(os.environ.get("LOCAL_RANK", "0"))
    if world != n_gpus:
        # one process per GPU: N > 1 must be launched by torchrun (WORLD_SIZE = N); a mismatch
        # would silently measure a different GPU count
        raise SystemExit(f"bench.py: --gpus {n_gpus} but WORLD_SIZE={world}; launch N > 1 with "
                         f"python -m torch.distributed.run --nproc-per-node {n_gpus} bench.py --gpus {n_gpus}")
    if world > 1:
        import torch
        import torch.distributed as dist
        torch.cuda.set_device(local)
        dist.init_process_group("nccl", device_id=torch.device("cuda", local))
    return rank, world, local


def numa_bind(local):
    """Restrict this rank (and the threads it starts: data generation, the library's ingest
    and host unit-A threads) to the CPUs of its GPU's NUMA node, so the pinned host shard is
    first-touched there and unit A reads local DRAM.  Returns the node, or None when the
    topology is not exposed (single-node boxes, containers)."""
    try:
        import torch
        pr = torch.cuda.get_device_properties(local)
        bus = f"{pr.pci_domain_id:04x}:{pr.pci_bus_id:02x}:{pr.pci_device_id:02x}.0"
        node = int(open(f"/sys/bus/pci/devices/{bus}/numa_node").read().strip())
        if node < 0:
            return None
        cpus = set()
        for part in open(f"/sys/devices/system/node/node{node}/cpulist").read().strip().split(","):
            lo, _, hi = part.partition("-")
            cpus.update(range(int(lo), int(hi or lo) + 1))
        cpus &= os.sched_getaffinity(0)
        if not cpus:
            return None
        os.sched_setaffinity(0, cpus)
        return node
    except Exception:
        return None


def barrier(world):
    if world > 1:
        import torch.distributed as dist
        dist.barrier()


def max_over_ranks(x, world):
    if world == 1:
        return x
    import torch
    import torch.distributed as dist
    t = torch.tensor([x], dtype=torch.float64, device="cuda")
    dist.all_reduce(t, op=dist.ReduceOp.MAX)
    return float(t.item())


# ------------------------------------------------------------------ clocks
class ClockSampler:
    """nvidia-smi clocks + throttle reasons sampled during the timed region."""
    Q = ("clocks.sm,clocks.max.sm,clocks_event_reasons.hw_slowdown,"
         "clocks_event_reasons.hw_thermal_slowdown,clocks_event_reasons.sw_thermal_slowdown,"
         "clocks_event_reasons.sw_power_cap,utilization.gpu")

    def __init__(self, device):
        self.device = device
        self.rows = []
        self._stop = threading.Event()
        self._t = threading.Thread(target=self._run, daemon=True)

    def _run(self):
        while not self._stop.is_set():
            try:
                out = subprocess.run(["nvidia-smi", f"--id={self.device}", f"--query-gpu={self.Q}",
                                      "--format=csv,noheader,nounits"], capture_output=True,
                                     text=True, timeout=5).stdout.strip()
                if out:
                    self.rows.append([c.strip() for c in out.split(",")])
            except Exception:
                pass
            self._stop.wait(0.2)

    def __enter__(self):
        self._t.start()
        return self

    def __exit__(self, *a):
        self._stop.set()
        self._t.join(timeout=10)

    def summary(self):
        if not self.rows:
            return {"sm_mhz": None, "sm_max_mhz": None, "reasons": ["unsampled"], "samples": 0}
        sm = [float(r[0]) for r in self.rows if r[0].replace(".", "").isdigit()]
        mx = [float(r[1]) for r in self.rows if r[1].replace(".", "").isdigit()]
        names = ["hw_slowdown", "hw_thermal_slowdown", "sw_thermal_slowdown", "sw_power_cap"]
        reasons = sorted({names[k] for r in self.rows for k in range(4)
                          if len(r) > 2 + k and r[2 + k].lower() == "active"})
        util = [float(r[6]) for r in self.rows if len(r) > 6 and r[6].replace(".", "").isdigit()]
        loaded = [s for s, u in zip(sm, util) if u > 0] or sm
        return {"sm_mhz": statistics.median(loaded) if loaded else None,
                "sm_max_mhz": max(mx) if mx else None, "reasons": reasons, "samples": len(self.rows)}


def pcie_h2d_peak(local):
    """Measured copy-engine H2D bandwidth of this box (1 GiB pinned -> HBM, best of 5)."""
    import torch
    x = torch.empty(1 << 28, dtype=torch.float32).pin_memory()
    g = torch.empty(1 << 28, dtype=torch.float32, device=f"cuda:{local}")
    best = 0.0
    for _ in range(6):
        a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        a.record()
        g.copy_(x, non_blocking=True)
        b.record()
        b.synchronize()
        best = max(best, x.numel() * 4 / (a.elapsed_time(b) / 1e3) / 1e9)
    del x, g
    return best


# ------------------------------------------------------------------ data
def _allreduce_host(x, world, op="sum"):
    """Sum / max of a host float64 array over the ranks (set-up only, not timed)."""
    if world == 1:
        return x
    import torch
    import torch.distributed as dist
    t = torch.from_numpy(np.ascontiguousarray(x, dtype=np.float64)).cuda()
    dist.all_reduce(t, op=dist.ReduceOp.SUM if op == "sum" else dist.ReduceOp.MAX)
    return t.cpu().numpy()


class Sparse:
    """A CSC column block (col_ptr, rows, vals) of a sparse config."""

    def __init__(self, cp, rows, vals, d):
        self.cp, self.rows, self.vals, self.d = cp, rows, vals, d
        self.shape = (cp.size - 1, d)

    def dense(self, ncols):
        import synth
        k = min(ncols, self.shape[0])
        e = self.cp[k]
        return synth.csc_to_dense(self.cp[:k + 1], self.rows[:e], self.vals[:e], self.d)

    def __matmul__(self, b):  # A^T b over the block's columns (lambda_max)
        out = np.add.reduceat(self.vals.astype(np.float64) * b[self.rows], self.cp[:-1])
        return np.where(np.diff(self.cp) > 0, out, 0.0)


def pin_host(A):
    """Page-lock the host matrix once (cudaHostRegister, mapped), as a caller keeping its data in
    pinned memory would; duhl_create(borrow_host=1) then uses it in place.  Returns bytes pinned."""
    if isinstance(A, Sparse):
        return 0
    import torch
    cr = torch.cuda.cudart()
    for flags in (2 | 8, 2):   # cudaHostRegisterMapped | ReadOnly, else Mapped
        if int(cr.cudaHostRegister(A.ctypes.data, A.nbytes, flags)) == 0:
            return A.nbytes
    return 0


def state_check(P, A, lab, cfg):
    """Outside the timed region: the solved state's shared vector against A alpha (- b) recomputed
    in fp64 by torch on the GPU from the host matrix (v is what the certificate used)."""
    if isinstance(A, Sparse):
        return None
    import torch
    a, v, _ = P.get_state()
    nz = np.flatnonzero(a)
    out = torch.zeros(A.shape[1], dtype=torch.float64, device="cuda")
    At = torch.from_numpy(A)
    for k in range(0, len(nz), 2048):
        idx = torch.from_numpy(nz[k:k + 2048])
        out += At.index_select(0, idx).cuda().double().t() @ torch.from_numpy(a[nz[k:k + 2048]]).cuda()
    ref = out.cpu().numpy() - (0.0 if cfg["model"] == 1 else lab)
    return {"max_abs_v_minus_A_alpha": float(np.abs(v - ref).max()), "max_abs_v": float(np.abs(ref).max())}


def rho_mean(trace):
    """Mean rho_{t,P} (Eq. 6) over a solve's rounds (on the gap memory, DESIGN R21)."""
    return float(np.mean([t.rho for t in trace])) if trace else None


def swaps_trend(trace):
    """Mean swaps per round over the first and the last quarter of a solve (Fig. 4b)."""
    if not trace:
        return None
    q = max(1, len(trace) // 4)
    return [float(np.mean([t.swaps for t in trace[:q]])), float(np.mean([t.swaps for t in trace[-q:]]))]


def create(D, A, lab, lam, model, **kw):
    """duhl_create (dense) or duhl_create_csc (sparse) with the bench's options."""
    if isinstance(A, Sparse):
        for k in ("hbm_budget_bytes", "borrow_host", "unit_a_ctas", "unit_a_host_threads", "unit_a_host_share",
                  "scd_async", "scd_block"):
            kw.pop(k, None)
        return D.create_csc(A.cp, A.rows, A.vals, A.d, lab, lam, model, **kw)
    return D.create(A, lab, lam, model, **kw)


def make_data(cfg, seed, col_lo=0, col_hi=None, world=1):
    """The columns [col_lo, col_hi) of the config's matrix and the (global) labels."""
    import synth
    d, n = cfg["d"], cfg["n"]
    col_hi = n if col_hi is None else col_hi
    if cfg.get("sparse"):
        cp, rows, vals = synth.csc_lasso(d, n, seed, density=cfg["density"], col_lo=col_lo, col_hi=col_hi)
        sig = synth.csc_lasso_signal(cp, rows, vals, d, seed, support=cfg["support"], col_lo=col_lo, n_total=n)
        return Sparse(cp, rows, vals, d), synth.lasso_finish(_allreduce_host(sig, world), d, seed)
    A = np.empty((col_hi - col_lo, d), dtype=np.float32)
    if cfg["model"] == 1:
        lab = synth.svm_fill(A, d, n, seed, col_lo=col_lo)
    else:
        synth.lasso_fill(A, d, n, seed, col_lo=col_lo)
        sig = synth.lasso_signal(A, d, seed, col_lo=col_lo, n_total=n)
        lab = synth.lasso_finish(_allreduce_host(sig, world), d, seed)
    return A, lab


def lam_of(cfg, A=None, lab=None, world=1):
    """lambda: given, 1/n (SVM), or lam_rel * lambda_max with lambda_max = ||A^T b||_inf / d."""
    if cfg["lam"] is not None:
        return cfg["lam"]
    if cfg.get("lam_rel") is None:
        return 1.0 / cfg["n"]
    s = np.abs(A @ (lab if isinstance(A, Sparse) else lab.astype(np.float32))).max()
    lmax = float(_allreduce_host(np.array([s], dtype=np.float64), world, "max")[0]) / cfg["d"]
    return cfg["lam_rel"] * lmax


# ------------------------------------------------------------------ oracle arm
def oracle_sample(cfg, A, lab, lam, ncols, passes=1):
    """Time the CPU oracle (single thread, as it stands) on a bounded sample:
    `passes` sequential SCD passes over `ncols` columns of the same data, plus a
    gap pass over them.  Returns (updates/s, gap GB/s, seconds)."""
    import oracle as O
    Asub = A.dense(ncols) if isinstance(A, Sparse) else np.ascontiguousarray(A[:ncols])
    lab_s = lab[:ncols] if cfg["model"] == 1 else lab
    norms = O.col_norms(Asub)
    alpha = np.zeros(ncols)
    vt = np.zeros(cfg["d"]) if cfg["model"] == 1 else -lab_s.copy()
    y = lab_s if cfg["model"] == 1 else None
    order = np.arange(ncols)
    t0 = time.perf_counter()
    for p in range(passes):
        O.scd_pass(cfg["model"], Asub, norms, y, lam, alpha, vt, order)
    t_scd = time.perf_counter() - t0
    w = O.primal_dual_w(cfg["model"], vt if cfg["model"] == 1 else vt + lab_s,
                        None if cfg["model"] == 1 else lab_s, cfg["n"], lam)
    t0 = time.perf_counter()
    O.coord_gaps(cfg["model"], Asub, alpha, y, w, lam, 1.0)
    t_gap = time.perf_counter() - t0
    return passes * ncols / t_scd, ncols * cfg["d"] * 4 / t_gap / 1e9, t_scd + t_gap


def oracle_time_to_eps(cfg, A, lab, lam, eps, cap_s):
    """The oracle as it stands (oracle/duhl_oracle.c, one thread): plain SCD over all n
    coordinates, one permutation per epoch (or_solve_scd's order), certificate after every
    epoch, until gap <= eps or the wall cap.  Unconverged: the gap reached, and an
    extrapolated time to eps from the last epochs' linear rate (flagged)."""
    import oracle as O
    if isinstance(A, Sparse):
        return None
    n = A.shape[0]
    model = cfg["model"]
    B = O.lasso_B(lab, lam) if model == 0 else 0.0
    norms = O.col_norms(A)
    alpha = np.zeros(n)
    vt = np.zeros(cfg["d"]) if model == 1 else -np.asarray(lab, dtype=np.float64).copy()
    y = lab if model == 1 else None
    allc = np.arange(n, dtype=np.int64)
    t0 = time.perf_counter()
    gaps, times, t_scd = [], [], 0.0
    e = 0
    while True:
        t1 = time.perf_counter()
        O.scd_pass(model, A, norms, y, lam, alpha, vt, O.make_perm(allc, 0, e, 0))
        t_scd += time.perf_counter() - t1
        st, g, _, _ = O.duality_gap(model, A, alpha, lab, lam, B)
        e += 1
        gaps.append(g)
        times.append(time.perf_counter() - t0)
        if g <= eps or times[-1] >= cap_s:
            break
    out = {"kind": "oracle", "cores": 1, "eps": eps, "epochs": e, "gap_reached": gaps[-1],
           "wall_s": times[-1], "scd_s": t_scd, "converged": gaps[-1] <= eps,
           "gaps": gaps[:20], "wall_cap_s": cap_s,
           "note": "plain sequential SCD over all n columns (P:406 single-threaded CPU baseline), "
                   "certificate after every epoch (its time included)"}
    out["gap_reached"] = min(gaps)   # the duality gap of an SCD epoch need not decrease monotonically
    if not out["converged"] and len(gaps) >= 3:
        # linear convergence fitted to log(gap) over the epochs run, extrapolated to eps (flagged)
        e_idx = np.arange(1, len(gaps) + 1)
        slope, icpt = np.polyfit(e_idx, np.log(np.maximum(gaps, 1e-300)), 1)
        if slope < 0:
            epochs_eps = (np.log(eps) - icpt) / slope
            out["extrapolated_time_to_eps_s"] = float(epochs_eps * times[-1] / len(gaps))
            out["extrapolated_epochs_to_eps"] = float(epochs_eps)
            out["extrapolated"] = True
    return out


def run_reference(args, cfg, rank, world):
    if rank != 0:
        return
    seed = 170805357 + 3
    ncols = args.ref_cols
    A, lab = (make_data(cfg, seed, 0, ncols) if cfg["model"] == 1 or cfg.get("sparse") else
              make_data(cfg, seed))
    lam = lam_of(cfg, A, lab)
    for _ in range(args.warmup):
        oracle_sample(cfg, A, lab, lam, min(ncols, 64))
    vals, secs = [], 0.0
    for _ in range(args.steps):
        u, g, s = oracle_sample(cfg, A, lab, lam, ncols)
        vals.append(u)
        secs += s
    v = float(np.median(vals))
    sample = (f"per step: 1 sequential SCD pass over {ncols} columns of {args.config.upper()} "
              f"(d={cfg['d']}) + their gap pass, single-threaded C oracle")
    line = {"impl": "reference", "metric": METRIC, "value": v, "unit": "coord updates/s",
            "n_gpus": args.gpus, "steps": args.steps, "warmup": args.warmup,
            "ms_per_step": 1e3 * secs / max(1, args.steps), "higher_is_better": True,
            "scaling": "strong", "vs_baseline": None, "dtype": "f64", "data": "synthetic",
            "config": {"workload": cfg["label"], "oracle_sample_cols": ncols},
            "cpu_baseline": {"value": v, "unit": "coord updates/s", "cores": 1, "kind": "oracle",
                             "sample": sample},
            "e2e": {"value": v, "unit": "coord updates/s", "h2d_bytes_per_step": 0,
                    "d2h_bytes_per_step": 0}}
    print(json.dumps(line), flush=True)


# ------------------------------------------------------------------ product arm
def run_duhl(args, cfg, rank, world, local):
    import torch
    import paper_1708_05357_b200 as D
    torch.cuda.set_device(local)
    numa = numa_bind(local) if world > 1 else None   # the shard is first-touched on the GPU's node
    seed = 170805357 + 3
    d, n = cfg["d"], cfg["n"]
    # CoCoA-style sharding of the columns across ranks (one block per rank)
    lo, hi = rank * n // world, (rank + 1) * n // world
    t_gen = time.perf_counter()
    A, lab = make_data(cfg, seed, lo, hi, world)
    lam = lam_of(cfg, A, lab, world)
    t_gen = time.perf_counter() - t_gen
    t_pin = time.perf_counter()
    pinned = pin_host(A)   # the caller's data lives in pinned host memory (the e2e precondition)
    t_pin = time.perf_counter() - t_pin
    common = launch_kwargs(args, cfg, rank, world, local)
    budget, m = common["hbm_budget_bytes"], common["m"]
    uid = None
    if world > 1:  # NCCL group for the dv allreduce: id from rank 0, broadcast by torch.distributed
        import torch.distributed as dist
        obj = [D.comm_unique_id() if rank == 0 else None]
        dist.broadcast_object_list(obj, src=0)
        uid = obj[0]
    policy = {"gap": D.SEL_GAP, "sequential": D.SEL_SEQUENTIAL, "uniform": D.SEL_UNIFORM,
              "importance": D.SEL_IMPORTANCE}[args.policy]

    # ---------------- device-timed steady-state rounds
    t_create = time.perf_counter()
    P = create(D, A, lab, lam, cfg["model"], profile=True, cert_every=1 << 40, scd_exact=args.exact,
                 **common)
    if uid is not None:
        P.comm_init(uid, world, rank)
    t_create = time.perf_counter() - t_create
    scd_name, scd_W, scd_G, scd_R = P.scd_shape()
    stream = torch.cuda.ExternalStream(P.stream())
    for t in range(args.warmup):
        P.round(t, passes=args.passes, policy=policy)
    barrier(world)
    torch.cuda.synchronize()
    c0 = P.counters()
    k0 = {k: P.kernel_stats(k) for k in range(7)}
    ev0, ev1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    swaps = refreshed = 0
    with ClockSampler(local) as clk:
        ev0.record(stream)
        for t in range(args.warmup, args.warmup + args.steps):
            r = P.round(t, passes=args.passes, policy=policy)
            swaps += r.swaps
            refreshed += r.refreshed
        ev1.record(stream)
        ev1.synchronize()
    torch.cuda.synchronize()
    barrier(world)
    elapsed = max_over_ranks(ev0.elapsed_time(ev1) / 1e3, world)
    c1 = P.counters()
    pcie_peak = pcie_h2d_peak(local)
    pcie_bytes = (c1["h2d_bytes"] - c0["h2d_bytes"] + c1["zc_bytes"] - c0["zc_bytes"]) / args.steps
    pcie_step = None if budget == 0 else {"bytes_per_step": pcie_bytes,
            "copy_bytes_per_step": (c1["h2d_bytes"] - c0["h2d_bytes"]) / args.steps,
            "zero_copy_bytes_per_step": (c1["zc_bytes"] - c0["zc_bytes"]) / args.steps,
            "achieved_GBps": pcie_bytes / (elapsed / args.steps) / 1e9,
            "peak_GBps": pcie_peak, "frac": pcie_bytes / (elapsed / args.steps) / 1e9 / pcie_peak}
    k1 = {k: P.kernel_stats(k) for k in range(7)}
    # kernel-only SCD roofline: extra passes over the working set now resident in HBM
    # (no staging waits inside the launch), outside the timed region
    P.scd_epoch(passes=3, seed=12345, round=10 ** 6)
    k2 = P.kernel_stats(0)
    ko_ms = (k2[1] - k1[0][1]) / max(1, k2[0] - k1[0][0])
    ko_bytes = (k2[2] - k1[0][2]) / max(1, k2[0] - k1[0][0])
    hua = P.unit_a_host()
    P.close()
    updates = args.steps * m * args.passes * world
    value = updates / elapsed
    ms = {k: k1[k][1] - k0[k][1] for k in range(7)}
    nl = {k: k1[k][0] - k0[k][0] for k in range(7)}
    by = {k: k1[k][2] - k0[k][2] for k in range(7)}
    peak, peak_src = hbm_peak()
    scd_gbs = by[0] / (ms[0] / 1e3) / 1e9 if ms[0] > 0 else None
    gap_gbs = by[1] / (ms[1] / 1e3) / 1e9 if ms[1] > 0 else None
    # the HBM roofline kernel: the SCD epoch launches that wait for nothing (kind 0: passes >= 1,
    # and pass 0 of rounds without staging); pass-0 launches that consume staged columns as they
    # land (kind 5) are bound by the staging and reported under "pcie"
    dom = 0 if ms[0] >= ms[1] else 1
    dom_gbs = scd_gbs if dom == 0 else gap_gbs
    traffic = None
    tpath = os.path.join(ROOT, "profiles", "traffic.json")
    if os.path.exists(tpath):
        try:
            traffic = json.load(open(tpath)).get(args.config, {}).get(["scd", "gap"][dom])
        except Exception:
            traffic = None
    roofline = {"bound": "hbm", "kernel": [scd_name, "k_gap_tile"][dom],
                "achieved": dom_gbs, "peak": peak, "unit": "GB/s",
                "frac": (dom_gbs / peak) if dom_gbs else None, "traffic": traffic,
                "peak_source": peak_src,
                "share_of_step": (ms[dom] / 1e3) / elapsed,
                "algorithmic_bytes_per_launch": by[dom] / max(1, nl[dom]),
                "avg_launch_ms": ms[dom] / max(1, nl[dom]),
                "launches": nl[dom],
                "note": ("SCD launches that wait for no staged column (passes >= 1; pass 0 overlapping the "
                         "staging is under pcie.scd_overlapped)" if dom == 0 else "gap pass")}
    pcie = None
    if pcie_step is not None:
        stage_gbs = by[3] / (ms[3] / 1e3) / 1e9 if ms[3] > 0 else None
        pcie = dict(pcie_step,
                    staging={"kernel": "k_stage_gather (light rounds) / copy engine (heavy rounds)",
                             "achieved_GBps": stage_gbs, "peak_GBps": pcie_peak,
                             "frac": stage_gbs / pcie_peak if stage_gbs else None,
                             "ms_per_step": ms[3] / args.steps},
                    scd_overlapped={"kernel": scd_name, "launches": nl[5],
                                    "avg_launch_ms": ms[5] / max(1, nl[5]),
                                    "share_of_step": (ms[5] / 1e3) / elapsed},
                    note="the step's binding resource when the working set changes: staging (gather kernel "
                         "zero-copy reads / copy-engine copies) + unit-A zero-copy refresh reads over PCIe; peak "
                         "= 1 GiB pinned H2D copy measured in this run; pass 0 of the epoch consumes the staged "
                         "columns as they land (scd_overlapped)")

    # ---------------- end to end: create from host buffers + solve to certified eps
    e2e = None
    if not args.no_e2e:
        runs = []  # fresh create + solve each: time-to-eps is the median of --e2e-runs
        for rep in range(max(1, args.e2e_runs)):
            torch.cuda.synchronize()
            t0 = time.perf_counter()
            P2 = create(D, A, lab, lam, cfg["model"], cert_every=args.cert_every, scd_exact=args.exact,
                        **common)
            if uid is not None:
                P2.comm_init(uid, world, rank)
            t_c2 = time.perf_counter() - t0
            t1 = time.perf_counter()
            r = P2.solve(args.eps, args.max_rounds, passes=args.passes, policy=policy)
            t_solve = time.perf_counter() - t1
            wall = time.perf_counter() - t0
            c2 = P2.counters()
            state_err = state_check(P2, A, lab, cfg) if rep == 0 else None
            P2.close()
            c2["updates"] = int(max_over_ranks(c2["updates"], world)) * world
            runs.append(dict(r=r, c=c2, t_create=t_c2, t_solve=max_over_ranks(t_solve, world),
                             wall=max_over_ranks(wall, world), state_err=state_err))
        # the median run by create + solve wall time (value, bytes, create_s); time_to_eps_s is the
        # median duhl_solve time on its own (the two medians may come from different runs)
        order = sorted(range(len(runs)), key=lambda q: runs[q]["wall"])
        med = runs[order[len(runs) // 2]]
        r, c2, wall = med["r"], med["c"], med["wall"]
        t_solve_med = sorted(q["t_solve"] for q in runs)[len(runs) // 2]
        rounds = max(1, r["rounds"])
        e2e = {"value": c2["updates"] / wall, "unit": "coord updates/s",
               "h2d_bytes_per_step": int(c2["h2d_bytes"] / rounds),
               "zero_copy_bytes_per_step": int(c2["zc_bytes"] / rounds),
               "d2h_bytes_per_step": int(c2["d2h_bytes"] / rounds),
               "time_to_eps_s": t_solve_med, "time_to_eps_runs_s": [q["t_solve"] for q in runs],
               "create_plus_solve_runs_s": [q["wall"] for q in runs],
               "eps": args.eps, "certified_gap": r["gap"], "create_plus_solve_s": wall,
               "converged": all(q["r"]["status"] == 0 for q in runs), "rounds": r["rounds"],
               "rho_mean": rho_mean(r["trace"]),
               "swaps_per_round_first_last": swaps_trend(r["trace"]),
               "create_s": med["t_create"],
               "state_check": runs[0]["state_err"],
               "note": "median (by create + solve wall) of --e2e-runs fresh (create, solve) pairs; value = updates / (duhl_create "
                       "from the caller's pinned host buffers (used in place; one device pass over A for "
                       "norms + z at alpha=0, which also leaves columns 0..S-1 in the S HBM slots) + "
                       "duhl_solve to the certified gap); time_to_eps_s = the median duhl_solve alone (the rest of the "
                       "cold HBM fill included); h2d = fill + swaps (copy engine and staging gather); "
                       "zero-copy = create's pass + refresh + certificate reads of non-resident columns; "
                       "d2h = the library's read-backs (counted)"}

    # ---------------- baselines: same library, budget and kernels, batch selection
    # sequential blocks [Yu 2012] / uniform / importance sampling instead of gap top-m
    baselines = None
    if not args.no_baselines and not cfg.get("sparse") and budget > 0:
        baselines = {}
        caps = {"uniform": args.baseline_rounds, "sequential": args.seq_rounds,
                "importance": args.baseline_rounds}
        for pol_name in (("sequential", "uniform", "importance") if args.baselines else ("uniform", "sequential")):
            pol = {"sequential": D.SEL_SEQUENTIAL, "uniform": D.SEL_UNIFORM, "importance": D.SEL_IMPORTANCE}[pol_name]
            t0 = time.perf_counter()
            cb = dict(common, refresh_fraction=0.0)  # batch baselines do not read z
            P3 = create(D, A, lab, lam, cfg["model"], cert_every=args.cert_every, scd_exact=args.exact,
                          **cb)
            if uid is not None:
                P3.comm_init(uid, world, rank)
            rounds_cap = caps[pol_name]
            t1 = time.perf_counter()
            r = P3.solve(args.eps, rounds_cap, passes=args.passes, policy=pol)
            wall = max_over_ranks(time.perf_counter() - t1, world)
            c3 = P3.counters()
            g3, _, _ = P3.duality_gap()
            P3.close()
            baselines[pol_name] = {"time_s": wall, "rounds": r["rounds"], "converged": r["status"] == 0,
                                   "certified_gap": g3, "h2d_GB": c3["h2d_bytes"] / 1e9,
                                   "rho_mean": rho_mean(r["trace"]), "rounds_cap": rounds_cap,
                                   "time_to_eps_s": wall if r["status"] == 0 else None}
        baselines["note"] = ("same library, kernels, HBM budget and passes; selection by sequential blocks "
                             "[Yu 2012] (P:401) / uniform (P:434) instead of the gap memory; no unit-A refresh; "
                             "time_s = duhl_solve wall (data in pinned host memory), capped at rounds_cap rounds")

    # ---------------- the oracle's plain SCD to eps (the paper's single-threaded CPU baseline,
    # P:406): full at small configs, wall-capped at the large ones with the gap it reached, the
    # GPU's time to that same certified gap, and an extrapolated oracle time to eps
    oracle_tte = None
    if not args.no_cpu and not args.no_oracle_tte and rank == 0 and world == 1:
        oracle_tte = oracle_time_to_eps(cfg, A, lab, lam, args.eps, args.oracle_cap)
        if oracle_tte and not oracle_tte["converged"] and oracle_tte["gap_reached"] is not None:
            P4 = create(D, A, lab, lam, cfg["model"], cert_every=args.cert_every, scd_exact=args.exact, **common)
            t1 = time.perf_counter()
            r4 = P4.solve(oracle_tte["gap_reached"], args.max_rounds, passes=args.passes, policy=policy)
            oracle_tte["gpu_time_to_same_gap_s"] = time.perf_counter() - t1
            oracle_tte["gpu_rounds_to_same_gap"] = r4["rounds"]
            P4.close()

    # ---------------- CPU oracle on a bounded sample of the same workload
    cpu = None
    if not args.no_cpu and rank == 0:
        u, g, s = oracle_sample(cfg, A, lab, lam, min(args.ref_cols, hi - lo))
        cpu = {"value": u, "unit": "coord updates/s", "cores": 1, "kind": "oracle",
               "sample": f"1 sequential SCD pass over {min(args.ref_cols, hi - lo)} columns of the "
                         f"same {args.config.upper()} data, single-threaded C oracle ({s:.1f} s); "
                         f"oracle gap pass {g:.2f} GB/s",
               "gap_pass_GBps": g}

    line = {"metric": METRIC, "value": value, "unit": "coord updates/s", "n_gpus": world,
            "steps": args.steps, "warmup": args.warmup, "ms_per_step": 1e3 * elapsed / args.steps,
            "higher_is_better": True, "scaling": "strong", "vs_baseline": None,
            "dtype": "f64" if args.exact else "f32",
            "data": "synthetic",
            "config": {"workload": cfg["label"], "d": d, "n": n, "m": m, "passes": args.passes,
                       "arithmetic": ("fp32 data; SCD Gram products fp64 (scd_exact)" if args.exact else
                                      "fp32 data; SCD Gram tiles fp32 (FFMA2 / 3xTF32 mma) within a warp, "
                                      "fp64 across warps; dots, v, alpha, gaps and certificates fp64"),
                       "scd_exact": bool(args.exact), "numa_node": numa,
                       "policy": args.policy, "refresh_fraction": args.refresh,
                       "hbm_budget_GB": budget / 1e9, "lambda": lam,
                       "scd_kernel": {"name": scd_name, "W": scd_W, "G": scd_G, "R": scd_R},
                       "l2": ("inputs larger than L2 (CSC matrix resident in HBM >> 126 MB L2)"
                              if cfg.get("sparse") else
                              "inputs larger than L2 (working set 8 GB >> 126 MB L2)" if budget
                              else "working set may be L2-resident (small config)"),
                       "parallelism": f"cocoa{world}",
                       "unit_a_host": ({"threads": args.unit_a_host,
                                        "share": hua[1], "cols_total": hua[0]}
                                       if args.unit_a_host > 0 else None)},
            "roofline": roofline,
            "pcie": pcie,
            "roofline_scd_kernel_only": {"bound": "hbm", "kernel": scd_name, "unit": "GB/s",
                                         "achieved": ko_bytes / (ko_ms / 1e3) / 1e9,
                                         "peak": peak, "frac": ko_bytes / (ko_ms / 1e3) / 1e9 / peak,
                                         "avg_launch_ms": ko_ms,
                                         "note": "3 passes over the HBM-resident working set after the "
                                                 "timed rounds (no staging waits in the launch)"},
            "gap_pass_GBps": gap_gbs, "scd_GBps": scd_gbs,
            "kernel_ms": {"scd": ms[0], "scd_overlapped_staging": ms[5], "tpa_resync": ms[6], "gap_zP": ms[1], "topm": ms[2],
                          "stage_h2d": ms[3],
                          "refresh_unitA": ms[4]},
            "refresh_GBps": (by[4] / (ms[4] / 1e3) / 1e9) if ms[4] > 0 else None,
            "swaps_per_step": swaps / args.steps, "refreshed_per_step": refreshed / args.steps,
            "cpu_baseline": cpu, "e2e": e2e, "batch_baselines": baselines,
            "oracle_time_to_eps": oracle_tte,
            "gpu_launches": c1["launches"] - c0["launches"],
            "clocks": clk.summary(),
            "setup_s": {"generate": t_gen, "pin_host": t_pin, "pinned_bytes": pinned, "create": t_create}}
    if rank == 0:
        print(json.dumps(line), flush=True)


def launch_kwargs(args, cfg, rank=0, world=1, local=0):
    """duhl_create options of the bench's launch (also used by tests/test_gpu_fullsize.py so the
    full-size parity runs the timed configuration).  Strong scaling: the aggregate budget and
    working set stay those of the config; rank k owns columns [k n/N, (k+1) n/N)."""
    d, n = cfg["d"], cfg["n"]
    col_bytes = ((d + 3) // 4) * 16
    budget = int(cfg["budget_frac"] * n * col_bytes) // world if cfg["budget_frac"] > 0 else 0
    return dict(hbm_budget_bytes=budget, m=cfg["m"] // world, device=local, refresh_fraction=args.refresh,
                seed=170805357 + 3, borrow_host=True, n_global=n, col_offset=rank * n // world,
                linesearch=world > 1 or args.linesearch, unit_a_ctas=args.unit_a_ctas,
                unit_a_host_threads=args.unit_a_host, unit_a_host_share=args.host_share,
                scd_async=bool(cfg.get("scd_async")) and not args.exact, scd_block=cfg.get("scd_block", 0))


def parse_args(argv=None):
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=20)
    ap.add_argument("--warmup", type=int, default=30)
    ap.add_argument("--impl", default="duhl", choices=["duhl", "reference"])
    ap.add_argument("--config", default="c4", choices=sorted(CONFIGS))
    ap.add_argument("--passes", type=int, default=0, help="SCD passes per round (0: the config's)")
    ap.add_argument("--refresh", type=float, default=0.10)
    ap.add_argument("--policy", default="gap", choices=["gap", "sequential", "uniform", "importance"])
    ap.add_argument("--eps", type=float, default=1e-5)
    ap.add_argument("--max-rounds", type=int, default=2000)
    ap.add_argument("--cert-every", type=int, default=1 << 30,
                    help="scheduled certificates every R rounds (default: adaptive ones only)")
    ap.add_argument("--ref-cols", type=int, default=2000)
    ap.add_argument("--no-e2e", action="store_true")
    ap.add_argument("--e2e-runs", type=int, default=3, help="fresh create + solve runs; the median is reported")
    ap.add_argument("--exact", action="store_true", help="fp64 Gram products in the SCD kernel")
    ap.add_argument("--linesearch", action="store_true", help="gamma line search also at N=1")
    ap.add_argument("--baselines", action="store_true",
                    help="also time the importance-sampling baseline (uniform and sequential run by default)")
    ap.add_argument("--baseline-rounds", type=int, default=200,
                    help="round cap of the uniform / importance baselines")
    ap.add_argument("--seq-rounds", type=int, default=40, help="round cap of the sequential baseline")
    ap.add_argument("--no-baselines", action="store_true", help="skip the default uniform / sequential baselines")
    ap.add_argument("--no-oracle-tte", action="store_true", help="skip the oracle time-to-eps run")
    ap.add_argument("--oracle-cap", type=float, default=60.0,
                    help="wall cap (s) of the oracle's plain SCD run to eps (rank 0, N = 1)")
    ap.add_argument("--no-cpu", action="store_true")
    ap.add_argument("--unit-a-ctas", type=int, default=0,
                    help="CTAs of the unit-A refresh beside the epoch (0 auto, -1 off)")
    ap.add_argument("--unit-a-host", type=int, default=-1,
                    help="host threads that take part of the unit-A refresh (the paper's CPU unit A, P:332); "
                         "0 off (GPU-only refresh); -1 auto: min(14, cores - 2) on the out-of-core dense configs")
    ap.add_argument("--host-share", type=float, default=-1.0,
                    help="their share of the refresh's non-resident columns (<0: balanced per round)")
    args = ap.parse_args(argv)
    args.warmup = max(args.warmup, 0)
    cfg = CONFIGS[args.config]
    if args.unit_a_host < 0:  # out-of-core dense configs only: the refresh reads host columns there
        # the host's cores are shared by the ranks of this node (one process per GPU)
        cores = (os.cpu_count() or 1) // max(1, int(os.environ.get("LOCAL_WORLD_SIZE", "1")))
        args.unit_a_host = (min(14, cores - 2) if cfg["budget_frac"] > 0 and not cfg.get("sparse")
                            and cores >= 4 else 0)
    if args.passes <= 0:
        args.passes = cfg.get("passes_host", cfg.get("passes", 1)) if args.unit_a_host > 0 else cfg.get("passes", 1)
    return args, cfg


def main():
    args, cfg = parse_args()
    if args.impl == "reference":  # the CPU oracle: rank 0 alone, no process group needed
        run_reference(args, cfg, int(os.environ.get("RANK", "0")), int(os.environ.get("WORLD_SIZE", "1")))
        return
    rank, world, local = dist_init(args.gpus)
    run_duhl(args, cfg, rank, world, local)


if __name__ == "__main__":
    main()
