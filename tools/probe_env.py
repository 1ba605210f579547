"""One-shot environment probe for the GPU box."""
import os, subprocess, time, json
import torch

out = {}
def sh(c):
    try:
        return subprocess.run(c, shell=True, capture_output=True, text=True, timeout=60).stdout
    except Exception as e:
        return str(e)
out["nproc"] = os.cpu_count()
out["lscpu"] = sh("lscpu | head -20")
out["free"] = sh("free -g")
out["smi"] = sh("nvidia-smi --query-gpu=name,pcie.link.gen.current,pcie.link.gen.max,pcie.link.width.current,memory.total,clocks.max.sm --format=csv")
out["topo"] = sh("nvidia-smi topo -m")
p = torch.cuda.get_device_properties(0)
out["props"] = {k: getattr(p, k) for k in dir(p) if not k.startswith("_") and isinstance(getattr(p, k), (int, float, str))}
def t(fn, it=10):
    fn(); torch.cuda.synchronize()
    s = torch.cuda.Event(enable_timing=True); e = torch.cuda.Event(enable_timing=True)
    best = 1e9
    for _ in range(it):
        s.record(); fn(); e.record(); e.synchronize(); best = min(best, s.elapsed_time(e) / 1e3)
    return best
N = 1 << 30
h = torch.empty(N, dtype=torch.uint8, pin_memory=True)
dv = torch.empty(N, dtype=torch.uint8, device="cuda")
out["h2d_GBps"] = N / t(lambda: dv.copy_(h, non_blocking=True)) / 1e9
out["d2h_GBps"] = N / t(lambda: h.copy_(dv, non_blocking=True)) / 1e9
x = torch.randn(1 << 30, device="cuda")
out["read_sum_GBps"] = 4 * x.numel() / t(lambda: x.sum()) / 1e9
y = torch.empty_like(x)
out["copy_GBps"] = 8 * x.numel() / t(lambda: y.copy_(x)) / 1e9
del x, y
res = {}
for (d, n) in [(200704, 10000), (40000, 50176), (500, 2000000)]:
    A = torch.randn(n, d, device="cuda")  # row i = column a_i (column-major A)
    w = torch.randn(d, device="cuda")
    tt = t(lambda: torch.mv(A, w))
    res[f"{d}x{n}"] = 4 * d * n / tt / 1e9
    del A
out["torch_mv_GBps"] = res
v = torch.zeros(200704, device="cuda")
idx = torch.randint(0, 200704, (1 << 27,), device="cuda")
src = torch.randn(1 << 27, device="cuda")
tt = t(lambda: v.index_add_(0, idx, src))
out["index_add_f32_Gops"] = (1 << 27) / tt / 1e9
v64 = torch.zeros(200704, device="cuda", dtype=torch.float64)
src64 = src.double()
tt = t(lambda: v64.index_add_(0, idx, src64))
out["index_add_f64_Gops"] = (1 << 27) / tt / 1e9
print(json.dumps(out, indent=1, default=str))
os.makedirs("gpurun_out", exist_ok=True)
json.dump(out, open("gpurun_out/probe_env.json", "w"), indent=1, default=str)
