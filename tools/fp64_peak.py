"""Measure FP64 peaks on the box: cuBLAS DGEMM (torch.matmul float64) and HBM copy.

Writes gpurun_out/fp64_peak.json. Used once per pool to fill the FP64 roofline
denominator that MEASURED_PEAKS.json does not carry.
"""
import json, os, subprocess, time
import torch

def bench(fn, iters=10):
    s = torch.cuda.Event(enable_timing=True); e = torch.cuda.Event(enable_timing=True)
    best = 1e30
    for _ in range(3): fn()
    torch.cuda.synchronize()
    for _ in range(iters):
        s.record(); fn(); e.record(); torch.cuda.synchronize()
        best = min(best, s.elapsed_time(e))
    return best

out = {"gpu": torch.cuda.get_device_name(0)}
for n in (4096, 8192):
    a = torch.randn(n, n, dtype=torch.float64, device="cuda")
    b = torch.randn(n, n, dtype=torch.float64, device="cuda")
    c = torch.empty_like(a)
    ms = bench(lambda: torch.matmul(a, b, out=c))
    out[f"dgemm_{n}_tflops"] = 2 * n**3 / ms / 1e9
# sustained DGEMM for 4 s
n = 8192
a = torch.randn(n, n, dtype=torch.float64, device="cuda"); b = torch.randn_like(a); c = torch.empty_like(a)
torch.cuda.synchronize(); t0 = time.time(); cnt = 0
s = torch.cuda.Event(enable_timing=True); e = torch.cuda.Event(enable_timing=True); s.record()
while time.time() - t0 < 4.0:
    torch.matmul(a, b, out=c); cnt += 1
    if cnt % 4 == 0: torch.cuda.synchronize()
e.record(); torch.cuda.synchronize()
out["dgemm_8192_sustained_tflops"] = 2 * n**3 * cnt / s.elapsed_time(e) / 1e9
x = torch.empty(1 << 28, dtype=torch.float64, device="cuda"); y = torch.empty_like(x)
ms = bench(lambda: y.copy_(x))
out["hbm_copy_gbs"] = 2 * x.numel() * 8 / ms / 1e6
print(json.dumps(out))
os.makedirs("gpurun_out", exist_ok=True)
json.dump(out, open("gpurun_out/fp64_peak.json", "w"), indent=1)
