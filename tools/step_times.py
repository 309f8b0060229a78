"""Per-step factorization wall times through the bench's path (device matrix), timing on/off."""
import sys, time
sys.path.insert(0, ".")
import torch
from paper_1808_01364_b200.grid import CONFIGS, baseline_problem
from paper_1808_01364_b200 import factorization as gf
name = sys.argv[1] if len(sys.argv) > 1 else "c5"
cfg = CONFIGS[name]
spec, A, _ = baseline_problem(name, 0, None)
stream = torch.cuda.current_stream().cuda_stream
dm = gf.device_matrix(A, stream)
for timing in (True, False, True, False):
    ts = []
    for _ in range(3):
        torch.cuda.synchronize()
        t = time.perf_counter()
        F = None
        F = gf.factorize(dm, spec, cfg.eps[0], cfg.method, stream=stream, timing=timing)
        torch.cuda.synchronize()
        ts.append((time.perf_counter() - t) * 1e3)
    print("timing", timing, ["%.1f" % x for x in ts], "plan", round(F.stats["t_plan_ms"], 1))
