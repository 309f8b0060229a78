"""Time F^-1 applies on a device-resident N x k block (c5): python tools/apply_probe.py [k] [reps]"""
import sys, time
sys.path.insert(0, ".")
import ctypes as C
import torch
from paper_1808_01364_b200.grid import CONFIGS, baseline_problem
from paper_1808_01364_b200 import factorization as gf, _lib
k = int(sys.argv[1]) if len(sys.argv) > 1 else 32
reps = int(sys.argv[2]) if len(sys.argv) > 2 else 5
spec, A, _ = baseline_problem("c5", 0, None)
F = gf.factorize(A, spec, 1e-2, "phif")
X = torch.randn(spec.ndofs, k, dtype=torch.float64, device="cuda")
L = _lib.lib()
err = _lib.phif_error()
prof = len(sys.argv) > 3
for it in range(reps):
    torch.cuda.synchronize(); t0 = time.perf_counter()
    if prof and it == reps - 1: torch.cuda.profiler.start()
    rc = L.phif_apply(F.handle, C.c_void_p(X.data_ptr()), k, 0, C.byref(err))
    if prof and it == reps - 1: torch.cuda.synchronize(); torch.cuda.profiler.stop()
    torch.cuda.synchronize(); t1 = time.perf_counter()
    print(f"apply F^-1 k={k}: {1e3*(t1-t0):.2f} ms rc={rc}", flush=True)
