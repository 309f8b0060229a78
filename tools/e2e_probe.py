"""Where does the end-to-end (host CSR -> factor) time go? python tools/e2e_probe.py [cfg]"""
import sys, time
sys.path.insert(0, ".")
import torch
from paper_1808_01364_b200.grid import CONFIGS, baseline_problem
from paper_1808_01364_b200 import factorization as gf
name = sys.argv[1] if len(sys.argv) > 1 else "c5"
spec, A, _ = baseline_problem(name, 0, None)
eps = CONFIGS[name].eps[0] if hasattr(CONFIGS[name], "eps") else 1e-2
F = gf.factorize(A, spec, 1e-2, CONFIGS[name].method); F = None
for rep in range(3):
    torch.cuda.synchronize()
    t0 = time.perf_counter(); A._device = None; dm = gf.device_matrix(A); torch.cuda.synchronize(); t1 = time.perf_counter()
    F = gf.factorize(dm, spec, 1e-2, CONFIGS[name].method); _ = F.stats["SL"]; torch.cuda.synchronize(); t2 = time.perf_counter()
    F = None; torch.cuda.synchronize(); t3 = time.perf_counter()
    print(f"create {1e3*(t1-t0):.1f} ms  factorize {1e3*(t2-t1):.1f} ms  free {1e3*(t3-t2):.1f} ms", flush=True)
