"""Where does the host-array solve go? python tools/solve_probe.py"""
import sys, time
sys.path.insert(0, ".")
import ctypes as C
import numpy as np
import torch
from paper_1808_01364_b200.grid import CONFIGS, baseline_problem, baseline_rhs
from paper_1808_01364_b200 import factorization as gf, krylov, _lib
name = sys.argv[1] if len(sys.argv) > 1 else "c5"
cfg = CONFIGS[name]
spec, A, _ = baseline_problem(name, 0, None)
F = gf.factorize(A, spec, cfg.eps[0] if isinstance(cfg.eps, (list, tuple)) else 1e-2, cfg.method)
B = baseline_rhs(cfg, spec.ndofs, 0)
L = _lib.lib()
for rep in range(3):
    t0 = time.perf_counter()
    X, r = krylov.pcg(A, B, precond=F, tol=cfg.tol)
    t1 = time.perf_counter()
    print(f"host pcg: {1e3*(t1-t0):.1f} ms ({1e3*(t1-t0)/B.shape[1]:.2f} ms/RHS) n_i max {int(np.max(r.n_i))}", flush=True)
Bd = torch.from_numpy(B).cuda(); Xd = torch.zeros_like(Bd)
it = np.zeros(B.shape[1], dtype=np.int32); rr = np.zeros(B.shape[1]); cv = np.zeros(B.shape[1], dtype=np.int32)
err = _lib.phif_error()
dm = gf.device_matrix(A, None)
for rep in range(3):
    torch.cuda.synchronize(); t0 = time.perf_counter()
    rc = L.phif_pcg(dm.handle, F.handle, C.c_void_p(Bd.data_ptr()), C.c_void_p(Xd.data_ptr()), B.shape[1], cfg.tol, 500,
                    None, _lib.ptr(it), _lib.ptr(rr), _lib.ptr(cv), None, None, C.byref(err))
    torch.cuda.synchronize(); t1 = time.perf_counter()
    print(f"device pcg: {1e3*(t1-t0):.1f} ms ({1e3*(t1-t0)/B.shape[1]:.2f} ms/RHS) rc={rc}", flush=True)
# pieces
X = np.zeros_like(B)
for rep in range(2):
    t0 = time.perf_counter(); X2 = np.zeros_like(B); t1 = time.perf_counter(); X2[:] = 1.0; t2 = time.perf_counter()
    print(f"np.zeros_like {1e3*(t1-t0):.1f} ms, first touch fill {1e3*(t2-t1):.1f} ms", flush=True)
    for mode in (0,):
        Y = B.copy()
        t0 = time.perf_counter(); rc = L.phif_apply(F.handle, _lib.ptr(Y), B.shape[1], 0, C.byref(err)); t1 = time.perf_counter()
        print(f"host apply (upload+apply+download): {1e3*(t1-t0):.1f} ms", flush=True)
