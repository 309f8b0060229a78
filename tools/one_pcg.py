"""Factorize once, then one block PCG solve (for profiling the apply)."""
import sys, time
import numpy as np
sys.path.insert(0, ".")
from paper_1808_01364_b200.grid import CONFIGS, baseline_problem, baseline_rhs
from paper_1808_01364_b200 import factorization as gf, krylov as gk
name, eps = sys.argv[1], float(sys.argv[2])
n = int(sys.argv[3]) if len(sys.argv) > 3 and sys.argv[3] != "-" else None
spec, A, _ = baseline_problem(name, 0, n)
F = gf.factorize(A, spec, eps, CONFIGS[name].method)
B = baseline_rhs(name, A.n, 0)
t = time.time(); X, rep = gk.pcg(A, B, precond=F, tol=CONFIGS[name].tol); print("pcg %.1f ms n_i %s" % ((time.time() - t) * 1e3, rep.n_i))
