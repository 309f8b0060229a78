"""One timed factorization (for profiling): python tools/one_factor.py <cfg> <eps> [n] [reps]"""
import sys, time
sys.path.insert(0, ".")
from paper_1808_01364_b200.grid import CONFIGS, baseline_problem
from paper_1808_01364_b200 import factorization as gf
name, eps = sys.argv[1], float(sys.argv[2])
n = int(sys.argv[3]) if len(sys.argv) > 3 and sys.argv[3] != "-" else None
reps = int(sys.argv[4]) if len(sys.argv) > 4 else 1
spec, A, _ = baseline_problem(name, 0, n)
F = None
for _ in range(reps):
    F = None
    t = time.time(); F = gf.factorize(A, spec, eps, CONFIGS[name].method); print("factorize %.1f ms SL %d" % ((time.time() - t) * 1e3, F.SL), flush=True)
