"""One timed factorization (for profiling): python tools/one_factor.py <cfg> <eps> [n] [reps] [-v]"""
import json, sys, time
sys.path.insert(0, ".")
from paper_1808_01364_b200.grid import CONFIGS, baseline_problem
from paper_1808_01364_b200 import factorization as gf
name, eps = sys.argv[1], float(sys.argv[2])
n = int(sys.argv[3]) if len(sys.argv) > 3 and sys.argv[3] != "-" else None
reps = int(sys.argv[4]) if len(sys.argv) > 4 else 1
verbose = "-v" in sys.argv
spec, A, _ = baseline_problem(name, 0, n)
F = None
for _ in range(reps):
    F = None
    t = time.time(); F = gf.factorize(A, spec, eps, CONFIGS[name].method, timing=verbose); print("factorize %.1f ms SL %d" % ((time.time() - t) * 1e3, F.SL), flush=True)
if verbose:
    st = F.stats
    keys = ["level", "p", "q", "cell_n_max", "cell_b_max", "sep_k_max", "rho_max", "t_plan_ms", "t_wall_ms", "t_repack_ms",
            "t_eliminate_ms", "t_precondition_ms", "t_id_ms", "t_skel_update_ms"]
    print("t_plan_ms", st["t_plan_ms"])
    for lv in st["levels"]:
        print(" ".join(f"{k}={lv[k]:.1f}" if isinstance(lv[k], float) else f"{k}={lv[k]}" for k in keys),
              "GF:", [round(f / 1e9, 2) for f in lv["flops"]])
