"""Full-size GPU run of a BASELINE config: factorize (timed per stage), PCG, e_s."""
import json, sys, time
import numpy as np
sys.path.insert(0, ".")
from paper_1808_01364_b200.grid import CONFIGS, baseline_problem, baseline_rhs
from paper_1808_01364_b200 import factorization as gf, krylov as gk, diagnostics as gd

name = sys.argv[1]
eps = float(sys.argv[2]) if len(sys.argv) > 2 else CONFIGS[name].eps[-1]
n = int(sys.argv[3]) if len(sys.argv) > 3 and sys.argv[3] != "-" else None
seed = int(sys.argv[4]) if len(sys.argv) > 4 else 0
cfg = CONFIGS[name]
t = time.time(); spec, A, _ = baseline_problem(name, seed, n); print("problem %.1fs N=%d nnz=%d" % (time.time() - t, A.n, A.nnz), flush=True)
gf.device_matrix(A)
for rep in range(2):
    t = time.time(); F = gf.factorize(A, spec, eps, cfg.method, timing=True); tf = time.time() - t
    st = F.stats
    print(f"factorize wall {tf*1e3:.1f} ms  engine {st['t_factor_ms']:.1f} ms  plan {st['t_plan_ms']:.1f} ms  SL {st['SL']}  rec {st['mem_bytes']/1e9:.2f} GB", flush=True)
for lv in st["levels"]:
    print("  ", json.dumps(lv), flush=True)
B = baseline_rhs(cfg, A.n, seed)
t = time.time(); X, rep = gk.pcg(A, B, precond=F, tol=cfg.tol); ts = time.time() - t
print(f"pcg nrhs={B.shape[1]} n_i={rep.n_i} relres max={np.max(rep.relres):.2e} time {ts*1e3:.1f} ms ({ts*1e3/B.shape[1]:.2f} ms/RHS)", flush=True)
t = time.time(); es = gd.estimate_solve_error(A, F); print(f"e_s={es.value:.3e} it={es.iterations} conv={es.converged} t={time.time()-t:.2f}s", flush=True)
