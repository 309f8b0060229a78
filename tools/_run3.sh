timeout 600 python -m pytest tests/test_gpu_parity.py -x -q -k "history or spec_examples or parity_with_oracle" > gpurun_out/r2c_pytest.txt 2>&1
tail -3 gpurun_out/r2c_pytest.txt
python tools/one_factor.py c5 1e-2 - 3 -v > gpurun_out/r2c_onefactor.txt 2>&1
PHIF_PLAN_TIMING=1 python tools/one_factor.py c5 1e-2 - 2 > gpurun_out/r2c_plantiming.txt 2>&1
python - > gpurun_out/r2c_pcg.txt 2>&1 <<'PY'
import sys, time
sys.path.insert(0, ".")
import numpy as np
from paper_1808_01364_b200.grid import CONFIGS, baseline_problem, baseline_rhs
from paper_1808_01364_b200 import factorization as gf, krylov as gk
spec, A, _ = baseline_problem("c5", 0, None)
F = gf.factorize(A, spec, 1e-2, "phif")
B = baseline_rhs(CONFIGS["c5"], A.n, 0)
for rep in range(3):
    t = time.perf_counter(); X, r = gk.pcg(A, B, precond=F, tol=1e-10); dt = time.perf_counter() - t
    print("pcg e2e %.1f ms  %.2f ms/RHS  n_i %s" % (dt * 1e3, dt * 1e3 / 32, list(r.n_i)), flush=True)
PY
