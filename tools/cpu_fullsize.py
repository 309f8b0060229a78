"""Full-size CPU-oracle factorization timing on this host (the GPU box host for the committed
profile): python tools/cpu_fullsize.py c5 [out.json]. Same seeded problem as bench.py's
workload; numpy/scipy OpenBLAS with all host threads (cores recorded)."""
import json
import os
import sys
import time

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

from bench import WORKLOADS  # noqa: E402
from oracle import phif as ophif  # noqa: E402
from paper_1808_01364_b200.grid import CONFIGS, baseline_problem  # noqa: E402
sys.path.insert(0, os.path.join(ROOT, "tests", "golden"))
from make_fullsize import cpu_model, csr_sha  # noqa: E402

wl = sys.argv[1] if len(sys.argv) > 1 else "c5"
out = sys.argv[2] if len(sys.argv) > 2 else os.path.join(ROOT, "profiles", f"cpu_fullsize_{wl}_r02.json")
cfg_name, eps, n, _ = WORKLOADS[wl]
spec, A, _ = baseline_problem(cfg_name, 0, n)
t0 = time.perf_counter()
F = ophif.factorize(A, spec, eps, CONFIGS[cfg_name].method)
dt = time.perf_counter() - t0
rec = {"workload": wl, "config": cfg_name, "eps": eps, "N": int(A.n), "csr_sha256": csr_sha(A), "SL": int(F.SL),
       "t_factor_s": dt, "dofs_per_s": A.n / dt, "cores": os.cpu_count(), "cpu_model": cpu_model(),
       "blas_threads": os.environ.get("OPENBLAS_NUM_THREADS", "all"),
       "levels": F.stats["levels"], "kind": "port (oracle/, restating SPEC.md:229-453 on the reference's "
                                             "own kernels.py / hierarchy.py primitives)"}
json.dump(rec, open(out, "w"), indent=1)
print(json.dumps({k: rec[k] for k in ("N", "SL", "t_factor_s", "dofs_per_s", "cores", "cpu_model")}))
