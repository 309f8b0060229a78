"""Small factorize + apply + PCG runs for compute-sanitizer (racecheck / synccheck / memcheck):
c1 at n=64 (one-CTA cells, dependency-driven small-separator IDs, warp block-Jacobi) and the c5
recipe at n=32 (Gram-path cluster IDs with the st.async/mbarrier row exchange, tile-parallel big
cells with the look-ahead streams, batched GEMMs, the device planner).
    compute-sanitizer --tool racecheck python tools/sanitize.py"""
import sys

sys.path.insert(0, ".")
import numpy as np  # noqa: E402

from paper_1808_01364_b200 import factorization as gf  # noqa: E402
from paper_1808_01364_b200 import krylov as gk  # noqa: E402
from paper_1808_01364_b200.grid import baseline_problem  # noqa: E402

for cfg, eps, n in (("c1", 1e-6, 64), ("c5", 1e-2, 32)):
    spec, A, _ = baseline_problem(cfg, 0, n)
    F = gf.factorize(A, spec, eps, "phif")
    b = np.random.default_rng(1).standard_normal((A.n, 2))
    x, rep = gk.pcg(A, b, precond=F, tol=1e-10)
    print(cfg, n, "SL", F.SL, "n_i", list(rep.n_i), flush=True)
