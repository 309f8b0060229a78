"""Race evidence without compute-sanitizer (closed on this GPU pool, see profiles/sanitizer_r02.txt):
the engine's synchronisation-heavy paths -- dependency-counter scheduling of the small-separator
IDs, the cluster CPQR's st.async/mbarrier row exchange with back-pressure tokens, the look-ahead
streams of the big-cell elimination, the host pre-plan thread, the concurrent-caller lock -- must
give BITWISE identical factors and solutions across repeated runs and across schedule
perturbations that do not change the arithmetic (look-ahead on/off, pre-plan on/off). A data race
shows up as run-to-run differences."""
import json
import os
import subprocess
import sys

import numpy as np
import pytest

from conftest import gpu_available

pytestmark = [pytest.mark.gpu,
              pytest.mark.skipif(not gpu_available(), reason="needs a CUDA device")]

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))

_RUN = r"""
import hashlib, json, sys
sys.path.insert(0, sys.argv[1])
import numpy as np
from paper_1808_01364_b200 import factorization as gfac
from paper_1808_01364_b200.grid import baseline_problem
cfg, n, eps, reps = sys.argv[2], int(sys.argv[3]), float(sys.argv[4]), int(sys.argv[5])
spec, A, _ = baseline_problem(cfg, 0, n)
B = np.random.default_rng(5).standard_normal((A.n, 3))
out = []
for _ in range(reps):
    F = gfac.factorize(A, spec, eps, "phif")
    X = gfac.apply_inverse(F, B)
    sets = [[sorted(int(v) for v in r) for _, r in F.skeleton_sets(l)] for l in range(spec.levels)]
    out.append({"x": hashlib.sha256(X.tobytes()).hexdigest(), "sets": hashlib.sha256(json.dumps(sets).encode()).hexdigest(),
                "SL": F.SL})
print(json.dumps(out))
"""


def _run(cfg, n, eps, reps, **env):
    e = dict(os.environ, **env)
    res = subprocess.run([sys.executable, "-c", _RUN, ROOT, cfg, str(n), str(eps), str(reps)], env=e,
                         capture_output=True, text=True, timeout=900)
    assert res.returncode == 0, res.stderr[-2000:]
    return json.loads(res.stdout.strip().splitlines()[-1])


@pytest.mark.parametrize("cfg,n,eps", [("c5", 64, 1e-2), ("c4", 32, 1e-3), ("c3p", 256, 1e-4), ("c1", 128, 1e-6)])
def test_repeated_runs_are_bitwise_identical(cfg, n, eps):
    runs = _run(cfg, n, eps, 3)
    assert all(r == runs[0] for r in runs), runs


def test_schedule_perturbations_do_not_change_bits():
    base = _run("c5", 64, 1e-2, 1)[0]
    assert _run("c5", 64, 1e-2, 1, PHIF_NO_LOOKAHEAD="1")[0] == base
    assert _run("c5", 64, 1e-2, 1, PHIF_NO_PREPLAN="1")[0] == base
    assert _run("c5", 64, 1e-2, 1, PHIF_HOST_PLAN="1")[0] == base
