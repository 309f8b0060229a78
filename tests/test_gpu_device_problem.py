"""On-device generation + assembly + matrix-free SpMV against the host
reference recipe (grid.py:182-260 as restated in paper_1808_01364_b200/grid.py, itself pinned bit for
bit to the reference's assemble_operator by tests/test_grid.py)."""
import numpy as np
import pytest

from conftest import gpu_available

pytestmark = [pytest.mark.gpu,
              pytest.mark.skipif(not gpu_available(), reason="needs a CUDA device")]

from paper_1808_01364_b200 import factorization as gfac  # noqa: E402
from paper_1808_01364_b200 import krylov as gkry  # noqa: E402
from paper_1808_01364_b200.device_problem import device_baseline_problem  # noqa: E402
from paper_1808_01364_b200.grid import CONFIGS, baseline_problem, baseline_rhs  # noqa: E402

CASES = [("c5", 32), ("c5", None), ("c3p", 256), ("c3", 128), ("c2", 128), ("c4", 32), ("c1", None)]


@pytest.mark.parametrize("cfg,n", CASES, ids=[f"{c}-{n or 'full'}" for c, n in CASES])
def test_device_assembly_is_bit_identical(cfg, n):
    spec, A, field = baseline_problem(cfg, 0, n)
    dspec, M = device_baseline_problem(cfg, 0, n)
    rp, ci, va, fd = M.csr()
    assert np.array_equal(fd, np.asarray(field.values).ravel(order="F"))
    assert np.array_equal(rp, A.csr.indptr.astype(np.int64))
    assert np.array_equal(ci, A.csr.indices.astype(np.int32))
    assert np.array_equal(va, A.csr.data)
    X = np.random.default_rng(3).standard_normal((A.n, 3))
    y_mf = M.matvec(X)
    y_csr = M.matvec(X, force_csr=True)
    assert np.array_equal(y_mf, y_csr)
    assert np.allclose(y_mf, A.csr @ X, rtol=1e-13, atol=1e-13 * np.abs(A.csr.data).max())


def test_factorize_and_solve_from_device_problem():
    cfg = CONFIGS["c5"]
    spec, A, _ = baseline_problem("c5", 0, 64)
    _, M = device_baseline_problem("c5", 0, 64)
    Fh = gfac.factorize(A, spec, 1e-2, "phif")
    Fd = gfac.factorize(M, spec, 1e-2, "phif")
    for lev in range(spec.levels):
        a = [tuple(r) for _, r in Fh.skeleton_sets(lev)]
        b = [tuple(r) for _, r in Fd.skeleton_sets(lev)]
        assert a == b
    B = baseline_rhs(cfg, A.n, 0, 4)
    Xh, rh = gkry.pcg(A, B, precond=Fh, tol=cfg.tol)
    Xd, rd = gkry.pcg(M, B, precond=Fd, tol=cfg.tol)
    assert np.array_equal(rh.n_i, rd.n_i)
    assert np.array_equal(Xh, Xd)   # matrix-free SpMV: same terms, same order, same FMAs
