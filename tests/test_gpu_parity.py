"""GPU parity: the B200 path (through the C-ABI) vs the CPU oracle on identical seeded inputs.

North-star criteria (BASELINE.json): identical skeleton sets (pivot gaps > 1e-12),
e_s within 2x, PCG iteration counts within +-1, solution relative difference <= 1e-8,
NotSpd reported at the same (level, stage, group, pivot).
"""
import numpy as np
import pytest
import scipy.sparse as sp

from conftest import gpu_available

pytestmark = [pytest.mark.gpu,
              pytest.mark.skipif(not gpu_available(), reason="needs a CUDA device")]

from oracle import diagnostics as odiag  # noqa: E402
from oracle import krylov as okry  # noqa: E402
from oracle import phif as ophif  # noqa: E402
from oracle.errors import NotSpdError as OracleNotSpd  # noqa: E402
from paper_1808_01364_b200 import NotSpdError  # noqa: E402
from paper_1808_01364_b200 import diagnostics as gdiag  # noqa: E402
from paper_1808_01364_b200 import factorization as gfac  # noqa: E402
from paper_1808_01364_b200 import krylov as gkry  # noqa: E402
from paper_1808_01364_b200.grid import (CONFIGS, CoefficientField, GridSpec, assemble_operator,  # noqa: E402
                                        baseline_problem, baseline_rhs, generate_field)

X_TOL = 1e-8          # final solution relative difference
APPLY_TOL = 1e-8      # F^-1 b relative difference


def _small(dim, n, m, seed=1, contrast=1e4):
    spec = GridSpec(dim, n, m)
    return spec, assemble_operator(generate_field(spec, seed, contrast), 0.0)


CASES = [
    ("exact-2d", lambda: _small(2, 16, 4), "exact", 0.0, 1e-12),
    ("phif-2d", lambda: _small(2, 32, 4), "phif", 1e-6, 1e-12),
    ("hif-2d", lambda: _small(2, 32, 8), "hif", 1e-6, 1e-12),
    ("exact-3d", lambda: _small(3, 16, 4), "exact", 0.0, 1e-12),
    ("phif-3d", lambda: _small(3, 16, 4), "phif", 1e-3, 1e-12),
    ("c1", lambda: baseline_problem("c1", 0)[:2], "phif", 1e-6, 1e-12),
    ("c2-n128-phif", lambda: baseline_problem("c2", 0, 128)[:2], "phif", 1e-3, 1e-12),
    ("c2-n128-hif", lambda: baseline_problem("c2", 0, 128)[:2], "hif", 1e-3, 1e-12),
    ("c3-n128-1e-4", lambda: baseline_problem("c3", 0, 128)[:2], "phif", 1e-4, 1e-12),
    ("c4-n32", lambda: baseline_problem("c4", 0, 32)[:2], "phif", 1e-3, 1e-12),
    ("c5-n32", lambda: baseline_problem("c5", 0, 32)[:2], "phif", 1e-2, 1e-10),
    # full-size 3D config: large separators (team CPQR) and big cells (tile-parallel path)
    ("c4-full", lambda: baseline_problem("c4", 0)[:2], "phif", 1e-3, 1e-12),
    ("c5-n64", lambda: baseline_problem("c5", 0, 64)[:2], "phif", 1e-2, 1e-10),
]


def _redundant_sets(Fo, lev):
    return {tuple(int(v) for v in np.sort(r.redundant)) for r in Fo.levels[lev].skeletonize}


@pytest.mark.parametrize("name,make,method,eps,tol", CASES, ids=[c[0] for c in CASES])
def test_parity_with_oracle(name, make, method, eps, tol):
    spec, A = make()
    try:
        Fo = ophif.factorize(A, spec, eps, method)
    except OracleNotSpd as e:
        with pytest.raises(NotSpdError) as g:
            gfac.factorize(A, spec, eps, method)
        assert (g.value.level, g.value.stage, g.value.group, g.value.pivot) == (e.level, e.stage, e.group, e.pivot)
        return
    Fg = gfac.factorize(A, spec, eps, method)
    assert Fg.SL == Fo.SL
    for lev in range(spec.levels):
        got = {tuple(int(v) for v in np.sort(r)) for _, r in Fg.skeleton_sets(lev) if len(r)}
        assert got == _redundant_sets(Fo, lev), f"skeleton sets differ at level {lev}"
    B = np.random.default_rng(7).standard_normal((A.n, 4))
    yo, yg = ophif.apply_inverse(Fo, B), gfac.apply_inverse(Fg, B)
    assert np.linalg.norm(yg - yo) <= APPLY_TOL * np.linalg.norm(yo)
    b = np.random.default_rng([0, 1]).standard_normal(A.n)
    xo, ro = okry.pcg(A, b, precond=Fo, tol=tol)
    xg, rg = gkry.pcg(A, b, precond=Fg, tol=tol)
    assert abs(rg.n_i - ro.n_i) <= 1
    assert np.linalg.norm(xg - xo) <= X_TOL * np.linalg.norm(xo)
    eo = odiag.estimate_solve_error(A, Fo).value
    eg = gdiag.estimate_solve_error(A, Fg).value
    assert eg <= 2 * eo + 1e-14 and eo <= 2 * eg + 1e-14


def test_c3_loose_tolerance_not_spd_parity():
    """c3's contrast-1e8 field at eps = 1e-2 loses positive definiteness (PAPER.md Remark 2)."""
    spec, A = baseline_problem("c3", 1, 256)[:2]
    with pytest.raises(OracleNotSpd) as e:
        ophif.factorize(A, spec, 1e-2, "phif")
    with pytest.raises(NotSpdError) as g:
        gfac.factorize(A, spec, 1e-2, "phif")
    assert (g.value.level, g.value.stage, g.value.group, g.value.pivot) == (e.value.level, e.value.stage,
                                                                            e.value.group, e.value.pivot)


def test_not_spd_input_location():
    spec = GridSpec(2, 16, 4)
    A = assemble_operator(CoefficientField(spec, np.ones(spec.shape), 0, 1.0, 1.0)).csr.tolil()
    A[spec.id_of([[6, 2]])[0], spec.id_of([[6, 2]])[0]] = -1.0
    with pytest.raises(NotSpdError) as g:
        gfac.factorize(sp.csr_matrix(A), spec, 1e-6, "phif")
    assert (g.value.level, g.value.stage, g.value.group) == (0, "eliminate", 4)


@pytest.mark.parametrize("dim,n", [(2, 32), (3, 16)])
def test_exact_mode_acceptance(dim, n):
    """SPEC.md AC1: exact mode, ||I - A F^-1|| <= 1e-9 (e_s form), 5 seeds."""
    for seed in range(5):
        spec = GridSpec(dim, n, 4)
        A = assemble_operator(generate_field(spec, seed))
        F = gfac.factorize(A, spec, 0.0, "exact")
        assert gdiag.estimate_solve_error(A, F).value <= 1e-9


def test_pcg_spec_examples_on_gpu():
    b = np.random.default_rng(5).standard_normal(7)
    x, rep = gkry.pcg(sp.identity(7, format="csr"), b)
    assert rep.n_i == 1 and np.allclose(x, b)
    A3 = sp.csr_matrix(np.array([[4.0, 2.0, 0.0], [2.0, 3.0, 1.0], [0.0, 1.0, 2.0]]))
    x, rep = gkry.pcg(A3, np.array([1.0, 0.0, 0.0]))
    assert np.allclose(x, [5 / 12, -1 / 3, 1 / 6], atol=1e-10)


def test_multi_rhs_block_equals_single_solves():
    spec, A = baseline_problem("c1", 0)[:2]
    F = gfac.factorize(A, spec, 1e-6, "phif")
    B = baseline_rhs("c1", A.n, 0, 8)
    X, rep = gkry.pcg(A, B, precond=F)
    for c in (0, 5):
        x, r1 = gkry.pcg(A, B[:, c], precond=F)
        assert r1.n_i == rep.n_i[c]
        assert np.linalg.norm(x - X[:, c]) <= 1e-12 * np.linalg.norm(x)


@pytest.mark.parametrize("nrhs", [32, 33, 48])
def test_wide_rhs_block_apply_matches_oracle(nrhs):
    # 32 right-hand sides: lane-per-RHS replay kernels; more than 32: the generic batched GEMM
    spec, A = baseline_problem("c4", 0, 32)[:2]
    Fo = ophif.factorize(A, spec, 1e-3, "phif")
    Fg = gfac.factorize(A, spec, 1e-3, "phif")
    B = np.random.default_rng(11).standard_normal((A.n, nrhs))
    yo, yg = ophif.apply_inverse(Fo, B), gfac.apply_inverse(Fg, B)
    assert np.linalg.norm(yg - yo) <= APPLY_TOL * np.linalg.norm(yo)


@pytest.mark.parametrize("cfg,n,eps", [("c4", 32, 1e-3), ("c1", None, 1e-6), ("c5", 32, 1e-2)])
def test_32_rhs_up_and_down_passes_match_oracle(cfg, n, eps):
    # 32 right-hand sides take the warp-level DMMA replay kernels (cells, block-Jacobi groups,
    # separators) and the pipelined replay GEMM: G^-1 and G^-T separately, and their composition
    spec, A = baseline_problem(cfg, 0, n)[:2]
    Fo = ophif.factorize(A, spec, eps, "phif")
    Fg = gfac.factorize(A, spec, eps, "phif")
    B = np.random.default_rng(23).standard_normal((A.n, 32))
    uo, ug = ophif.apply_ginv(Fo, B), gfac.apply_ginv(Fg, B)
    assert np.linalg.norm(ug - uo) <= APPLY_TOL * np.linalg.norm(uo)
    do, dg = ophif.apply_ginv_t(Fo, B), gfac.apply_ginv_t(Fg, B)
    assert np.linalg.norm(dg - do) <= APPLY_TOL * np.linalg.norm(do)
    yg = gfac.apply_ginv_t(Fg, ug)
    assert np.linalg.norm(yg - gfac.apply_inverse(Fg, B)) <= 1e-12 * np.linalg.norm(yg)
    # single right-hand sides through the lane-per-RHS kernels agree with the block
    y1 = gfac.apply_inverse(Fg, B[:, 7])
    assert np.linalg.norm(y1 - yg[:, 7]) <= 1e-11 * np.linalg.norm(y1)


def test_apply_inverse_symmetry_and_ginv_on_gpu():
    spec, A = baseline_problem("c4", 0, 32)[:2]
    F = gfac.factorize(A, spec, 1e-3, "phif")
    rng = np.random.default_rng(8)
    u, v = rng.standard_normal(A.n), rng.standard_normal(A.n)
    a, b = gfac.apply_inverse(F, u) @ v, u @ gfac.apply_inverse(F, v)
    assert abs(a - b) <= 1e-12 * abs(a)
    w = gfac.apply_ginv_t(F, gfac.apply_ginv(F, u))
    assert np.linalg.norm(w - gfac.apply_inverse(F, u)) <= 1e-12 * np.linalg.norm(w)


# ---- apply (F x), e_a, root_condition --------------------------------
FWD_CASES = [c for c in CASES if c[0] in ("exact-2d", "phif-2d", "hif-2d", "exact-3d", "phif-3d", "c4-n32")]


@pytest.mark.parametrize("name,make,method,eps,tol", FWD_CASES, ids=[c[0] for c in FWD_CASES])
def test_apply_forward_parity(name, make, method, eps, tol):
    """F x = G G^T x on the GPU vs the oracle's record replay (oracle/phif.py apply, _g, _gt)."""
    spec, A = make()
    Fo = ophif.factorize(A, spec, eps, method)
    Fg = gfac.factorize(A, spec, eps, method)
    rng = np.random.default_rng(7)
    X = rng.standard_normal((spec.ndofs, 3))
    ref = ophif.apply(Fo, X)
    got = gfac.apply(Fg, X)
    assert np.linalg.norm(got - ref) <= 1e-10 * np.linalg.norm(ref)
    gt = ophif._gt(Fo, X.copy())
    assert np.linalg.norm(gfac.apply_g_t(Fg, X) - gt) <= 1e-10 * np.linalg.norm(gt)
    g = ophif._g(Fo, X.copy())
    assert np.linalg.norm(gfac.apply_g(Fg, X) - g) <= 1e-10 * np.linalg.norm(g)
    # inverse pair and linearity
    x = X[:, 0]
    back = gfac.apply_inverse(Fg, gfac.apply(Fg, x))
    assert np.linalg.norm(back - x) <= 1e-9 * np.linalg.norm(x)
    y = X[:, 1]
    lin = gfac.apply(Fg, x + y) - gfac.apply(Fg, x) - gfac.apply(Fg, y)
    assert np.linalg.norm(lin) <= 1e-12 * np.linalg.norm(gfac.apply(Fg, x + y)) * 10
    if method == "exact":   # ||F x - A x|| / ||A x|| <= 1e-10
        Ax = A.csr @ x
        assert np.linalg.norm(gfac.apply(Fg, x) - Ax) <= 1e-10 * np.linalg.norm(Ax)


@pytest.mark.parametrize("name,make,method,eps,tol",
                         [c for c in FWD_CASES if c[0] in ("exact-2d", "phif-2d", "hif-2d", "phif-3d")],
                         ids=["exact-2d", "phif-2d", "hif-2d", "phif-3d"])
def test_apply_error_and_root_condition(name, make, method, eps, tol):
    """e_a = ||A - F|| / ||A|| and kappa(A_L) vs the oracle."""
    spec, A = make()
    Fo = ophif.factorize(A, spec, eps, method)
    Fg = gfac.factorize(A, spec, eps, method)
    ea_o = odiag.estimate_apply_error(A, Fo)
    ea_g = gdiag.estimate_apply_error(A, Fg)
    assert ea_g.converged
    if method == "exact":
        assert ea_g.value <= 1e-9
    else:
        assert ea_o.value / 2 <= ea_g.value <= 2 * ea_o.value
    ko = ophif.root_condition(Fo)
    kg = gfac.root_condition(Fg)
    assert abs(kg - ko) <= 1e-8 * ko


_GID_DUMP = r"""
import json, sys
sys.path.insert(0, sys.argv[1])
from paper_1808_01364_b200 import factorization as gfac
from paper_1808_01364_b200.grid import baseline_problem
spec, A, _ = baseline_problem("c5", 0, 64)
F = gfac.factorize(A, spec, 1e-2, "phif")
print(json.dumps({"SL": F.SL, "n_gid": sum(lv.get("n_gid", 0) for lv in F.stats["levels"]),
                  "red": [[sorted(int(v) for v in r) for _, r in F.skeleton_sets(l)] for l in range(spec.levels)]}))
"""


@pytest.mark.parametrize("clusters", ["16", "8"])
def test_gram_id_forced_cluster_matches_oracle(clusters):
    """Gram-path ID with a forced cluster size (mixed-k waves, C=16 leaves CTAs with no
    active columns while their peers run on): skeleton sets still equal the oracle's at c5 n=64."""
    import json
    import os
    import subprocess
    import sys
    root = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
    env = dict(os.environ, PHIF_GID_C=clusters)
    res = subprocess.run([sys.executable, "-c", _GID_DUMP, root], env=env, capture_output=True, text=True,
                         timeout=600)
    assert res.returncode == 0, res.stderr[-2000:]
    got = json.loads(res.stdout.strip().splitlines()[-1])
    assert got["n_gid"] > 0
    spec, A = baseline_problem("c5", 0, 64)[:2]
    Fo = ophif.factorize(A, spec, 1e-2, "phif")
    assert got["SL"] == Fo.SL
    for lev in range(spec.levels):
        g = {tuple(r) for r in got["red"][lev] if r}
        assert g == _redundant_sets(Fo, lev), f"level {lev}"


def test_pcg_residual_history_and_partial_stats():
    """SolveReport.history: one relative residual per iteration, matching the
    oracle's history to the PCG tolerance scale; NotSpdError.partial_stats (errors.py:21-30) holds
    the statistics of the levels completed before the failure."""
    spec, A = baseline_problem("c4", 0, 32)[:2]
    Fo = ophif.factorize(A, spec, 1e-3, "phif")
    Fg = gfac.factorize(A, spec, 1e-3, "phif")
    b = np.random.default_rng([0, 1]).standard_normal(A.n)
    xo, ro = okry.pcg(A, b, precond=Fo, tol=1e-12)
    xg, rg = gkry.pcg(A, b, precond=Fg, tol=1e-12)
    assert len(rg.history) == rg.n_i and rg.history[-1] == pytest.approx(rg.relres)
    m = min(len(rg.history), len(ro.history))
    ho = np.array([float(h[0]) for h in ro.history[:m]])
    assert np.allclose(np.array(rg.history[:m]), ho, rtol=1e-6, atol=1e-13)
    B = np.random.default_rng([0, 2]).standard_normal((A.n, 3))
    Xg, rb = gkry.pcg(A, B, precond=Fg, tol=1e-12)
    assert len(rb.history) == int(np.max(rb.n_i)) and rb.history[-1].shape == (3,)
    spec2, A2 = baseline_problem("c3", 1, 256)[:2]
    with pytest.raises(NotSpdError) as g:
        gfac.factorize(A2, spec2, 1e-2, "phif")
    ps = g.value.partial_stats
    assert ps is not None and len(ps["levels"]) == g.value.level and ps["complete"] is False


def test_concurrent_apply_on_one_factor():
    """a completed Factorization is safe for concurrent callers (the C-ABI serialises
    per factor; ctypes releases the GIL, so the threads really overlap on the host)."""
    import threading
    spec, A = baseline_problem("c4", 0, 32)[:2]
    F = gfac.factorize(A, spec, 1e-3, "phif")
    rhs = [np.random.default_rng([9, i]).standard_normal((A.n, 1 + i % 3)) for i in range(8)]
    ref = [gfac.apply_inverse(F, b) for b in rhs]
    out = [None] * len(rhs)

    def work(i):
        for _ in range(3):
            out[i] = gfac.apply_inverse(F, rhs[i])

    th = [threading.Thread(target=work, args=(i,)) for i in range(len(rhs))]
    for t in th:
        t.start()
    for t in th:
        t.join()
    for r, o in zip(ref, out):
        assert np.array_equal(r, o)
