"""Oracle factorization / PCG / estimators against SPEC.md's worked examples and invariants.

The reference ships no factorization, krylov or diagnostics module; these
examples and the acceptance invariants (SPEC.md:321-328,
519-527) are the pin of the oracle's composition.
"""
import numpy as np
import pytest
import scipy.sparse as sp

from oracle import diagnostics, krylov, phif
from oracle.errors import NotSpdError
from paper_1808_01364_b200.grid import CoefficientField, GridSpec, assemble_operator, generate_field

A3 = np.array([[4.0, 2.0, 0.0], [2.0, 3.0, 1.0], [0.0, 1.0, 2.0]])


def test_eliminate_cells_kat():
    st = phif.store_from_dense(A3, [[0], [1], [2]])
    recs = phif.eliminate_cells(st, [0])
    assert np.allclose(recs[0].L, [[2.0]])
    assert np.allclose(phif.store_to_dense(st, 3), [[1, 0, 0], [0, 2, 1], [0, 1, 2]])


def test_eliminate_uncoupled_and_commuting():
    D = np.diag([2.0, 3.0, 4.0])
    st = phif.store_from_dense(D, [[0], [1], [2]])
    phif.eliminate_cells(st, [0])
    assert np.allclose(phif.store_to_dense(st, 3), np.diag([1.0, 3.0, 4.0]))
    rng = np.random.default_rng(0)
    G = rng.standard_normal((5, 5))
    S = G @ G.T + 5 * np.eye(5)
    S[0, 1] = S[1, 0] = 0.0
    a = phif.store_from_dense(S, [[0], [1], [2, 3, 4]])
    b = phif.store_from_dense(S, [[0], [1], [2, 3, 4]])
    phif.eliminate_cells(a, [0, 1])
    phif.eliminate_cells(b, [1, 0])
    assert np.allclose(phif.store_to_dense(a, 5), phif.store_to_dense(b, 5), rtol=1e-13, atol=1e-13)


def test_precondition_kat():
    st = phif.store_from_dense(A3, [[0], [1], [2]])
    phif.precondition_blocks(st, [0])
    assert np.allclose(phif.store_to_dense(st, 3), [[1, 1, 0], [1, 3, 1], [0, 1, 2]])
    st = phif.store_from_dense(np.eye(3), [[0, 1], [2]])
    phif.precondition_blocks(st, [0, 1])
    assert np.allclose(phif.store_to_dense(st, 3), np.eye(3))


def test_skeletonize_edge_cases():
    # zero coupling to R: every DOF redundant (pure elimination)
    S = np.diag([2.0, 3.0, 5.0])
    st = phif.store_from_dense(S, [[0, 1], [2]])
    recs, ranks = phif.skeletonize_separators(st, [0], 1e-6)
    assert ranks == [0] and len(recs[0].redundant) == 2
    # full-rank coupling at eps=1e-15: nothing redundant, matrix unchanged
    rng = np.random.default_rng(2)
    G = rng.standard_normal((6, 6))
    S = G @ G.T + 6 * np.eye(6)
    st = phif.store_from_dense(S, [[0, 1, 2], [3, 4, 5]])
    recs, ranks = phif.skeletonize_separators(st, [0], 1e-15)
    assert recs == [] and ranks == [3]
    assert np.allclose(phif.store_to_dense(st, 6), S)


def _problem(dim, n, m, seed=1, contrast=1e4):
    spec = GridSpec(dim, n, m)
    return spec, assemble_operator(generate_field(spec, seed, contrast), 0.0)


@pytest.mark.parametrize("dim,n,m", [(2, 16, 4), (2, 32, 4), (3, 16, 4)])
def test_exact_mode_inverts(dim, n, m):
    spec, A = _problem(dim, n, m)
    F = phif.factorize(A, spec, 0.0, "exact")
    rng = np.random.default_rng(3)
    X = rng.standard_normal((A.n, 10))
    Y = phif.apply_inverse(F, A.csr @ X)
    assert np.linalg.norm(Y - X) <= 1e-10 * np.linalg.norm(X)
    Z = phif.apply(F, X)
    assert np.linalg.norm(Z - A.csr @ X) <= 1e-10 * np.linalg.norm(A.csr @ X)


def test_apply_inverse_symmetric_and_ginv_composition():
    spec, A = _problem(2, 32, 4)
    F = phif.factorize(A, spec, 1e-6, "phif")
    rng = np.random.default_rng(4)
    u, v = rng.standard_normal(A.n), rng.standard_normal(A.n)
    a, b = phif.apply_inverse(F, u) @ v, u @ phif.apply_inverse(F, v)
    assert abs(a - b) <= 1e-12 * abs(a)
    w = phif.apply_ginv_t(F, phif.apply_ginv(F, u))
    assert np.linalg.norm(w - phif.apply_inverse(F, u)) <= 1e-12 * np.linalg.norm(w)
    # linearity of apply
    assert np.allclose(phif.apply(F, u + v), phif.apply(F, u) + phif.apply(F, v), rtol=1e-12, atol=1e-12)


def test_pcg_spec_examples():
    b = np.random.default_rng(5).standard_normal(7)
    x, rep = krylov.pcg(sp.identity(7, format="csr"), b)
    assert rep.n_i == 1 and np.allclose(x, b)
    x, rep = krylov.pcg(sp.csr_matrix(A3), np.array([1.0, 0.0, 0.0]))
    assert np.allclose(x, [5 / 12, -1 / 3, 1 / 6], atol=1e-10)
    spec, A = _problem(2, 32, 4)
    F = phif.factorize(A, spec, 0.0, "exact")
    x, rep = krylov.pcg(A, np.ones(A.n), precond=F, tol=1e-12)
    assert rep.n_i <= 2 and rep.converged


def test_pcg_multi_rhs_equals_single():
    spec, A = _problem(2, 32, 4)
    F = phif.factorize(A, spec, 1e-3, "phif")
    B = np.random.default_rng(6).standard_normal((A.n, 3))
    X, rep = krylov.pcg(A, B, precond=F)
    for c in range(3):
        x, r1 = krylov.pcg(A, B[:, c], precond=F)
        assert r1.n_i == rep.n_i[c] and np.allclose(x, X[:, c], rtol=0, atol=1e-14 * np.abs(x).max())


def test_power_norm_examples():
    assert diagnostics.power_norm(lambda x: x, 10).value == pytest.approx(1.0)
    est = diagnostics.power_norm(lambda x: np.array([3.0, 1.0, 0.5]) * x, 3, rel_tol=1e-4)
    assert est.value == pytest.approx(3.0, rel=1e-2)


def test_solve_error_dense_crosscheck_and_phif_beats_hif():
    spec, A = _problem(2, 16, 4, contrast=1e4)
    F = phif.factorize(A, spec, 1e-2, "phif")
    exact = diagnostics.DenseOracle(A).solve_error(F)
    est = diagnostics.estimate_solve_error(A, F, rel_tol=1e-3)
    assert est.value == pytest.approx(exact, rel=0.1)
    spec, A = _problem(2, 64, 8, seed=2, contrast=1e4)
    es_p = diagnostics.estimate_solve_error(A, phif.factorize(A, spec, 1e-6, "phif")).value
    es_h = diagnostics.estimate_solve_error(A, phif.factorize(A, spec, 1e-6, "hif")).value
    assert es_p < es_h


def test_exact_mode_solve_error_tiny():
    spec, A = _problem(2, 32, 4)
    F = phif.factorize(A, spec, 0.0, "exact")
    assert diagnostics.estimate_solve_error(A, F).value <= 1e-9


def test_not_spd_reported_with_location():
    spec = GridSpec(2, 16, 4)
    f = CoefficientField(spec, np.ones(spec.shape), 0, 1.0, 1.0)
    A = assemble_operator(f)
    csr = A.csr.tolil()
    bad = spec.id_of([[6, 2]])[0]         # interior DOF of level-0 cell (1, 0)
    csr[bad, bad] = -1.0
    with pytest.raises(NotSpdError) as e:
        phif.factorize(sp.csr_matrix(csr), spec, 1e-6, "phif")
    assert e.value.level == 0 and e.value.stage == "eliminate" and e.value.group == 4
