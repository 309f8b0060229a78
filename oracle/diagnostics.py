"""Error estimators and dense oracle (restates the absent `diagnostics`).

TEST INFRASTRUCTURE ONLY (see oracle/__init__.py).

power_norm: power iteration from a unit start vector drawn from
default_rng(seed).standard_normal(dim); each step y = op(x), estimate |x^T y|
(the Rayleigh quotient of the unit iterate), x <- y / ||y||; converged when two
successive Rayleigh quotients agree to rel_tol. e_s = power_norm(x -> x - G^-1 A G^-T x),
e_a = power_norm(x -> A x - F x) / power_norm(A).
"""

from __future__ import annotations

from dataclasses import dataclass

import numpy as np

from . import phif


@dataclass
class NormEstimate:
    value: float
    iterations: int
    converged: bool
    rel_tol_achieved: float


def power_norm(op, dim, rel_tol=1e-2, maxit=200, seed=0):
    x = np.random.default_rng(seed).standard_normal(dim)
    x /= np.linalg.norm(x)
    prev = None
    est = 0.0
    for it in range(1, maxit + 1):
        y = np.asarray(op(x), dtype=np.float64)
        est = abs(float(x @ y))              # Rayleigh quotient of the unit iterate
        ny = float(np.linalg.norm(y))
        if ny == 0.0:
            return NormEstimate(0.0, it, True, 0.0)
        if prev is not None:
            rel = abs(est - prev) / est if est > 0.0 else abs(est - prev)
            if rel <= rel_tol:
                return NormEstimate(est, it, True, rel)
        prev = est
        x = y / ny
    rel = (abs(est - prev) / est if est > 0.0 else abs(est - prev)) if prev is not None else np.inf
    return NormEstimate(est, maxit, False, rel)


def estimate_solve_error(A, F, rel_tol=1e-2, maxit=200, seed=(0, 13)):
    csr = getattr(A, "csr", A)
    op = lambda x: x - phif.apply_ginv(F, csr @ phif.apply_ginv_t(F, x))
    return power_norm(op, csr.shape[0], rel_tol, maxit, list(seed))


def estimate_apply_error(A, F, rel_tol=1e-2, maxit=200, seed=(0, 12)):
    csr = getattr(A, "csr", A)
    num = power_norm(lambda x: csr @ x - phif.apply(F, x), csr.shape[0], rel_tol, maxit, list(seed))
    den = power_norm(lambda x: csr @ x, csr.shape[0], rel_tol, maxit, list(seed))
    return NormEstimate(num.value / den.value, num.iterations + den.iterations,
                        num.converged and den.converged, max(num.rel_tol_achieved, den.rel_tol_achieved))


class DenseOracle:
    """Densified A for N <= 4096."""

    def __init__(self, A):
        csr = getattr(A, "csr", A)
        if csr.shape[0] > 4096:
            raise ValueError("dense oracle limited to N <= 4096")
        self.A = csr.toarray()
        self.L = np.linalg.cholesky(self.A)

    def solve(self, b):
        import scipy.linalg
        return scipy.linalg.cho_solve((self.L, True), b)

    def cond(self):
        w = np.linalg.eigvalsh(self.A)
        return float(w[-1] / w[0])

    def solve_error(self, F):
        """Exact ||I - G^-1 A G^-T||_2 by densifying G^-1 and G^-T."""
        N = self.A.shape[0]
        E = np.eye(N)
        GtI = phif.apply_ginv_t(F, E)
        S = phif.apply_ginv(F, self.A @ GtI)
        return float(np.linalg.norm(np.eye(N) - S, 2))
