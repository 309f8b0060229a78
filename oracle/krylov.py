"""Preconditioned CG oracle (restates the absent `krylov.pcg`).

TEST INFRASTRUCTURE ONLY (see oracle/__init__.py).

Standard PCG per right-hand side column: x0 = 0, stop when ||r||/||b|| <= tol
(recursive residual, replaced by the true residual b - A x every 50 iterations,
SPEC.md:377), maxit 500, BreakdownError on a non-finite recurrence value
(SPEC.md:364). A column that has converged is frozen while the others go on,
so every column's (x, n_i) equals a single-RHS run. Call shape follows
grid.py:288-292: pcg(A, b, tol=..., maxit=...) -> (x, report).
"""

from __future__ import annotations

from dataclasses import dataclass, field

import numpy as np

from .errors import BreakdownError

REFRESH = 50


@dataclass
class SolveReport:
    n_i: object                 # int for one RHS, array for a block
    relres: object
    converged: object
    history: list = field(default_factory=list)
    wall_time: float = 0.0


def pcg(A, b, precond=None, tol=1e-12, maxit=500, apply_inverse=None):
    import time
    t0 = time.perf_counter()
    csr = getattr(A, "csr", A)
    B = np.asarray(b, dtype=np.float64)
    flat = B.ndim == 1
    B = B.reshape(B.shape[0], -1)
    N, k = B.shape
    if precond is None:
        M = lambda r: r.copy()
    else:
        if apply_inverse is None:
            from .phif import apply_inverse as _ai
            apply_inverse = _ai
        M = lambda r: apply_inverse(precond, r)
    X = np.zeros_like(B)
    bn = np.linalg.norm(B, axis=0)
    iters = np.zeros(k, dtype=np.int64)
    done = bn == 0.0
    relres = np.where(done, 0.0, 1.0)
    R = B.copy()
    Z = M(R)
    P = Z.copy()
    rz = np.einsum("ij,ij->j", R, Z)
    hist = []
    it = 0
    while not done.all() and it < maxit:
        it += 1
        act = ~done
        Q = csr @ P
        pq = np.einsum("ij,ij->j", P, Q)
        with np.errstate(divide="ignore", invalid="ignore"):
            alpha = np.where(act, rz / pq, 0.0)
        if not np.all(np.isfinite(alpha)):
            raise BreakdownError(f"non-finite alpha at iteration {it}")
        X += P * alpha
        if it % REFRESH == 0:
            R = np.where(act, B - csr @ X, R)
        else:
            R -= Q * alpha
        rn = np.linalg.norm(R, axis=0)
        with np.errstate(divide="ignore", invalid="ignore"):
            rr = np.where(act, rn / np.where(bn == 0, 1, bn), relres)
        if not np.all(np.isfinite(rr)):
            raise BreakdownError(f"non-finite residual at iteration {it}")
        relres = rr
        iters[act] = it
        hist.append(relres.copy())
        newly = act & (relres <= tol)
        done |= newly
        if done.all():
            break
        Z = M(R)
        rz_new = np.einsum("ij,ij->j", R, Z)
        with np.errstate(divide="ignore", invalid="ignore"):
            beta = np.where(~done, rz_new / rz, 0.0)
        if not np.all(np.isfinite(beta)):
            raise BreakdownError(f"non-finite beta at iteration {it}")
        P = np.where(~done, Z + P * beta, P)
        rz = np.where(~done, rz_new, rz)
    conv = relres <= tol
    rep = SolveReport(int(iters[0]) if flat else iters, float(relres[0]) if flat else relres,
                      bool(conv[0]) if flat else conv, hist, time.perf_counter() - t0)
    return (X[:, 0] if flat else X), rep
