"""Preconditioned CG on the GPU (drop-in for the absent `hifsolve.krylov`).

pcg(A, b, precond=None, tol=1e-12, maxit=500) -> (x, SolveReport), the call shape of
grid.py:288-292. Standard PCG per right-hand-side column with F^-1 from the B200
factorization, stop on ||r||/||b|| <= tol, true residual every 50 iterations,
BreakdownError on a non-finite recurrence value, maxit flagged in the report with
the partial x returned. Converged columns are frozen so a block of right-hand
sides behaves like independent single-RHS solves. SolveReport.history holds the
relative residual after every iteration (a float per iteration for
one right-hand side, an array per iteration for a block).
"""

from __future__ import annotations

import ctypes as C
import time
from dataclasses import dataclass, field

import numpy as np

from . import _lib
from .factorization import Factorization, device_matrix


@dataclass
class SolveReport:
    n_i: object
    relres: object
    converged: object
    history: list = field(default_factory=list)
    wall_time: float = 0.0

    @property
    def maxit_hit(self):
        return not bool(np.all(self.converged))


def pcg(A, b, precond: Factorization | None = None, tol: float = 1e-12, maxit: int = 500, stream=None):
    t0 = time.perf_counter()
    dm = device_matrix(A, stream)
    B = np.asarray(b, dtype=np.float64)
    flat = B.ndim == 1
    B = np.ascontiguousarray(B.reshape(B.shape[0], -1))
    k = B.shape[1]
    X = np.empty_like(B)   # phif_pcg overwrites every entry
    iters = np.zeros(k, dtype=np.int32)
    relres = np.zeros(k, dtype=np.float64)
    conv = np.zeros(k, dtype=np.int32)
    hist = np.zeros((max(int(maxit), 1), k), dtype=np.float64)
    nh = C.c_int(0)
    err = _lib.phif_error()
    rc = _lib.lib().phif_pcg(dm.handle, precond.handle if precond is not None else None, _lib.ptr(B),
                             _lib.ptr(X), k, float(tol), int(maxit), C.c_void_p(stream or 0), _lib.ptr(iters),
                             _lib.ptr(relres), _lib.ptr(conv), _lib.ptr(hist), C.byref(nh), C.byref(err))
    _lib.raise_for(rc, err)
    history = [float(h[0]) if flat else h.copy() for h in hist[:nh.value]]
    rep = SolveReport(int(iters[0]) if flat else iters.astype(np.int64),
                      float(relres[0]) if flat else relres,
                      bool(conv[0]) if flat else conv.astype(bool), history, time.perf_counter() - t0)
    return (X[:, 0] if flat else X), rep
