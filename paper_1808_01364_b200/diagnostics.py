"""Error estimators (drop-in for the absent `hifsolve.diagnostics`).

* power_norm(op, dim, rel_tol=1e-2, maxit=200, seed)  generic host-callback power iteration
  (SPEC.md:400-404): unit start vector from default_rng(seed).standard_normal(dim),
  estimate |x^T op(x)| (Rayleigh quotient), converged when two successive Rayleigh
  quotients agree to rel_tol.
* estimate_solve_error(A, Fz)   e_s = ||I - G^-1 A G^-T||, run
  entirely on the device: G^-T, SpMV, G^-1 per iteration through the C-ABI, with the
  same start vector and stopping rule as power_norm.
"""

from __future__ import annotations

import ctypes as C
from dataclasses import dataclass

import numpy as np

from . import _lib
from .errors import EstimationError
from .factorization import Factorization, apply_inverse, device_matrix


@dataclass
class NormEstimate:
    value: float
    iterations: int
    converged: bool
    rel_tol_achieved: float


def power_norm(op, dim, rel_tol=1e-2, maxit=200, seed=0) -> NormEstimate:
    x = np.random.default_rng(seed).standard_normal(dim)
    x /= np.linalg.norm(x)
    prev, est = None, 0.0
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
    rel = (abs(est - prev) / est if est > 0.0 else abs(est - prev)) if prev is not None else float("inf")
    return NormEstimate(est, maxit, False, rel)


def estimate_solve_error(A, Fz: Factorization, rel_tol=1e-2, maxit=200, seed=(0, 13)) -> NormEstimate:
    dm = device_matrix(A)
    x0 = np.ascontiguousarray(np.random.default_rng(list(seed)).standard_normal(dm.N))
    val = C.c_double()
    its = C.c_int()
    conv = C.c_int()
    rel = C.c_double()
    err = _lib.phif_error()
    rc = _lib.lib().phif_solve_error(dm.handle, Fz.handle, _lib.ptr(x0), float(rel_tol), int(maxit),
                                     C.byref(val), C.byref(its), C.byref(conv), C.byref(rel), C.byref(err))
    _lib.raise_for(rc, err)
    return NormEstimate(val.value, its.value, bool(conv.value), rel.value)


def estimate_apply_error(A, Fz: Factorization, rel_tol=1e-2, maxit=200, seed=(0, 12)) -> NormEstimate:
    """e_a = ||A - F|| / ||A||: two device power iterations from one start vector."""
    dm = device_matrix(A)
    x0 = np.ascontiguousarray(np.random.default_rng(list(seed)).standard_normal(dm.N))
    val = C.c_double()
    its = C.c_int()
    conv = C.c_int()
    rel = C.c_double()
    err = _lib.phif_error()
    rc = _lib.lib().phif_apply_error(dm.handle, Fz.handle, _lib.ptr(x0), float(rel_tol), int(maxit),
                                     C.byref(val), C.byref(its), C.byref(conv), C.byref(rel), C.byref(err))
    _lib.raise_for(rc, err)
    return NormEstimate(val.value, its.value, bool(conv.value), rel.value)


def estimate_inverse_error(A, Fz: Factorization, rel_tol=1e-2, maxit=200, seed=(0, 14)) -> NormEstimate:
    """||I - A F^-1|| through host callbacks (non-symmetric form; diagnostic only)."""
    csr = getattr(A, "csr", A)
    return power_norm(lambda x: x - csr @ apply_inverse(Fz, x), csr.shape[0], rel_tol, maxit, list(seed))


def require_converged(est: NormEstimate, what="estimator"):
    if not est.converged:
        raise EstimationError(f"{what} did not converge", partial=est.value)
    return est
