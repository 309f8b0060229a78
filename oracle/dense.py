"""Dense primitives of the oracle (restates reference kernels.py:23-119).

TEST INFRASTRUCTURE ONLY (see oracle/__init__.py).

The arithmetic goes through the same LAPACK routines the reference calls
(scipy's dpotrf, dtrtrs, dgeqp3), so oracle results equal the reference's on
the same inputs. `cpqr_dlaqp2` is an independent numpy restatement of the
dgeqp3 -> dlaqp2 algorithm (initial dnrm2 column norms, idamax pivot with
lowest-index ties, dlarfg/dlarf Householder step, partial-norm downdate with
recomputation when the downdate ratio drops below sqrt(dlamch('E'))). It is
what the CUDA CPQR kernel implements; tests pin it against scipy's dgeqp3.
"""

from __future__ import annotations

from dataclasses import dataclass

import numpy as np
import scipy.linalg
from scipy.linalg import lapack

from .errors import NotSpdError

EPS = float(np.finfo(np.float64).eps)          # 2^-52, kernels.py:20
TOL3Z = float(np.sqrt(EPS / 2.0))              # sqrt(dlamch('E')), dlaqp2


def cholesky(S) -> np.ndarray:
    """Lower Cholesky of symmetric S (kernels.py:23-35).

    dpotrf(lower, clean); a failed pivot raises NotSpdError with the 0-based
    pivot index info-1 (kernels.py:32), an empty matrix gives a (0, 0) factor.
    """
    S = np.ascontiguousarray(S, dtype=np.float64)
    if S.ndim != 2 or S.shape[0] != S.shape[1]:
        raise ValueError(f"expected a square matrix, got shape {S.shape}")
    if S.shape[0] == 0:
        return np.zeros((0, 0))
    fac, info = lapack.dpotrf(S, lower=1, clean=1, overwrite_a=0)
    if info > 0:
        raise NotSpdError(pivot=info - 1)
    if info < 0:
        raise ValueError(f"dpotrf rejected argument {-info}")
    return fac


def tri_solve(L, B, trans: bool = False, side: str = "left") -> np.ndarray:
    """op(L) X = B (left) or X op(L) = B (right) for lower L (kernels.py:38-62).

    A zero on the diagonal raises NotSpdError at argmin |diag| (kernels.py:50-51).
    """
    L = np.asarray(L)
    B = np.asarray(B)
    if L.shape[0] != L.shape[1]:
        raise ValueError("triangular factor must be square")
    if L.shape[0] and np.any(np.diag(L) == 0.0):
        raise NotSpdError(pivot=int(np.argmin(np.abs(np.diag(L)))))
    if L.shape[0] == 0 or B.size == 0:
        return np.zeros_like(B, dtype=np.float64)
    if side == "left":
        return scipy.linalg.solve_triangular(L, B, lower=True, trans="T" if trans else "N")
    if side == "right":
        return scipy.linalg.solve_triangular(L, B.T, lower=True, trans="N" if trans else "T").T
    raise ValueError(f"side must be 'left' or 'right', got {side!r}")


@dataclass(frozen=True)
class IdResult:
    """Column ID: M[:, redundant] ~= M[:, skeleton] @ interp (kernels.py:65-81)."""

    skeleton: np.ndarray
    redundant: np.ndarray
    interp: np.ndarray

    @property
    def rank(self) -> int:
        return len(self.skeleton)


def _id_from_r(R, perm, nrows, ncols, eps):
    """Rank cut and interpolation matrix from a pivoted R (kernels.py:100-119)."""
    none = np.zeros(0, dtype=np.intp)
    d = np.abs(np.diag(R))
    cut = max(eps, EPS * max(nrows, ncols)) * d[0]
    rank = int(np.count_nonzero(d > cut))
    perm = np.asarray(perm, dtype=np.intp)
    if rank == len(perm):
        return IdResult(np.sort(perm), none, np.zeros((len(perm), 0)))
    sk, rd = perm[:rank], perm[rank:]
    T = scipy.linalg.solve_triangular(R[:rank, :rank], R[:rank, rank:])
    so, ro = np.argsort(sk), np.argsort(rd)
    return IdResult(sk[so], rd[ro], np.ascontiguousarray(T[np.ix_(so, ro)]))


def interpolative_decomposition(M, eps: float) -> IdResult:
    """CPQR column ID at relative tolerance eps (kernels.py:84-119).

    cut = max(eps, eps_mach * max(rows, cols)) * |R11|; rank = #{|R_kk| > cut};
    full rank -> no redundant columns; no rows or all-zero M -> all redundant.
    """
    if eps < 0.0:
        raise ValueError(f"eps must be >= 0, got {eps}")
    M = np.asarray(M, dtype=np.float64)
    if M.ndim != 2:
        raise ValueError("expected a 2-d array")
    nrows, ncols = M.shape
    none = np.zeros(0, dtype=np.intp)
    if ncols == 0:
        return IdResult(none, none, np.zeros((0, 0)))
    if nrows == 0 or not np.any(M):
        return IdResult(none, np.arange(ncols, dtype=np.intp), np.zeros((0, ncols)))
    R, perm = scipy.linalg.qr(M, mode="r", pivoting=True)
    return _id_from_r(R, perm, nrows, ncols, eps)


# ---------------------------------------------------------------------------
# dgeqp3 / dlaqp2 restatement (what the CUDA CPQR kernel implements)
# ---------------------------------------------------------------------------

def _dnrm2(x):
    # scaled 2-norm; the ordering of the sum differs from OpenBLAS only at ulp level
    return float(np.sqrt(np.dot(x, x))) if x.size else 0.0


def cpqr_dlaqp2(M):
    """Column-pivoted Householder QR, LAPACK dgeqp3 semantics for min(m,n) <= nx.

    Returns (R, perm) like scipy.linalg.qr(M, mode='r', pivoting=True) (R is
    min(m,n) x n upper trapezoidal). Follows dlaqp2 step by step: pivot =
    first index of max partial norm, Householder reflector with
    beta = -sign(alpha) * hypot(alpha, xnorm), trailing update, then the
    partial-norm downdate vn1 *= sqrt(1 - (|r_kj|/vn1)^2) with recomputation
    from the trailing column when temp * (vn1/vn2)^2 <= sqrt(eps/2).
    """
    A = np.array(M, dtype=np.float64, copy=True)
    m, n = A.shape
    perm = np.arange(n)
    vn1 = np.array([_dnrm2(A[:, j]) for j in range(n)])
    vn2 = vn1.copy()
    k = min(m, n)
    for i in range(k):
        p = i + int(np.argmax(vn1[i:]))
        if p != i:
            A[:, [i, p]] = A[:, [p, i]]
            perm[[i, p]] = perm[[p, i]]
            vn1[p] = vn1[i]
            vn2[p] = vn2[i]
        alpha = A[i, i]
        xnorm = _dnrm2(A[i + 1:, i])
        if xnorm == 0.0:
            tau = 0.0
            beta = alpha
        else:
            beta = -np.copysign(np.hypot(alpha, xnorm), alpha)
            tau = (beta - alpha) / beta
            A[i + 1:, i] *= 1.0 / (alpha - beta)
        A[i, i] = beta
        if i < n - 1 and tau != 0.0:
            v = np.concatenate([[1.0], A[i + 1:, i]])
            w = v @ A[i:, i + 1:]
            A[i:, i + 1:] -= tau * np.outer(v, w)
        for j in range(i + 1, n):
            if vn1[j] != 0.0:
                t = 1.0 - (abs(A[i, j]) / vn1[j]) ** 2
                t = max(t, 0.0)
                t2 = t * (vn1[j] / vn2[j]) ** 2
                if t2 <= TOL3Z:
                    if i < m - 1:
                        vn1[j] = _dnrm2(A[i + 1:, j])
                        vn2[j] = vn1[j]
                    else:
                        vn1[j] = 0.0
                        vn2[j] = 0.0
                else:
                    vn1[j] *= np.sqrt(t)
    R = np.triu(A[:k, :])
    return R, perm


def interpolative_decomposition_dlaqp2(M, eps: float) -> IdResult:
    """Same contract as interpolative_decomposition, but CPQR via cpqr_dlaqp2."""
    M = np.asarray(M, dtype=np.float64)
    nrows, ncols = M.shape
    none = np.zeros(0, dtype=np.intp)
    if ncols == 0:
        return IdResult(none, none, np.zeros((0, 0)))
    if nrows == 0 or not np.any(M):
        return IdResult(none, np.arange(ncols, dtype=np.intp), np.zeros((0, ncols)))
    R, perm = cpqr_dlaqp2(M)
    return _id_from_r(R, perm, nrows, ncols, eps)
