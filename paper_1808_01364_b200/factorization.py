"""factorize / apply-inverse entry points (drop-in for the absent `hifsolve.factorization`).

Same names, arguments and error behaviour as SPEC.md:229-347:

* factorize(A, spec, eps, method)  SPEC.md:275-283 -> Factorization (device-resident records)
* apply_inverse(Fz, b)             SPEC.md:293-301  F^-1 b
* apply_ginv(Fz, x), apply_ginv_t  SPEC.md:302-310  G^-1 x, G^-T x
* NotSpdError(pivot, level, stage, group, partial_stats) on a failed pivot

The work runs in libphif_b200.so (csrc/): a C++ level planner plus batched
sm_100a FP64 kernels; this module only marshals numpy arrays across the C-ABI.
Vectors are numpy (N,) or (N, nrhs) arrays, as in the reference.
"""

from __future__ import annotations

import ctypes as C
import json

import numpy as np

from . import _lib
from .errors import ConfigurationError
from .grid import GridSpec, SymSparseMatrix


class DeviceMatrix:
    """Symmetric CSR uploaded to HBM once (cached on the SymSparseMatrix)."""

    def __init__(self, A: SymSparseMatrix, stream=None):
        csr = A.csr
        self.N = csr.shape[0]
        self.rowptr = np.ascontiguousarray(csr.indptr, dtype=np.int64)
        self.col = np.ascontiguousarray(csr.indices, dtype=np.int32)
        self.val = np.ascontiguousarray(csr.data, dtype=np.float64)
        L = _lib.lib()
        h = C.c_void_p()
        err = _lib.phif_error()
        rc = L.phif_matrix_create(_lib.ptr(self.rowptr), _lib.ptr(self.col), _lib.ptr(self.val), self.N,
                                  C.c_void_p(stream or 0), C.byref(h), C.byref(err))
        _lib.raise_for(rc, err)
        self.handle = h

    def __del__(self):
        h = getattr(self, "handle", None)
        try:
            if h and _lib._lib is not None:
                _lib._lib.phif_matrix_free(h)
        except (AttributeError, TypeError):   # interpreter shutdown: module globals already gone
            pass
        self.handle = None


def device_matrix(A, stream=None) -> DeviceMatrix:
    if isinstance(A, DeviceMatrix):
        return A
    if not isinstance(A, SymSparseMatrix):
        A = SymSparseMatrix(A)
    if getattr(A, "_device", None) is None:
        A._device = DeviceMatrix(A, stream)
    return A._device


class Factorization:
    """Handle to a device-resident PHIF/HIF factorization (F = G G^T, PAPER.md eq. eqF)."""

    def __init__(self, handle, method, eps, spec, N):
        self.handle = handle
        self.method = method
        self.eps = eps
        self.spec = spec
        self.N = N
        self._stats = None

    def __del__(self):
        h = getattr(self, "handle", None)
        try:
            if h and _lib._lib is not None:
                _lib._lib.phif_factor_free(h)
        except (AttributeError, TypeError):   # interpreter shutdown: module globals already gone
            pass
        self.handle = None

    @property
    def stats(self) -> dict:
        if self._stats is None:
            L = _lib.lib()
            n = L.phif_stats_json(self.handle, None, 0)
            buf = C.create_string_buffer(n + 1)
            L.phif_stats_json(self.handle, buf, n + 1)
            self._stats = json.loads(buf.value.decode())
        return self._stats

    @property
    def SL(self) -> int:
        return int(self.stats["SL"])

    @property
    def num_levels(self) -> int:
        return _lib.lib().phif_num_levels(self.handle)

    def skeleton_sets(self, level: int):
        """[(skeleton_dofs, redundant_dofs)] per separator group of `level` (classify order)."""
        L = _lib.lib()
        counts = np.zeros(3, dtype=np.int64)
        L.phif_skeleton_sets(self.handle, level, _lib.ptr(counts), None, None, None, None)
        nsk, rs, ks = (int(v) for v in counts)
        rank = np.zeros(max(nsk, 1), dtype=np.int32)
        nred = np.zeros(max(nsk, 1), dtype=np.int32)
        sk = np.zeros(max(rs, 1), dtype=np.int32)
        rd = np.zeros(max(ks, 1), dtype=np.int32)
        L.phif_skeleton_sets(self.handle, level, _lib.ptr(counts), _lib.ptr(rank), _lib.ptr(nred), _lib.ptr(sk),
                             _lib.ptr(rd))
        out, a, b = [], 0, 0
        for t in range(nsk):
            r, kt = int(rank[t]), int(nred[t])
            out.append((sk[a:a + r].astype(np.int64), rd[b:b + kt].astype(np.int64)))
            a += r
            b += kt
        return out


def factorize(A, spec: GridSpec, eps: float, method: str = "phif", stream=None, timing: bool = False):
    """Factor A on `spec` with ID tolerance eps; method in {"hif", "phif", "exact"}."""
    method = method.lower()
    if method not in _lib.METHODS:
        raise ConfigurationError(f"unknown method {method!r}")
    if eps < 0:
        raise ConfigurationError("eps must be >= 0")
    dm = device_matrix(A, stream)
    if dm.N != spec.ndofs:
        raise ConfigurationError(f"matrix order {dm.N} does not match the grid ({spec.ndofs} DOFs)")
    L = _lib.lib()
    h = C.c_void_p()
    err = _lib.phif_error()
    rc = L.phif_factorize(dm.handle, spec.dim, spec.n, spec.m, float(eps), _lib.METHODS[method],
                          C.c_void_p(stream or 0), 1 if timing else 0, C.byref(h), C.byref(err))
    _lib.raise_for(rc, err)
    return Factorization(h, method, 0.0 if method == "exact" else eps, spec, dm.N)


def _apply(Fz: Factorization, x, mode: int):
    x = np.asarray(x, dtype=np.float64)
    flat = x.ndim == 1
    X = np.ascontiguousarray(x.reshape(x.shape[0], -1)).copy()
    if X.shape[0] != Fz.N:
        raise ConfigurationError("vector length does not match the factorization")
    err = _lib.phif_error()
    rc = _lib.lib().phif_apply(Fz.handle, _lib.ptr(X), X.shape[1], mode, C.byref(err))
    _lib.raise_for(rc, err)
    return X[:, 0] if flat else X


def apply_inverse(Fz: Factorization, b):
    """F^-1 b = R_0 ... R_{L-1} A_L^-1 R_{L-1}^T ... R_0^T b (PAPER.md eq. eqAinv)."""
    return _apply(Fz, b, 0)


def apply_ginv(Fz: Factorization, x):
    """G^-1 x = B_L^-1 R_{L-1}^T ... R_0^T x."""
    return _apply(Fz, x, 1)


def apply_ginv_t(Fz: Factorization, x):
    """G^-T x = R_0 ... R_{L-1} B_L^-T x."""
    return _apply(Fz, x, 2)


def apply(Fz: Factorization, x):
    """F x = G G^T x = R_0^-T ... R_{L-1}^-T A_L R_{L-1}^-1 ... R_0^-1 x (PAPER.md eq. eqA):
    the records replayed in reverse with triangular multiplications."""
    return _apply(Fz, x, 3)


def apply_g(Fz: Factorization, x):
    """G x (the forward generalized Cholesky factor, F = G G^T)."""
    return _apply(Fz, x, 5)


def apply_g_t(Fz: Factorization, x):
    """G^T x."""
    return _apply(Fz, x, 4)


ROOT_DENSE_MAX = 5000


def root_factor(Fz: Factorization) -> np.ndarray:
    """The root Cholesky factor B_L (|S_L| x |S_L|, lower), copied to the host."""
    n = C.c_int()
    err = _lib.phif_error()
    L = _lib.lib()
    rc = L.phif_root_factor(Fz.handle, None, C.byref(n), C.byref(err))
    _lib.raise_for(rc, err)
    out = np.zeros((n.value, n.value), dtype=np.float64)
    if n.value:
        rc = L.phif_root_factor(Fz.handle, _lib.ptr(out), C.byref(n), C.byref(err))
        _lib.raise_for(rc, err)
    return out


def root_condition(Fz: Factorization) -> float:
    """kappa(A_L) of the retained root block: exact, from the singular values of
    its Cholesky factor (A_L = B_L B_L^T). Refuses |S_L| > 5000 like the reference's size guard."""
    n = C.c_int()
    err = _lib.phif_error()
    rc = _lib.lib().phif_root_factor(Fz.handle, None, C.byref(n), C.byref(err))
    _lib.raise_for(rc, err)
    if n.value == 0:
        return 1.0
    if n.value > ROOT_DENSE_MAX:
        raise ConfigurationError(f"root block too large for a dense condition number: |S_L| = {n.value}")
    s = np.linalg.svd(root_factor(Fz), compute_uv=False)
    return float((s[0] / s[-1]) ** 2)
