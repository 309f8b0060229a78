"""On-device problem generation and ingest (reference grid.py:182-260).

The random draws of a BASELINE field recipe stay on the host (numpy PCG64, default_rng(seed), the
same calls as grid.baseline_field), everything after them runs on the B200 through
`phif_matrix_from_field`: the Gaussian smoothing (scipy.ndimage.gaussian_filter's summation order,
reflect boundary, truncate 4), the threshold of the smoothed-threshold recipes, and the stencil
assembly of A = -div(a grad u) + b u straight into the device CSR. The result is bit-identical to
the host `baseline_problem` (tests/test_gpu_device_problem.py), skips the host assembly and uploads
one lattice of N doubles instead of the CSR; the matrix keeps its field, so PCG and the estimators
use the matrix-free stencil SpMV.

Recipes whose value transform is a power (10^x: iid_log2, smooth_log3_s2) apply it on the host
(numpy's pow is the reference; the device only smooths/assembles there).
"""

from __future__ import annotations

import ctypes as C

import numpy as np

from . import _lib
from .factorization import DeviceMatrix
from .grid import CONFIGS, BaselineConfig, GridSpec


def gaussian_weights(sigma: float, truncate: float = 4.0) -> np.ndarray:
    """scipy.ndimage's 1-D Gaussian kernel (radius int(truncate sigma + 0.5), normalised)."""
    radius = int(truncate * float(sigma) + 0.5)
    x = np.arange(-radius, radius + 1)
    phi = np.exp(np.polynomial.Polynomial([0, 0, -0.5 / (sigma * sigma)])(x), dtype=np.double)
    phi /= phi.sum()
    return phi


class DeviceProblemMatrix(DeviceMatrix):
    """A device matrix assembled on the GPU from a coefficient lattice (no host CSR)."""

    def __init__(self, spec: GridSpec, lattice: np.ndarray, weights, lo: float, hi: float, bh2: float, stream=None):
        self.N = spec.ndofs
        self.spec = spec
        lat = np.ascontiguousarray(np.asarray(lattice, dtype=np.float64).ravel(order="F"))
        w = np.ascontiguousarray(np.asarray(weights if weights is not None else [], dtype=np.float64))
        L = _lib.lib()
        h = C.c_void_p()
        err = _lib.phif_error()
        rc = L.phif_matrix_from_field(spec.dim, spec.n, _lib.ptr(lat), _lib.ptr(w) if w.size else None, int(w.size),
                                      float(lo), float(hi), float(bh2), C.c_void_p(stream or 0), C.byref(h),
                                      C.byref(err))
        _lib.raise_for(rc, err)
        self.handle = h
        self.h2d_bytes = lat.nbytes + w.nbytes

    def csr(self):
        """(rowptr, col, val, field) copied back to the host (checks)."""
        L = _lib.lib()
        nnz = C.c_int64()
        L.phif_matrix_csr(self.handle, C.byref(nnz), None, None, None, None)
        rp = np.zeros(self.N + 1, np.int64)
        ci = np.zeros(nnz.value, np.int32)
        va = np.zeros(nnz.value, np.float64)
        fd = np.zeros(self.N, np.float64)
        L.phif_matrix_csr(self.handle, C.byref(nnz), _lib.ptr(rp), _lib.ptr(ci), _lib.ptr(va), _lib.ptr(fd))
        return rp, ci, va, fd

    def matvec(self, x, force_csr=False):
        x = np.ascontiguousarray(np.asarray(x, dtype=np.float64))
        X = x.reshape(x.shape[0], -1)
        Y = np.zeros_like(X)
        err = _lib.phif_error()
        rc = _lib.lib().phif_matrix_apply(self.handle, _lib.ptr(np.ascontiguousarray(X)), _lib.ptr(Y), X.shape[1],
                                          1 if force_csr else 0, C.byref(err))
        _lib.raise_for(rc, err)
        return Y.reshape(x.shape)


def device_baseline_problem(cfg: BaselineConfig | str, seed: int = 0, n: int | None = None, stream=None):
    """(spec, DeviceProblemMatrix) of a BASELINE config, generated and assembled on the device."""
    if isinstance(cfg, str):
        cfg = CONFIGS[cfg]
    spec = GridSpec(cfg.dim, n or cfg.n, cfg.m)
    rng = np.random.default_rng(seed)
    shape = spec.shape
    bh2 = cfg.b * spec.h ** 2
    if cfg.recipe.startswith("thresh_"):
        _, _, sig, hi = cfg.recipe.split("_")
        sigma, top = float(sig[1:]), float(hi)
        noise = rng.standard_normal(shape)
        M = DeviceProblemMatrix(spec, noise, gaussian_weights(sigma), 1.0 / top, top, bh2, stream)
    elif cfg.recipe == "iid_log2":
        u = rng.random(shape)
        M = DeviceProblemMatrix(spec, 10.0 ** (2.0 * (2.0 * u - 1.0)), None, 0.0, 0.0, bh2, stream)
    elif cfg.recipe == "smooth_log3_s2":
        import scipy.ndimage
        us = scipy.ndimage.gaussian_filter(rng.random(shape), sigma=2.0, mode="reflect", truncate=4.0)
        M = DeviceProblemMatrix(spec, 10.0 ** (3.0 * (2.0 * us - 1.0)), None, 0.0, 0.0, bh2, stream)
    else:
        raise ValueError(f"unknown recipe {cfg.recipe}")
    return spec, M
