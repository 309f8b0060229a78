"""Problem setup: grid metadata, coefficient fields, 5/7-point operator assembly.

Host-side input construction for the factorize / PCG path. The public names and
semantics follow the reference `pkg/src/hifsolve/grid.py`:

* GridSpec(dim, n, m)           grid.py:26-89  (n = 2^L m, L >= 1, m >= 2; DOF ids x-fastest)
* CoefficientField              grid.py:92-121
* SymSparseMatrix               grid.py:124-179 (full symmetric CSR, matvec, lower_coo)
* generate_field                grid.py:182-210 (uniform -> Gaussian filter -> lower-median split)
* assemble_operator             grid.py:213-260 (arithmetic-mean half-point flux, h^2-scaled,
                                                 boundary half-points take the nodal value)

plus `baseline_field(cfg, seed)`: the five BASELINE.json coefficient recipes
(SURVEY.md section 8(d)), all on host numpy with the PCG64 generator.

This module is plumbing that builds the *input* of the hot path; nothing here
runs on the GPU and nothing here is timed as part of the factorization.
"""

from __future__ import annotations

import json
from dataclasses import dataclass

import numpy as np
import scipy.ndimage
import scipy.sparse as sp

from .errors import ConfigurationError

GENERATOR_NAME = "numpy-pcg64"


@dataclass(frozen=True)
class GridSpec:
    """Uniform grid, n subdivisions per axis with n = 2^L * m (grid.py:26-48)."""

    dim: int
    n: int
    m: int

    def __post_init__(self):
        if self.dim not in (2, 3):
            raise ConfigurationError(f"dim must be 2 or 3, got {self.dim}")
        if self.m < 2:
            raise ConfigurationError(f"leaf size m must be >= 2, got {self.m}")
        if self.n <= 0 or self.n % self.m:
            raise ConfigurationError(f"n={self.n} is not a multiple of m={self.m}")
        cells = self.n // self.m
        if cells < 2 or (cells & (cells - 1)):
            raise ConfigurationError(f"n={self.n} must equal 2^L * m with L >= 1 (m={self.m})")

    @property
    def levels(self) -> int:
        return (self.n // self.m).bit_length() - 1

    @property
    def h(self) -> float:
        return 1.0 / self.n

    @property
    def shape(self) -> tuple:
        return (self.n - 1,) * self.dim

    @property
    def ndofs(self) -> int:
        return (self.n - 1) ** self.dim

    def coords_of(self, ids) -> np.ndarray:
        """Lattice coordinates in 1..n-1 of DOF ids (x fastest), shape (..., dim)."""
        ids = np.asarray(ids, dtype=np.int64)
        side = self.n - 1
        strides = side ** np.arange(self.dim, dtype=np.int64)
        return (ids[..., None] // strides) % side + 1

    def id_of(self, coords) -> np.ndarray:
        c = np.asarray(coords, dtype=np.int64) - 1
        side = self.n - 1
        strides = side ** np.arange(self.dim, dtype=np.int64)
        return (c * strides).sum(axis=-1)


@dataclass(frozen=True)
class CoefficientField:
    """Nodal coefficient a on the interior lattice; values[x-1, y-1(, z-1)]."""

    spec: GridSpec
    values: np.ndarray
    seed: int
    contrast: float
    smoothing_width: float
    generator: str = GENERATOR_NAME

    def flat(self) -> np.ndarray:
        return np.ravel(self.values, order="F")

    def metadata(self) -> dict:
        s = self.spec
        return dict(dim=s.dim, n=s.n, m=s.m, L=s.levels, seed=int(self.seed),
                    contrast=float(self.contrast), smoothing_width=float(self.smoothing_width),
                    generator=self.generator)


class SymSparseMatrix:
    """Symmetric sparse matrix held as a full-pattern CSR (grid.py:124-179)."""

    def __init__(self, csr, check: bool = True):
        csr = sp.csr_array(csr)
        if csr.shape[0] != csr.shape[1]:
            raise ConfigurationError("matrix must be square")
        if check:
            asym = (csr - csr.T).tocsr()
            if asym.nnz:
                scale = max(1.0, float(np.abs(csr.data).max()))
                if float(np.abs(asym.data).max()) > 1e-12 * scale:
                    raise ConfigurationError("matrix is not symmetric")
        csr.sort_indices()
        self.csr = csr
        self._device = None  # cached device copy, owned by the B200 runtime

    @classmethod
    def from_coo_lower(cls, n, rows, cols, vals) -> "SymSparseMatrix":
        rows = np.asarray(rows, dtype=np.int64)
        cols = np.asarray(cols, dtype=np.int64)
        vals = np.asarray(vals, dtype=np.float64)
        if np.any(rows < cols):
            raise ConfigurationError("entries must lie in the lower triangle")
        off = rows != cols
        r = np.concatenate([rows, cols[off]])
        c = np.concatenate([cols, rows[off]])
        v = np.concatenate([vals, vals[off]])
        full = sp.coo_array((v, (r, c)), shape=(n, n)).tocsr()
        return cls(full, check=False)

    @property
    def n(self) -> int:
        return self.csr.shape[0]

    @property
    def nnz(self) -> int:
        return self.csr.nnz

    def matvec(self, x):
        return self.csr @ x

    def __matmul__(self, x):
        return self.csr @ x

    def to_dense(self) -> np.ndarray:
        return self.csr.toarray()

    def lower_coo(self):
        low = sp.tril(self.csr).tocoo()
        order = np.lexsort((low.col, low.row))
        return low.row[order], low.col[order], low.data[order]

    def write_coordinate(self, path):
        r, c, v = self.lower_coo()
        with open(path, "w") as fh:
            fh.write("%%MatrixMarket matrix coordinate real symmetric\n")
            fh.write(f"{self.n} {self.n} {len(v)}\n")
            fh.writelines(f"{i + 1} {j + 1} {x:.17g}\n" for i, j, x in zip(r, c, v))


def generate_field(spec: GridSpec, seed: int, contrast: float = 1e4,
                   smoothing_width: float = 4.0) -> CoefficientField:
    """Reference field recipe (grid.py:182-210): uniform, Gaussian smoothing, lower-median split."""
    if contrast < 1.0:
        raise ConfigurationError(f"contrast must be >= 1, got {contrast}")
    if smoothing_width <= 0.0:
        raise ConfigurationError("smoothing_width must be positive")
    raw = np.random.default_rng(seed).random(spec.shape)
    sm = scipy.ndimage.gaussian_filter(raw, sigma=smoothing_width, mode="reflect", truncate=4.0)
    flat = sm.ravel()
    k = (flat.size + 1) // 2
    median = np.partition(flat, k - 1)[k - 1]
    vals = np.where(sm <= median, contrast ** -0.5, contrast ** 0.5)
    return CoefficientField(spec, vals, seed, contrast, smoothing_width)


def assemble_operator(field: CoefficientField, b: float = 0.0) -> SymSparseMatrix:
    """h^2-scaled 5/7-point stencil of -div(a grad u) + b u (grid.py:213-260).

    Flux at a half-point between two lattice nodes is the mean of their a; a
    half-point next to the Dirichlet boundary uses the node's own a. The
    diagonal is accumulated in the same order as the reference (b h^2, then per
    axis the two interior half-points, then the boundary terms), so values agree
    bit for bit.
    """
    if b < 0.0:
        raise ConfigurationError(f"b must be >= 0, got {b}")
    spec = field.spec
    a = np.asarray(field.values, dtype=np.float64)
    if a.shape != spec.shape:
        raise ConfigurationError("field shape does not match its grid spec")
    side = spec.n - 1
    ids = np.arange(spec.ndofs, dtype=np.int64).reshape(spec.shape, order="F")
    diag = np.full(spec.shape, b * spec.h ** 2)
    lo_rows, lo_cols, lo_vals = [], [], []
    for d in range(spec.dim):
        lo = [slice(None)] * spec.dim
        hi = [slice(None)] * spec.dim
        lo[d] = slice(0, side - 1)
        hi[d] = slice(1, side)
        lo, hi = tuple(lo), tuple(hi)
        flux = 0.5 * (a[lo] + a[hi])
        diag[lo] += flux
        diag[hi] += flux
        lo_rows.append(ids[hi].ravel())
        lo_cols.append(ids[lo].ravel())
        lo_vals.append(-flux.ravel())
        first = [slice(None)] * spec.dim
        last = [slice(None)] * spec.dim
        first[d] = 0
        last[d] = side - 1
        diag[tuple(first)] += a[tuple(first)]
        diag[tuple(last)] += a[tuple(last)]
    lo_rows.append(ids.ravel())
    lo_cols.append(ids.ravel())
    lo_vals.append(diag.ravel())
    return SymSparseMatrix.from_coo_lower(spec.ndofs, np.concatenate(lo_rows),
                                          np.concatenate(lo_cols), np.concatenate(lo_vals))


# ---------------------------------------------------------------------------
# BASELINE.json configurations
# ---------------------------------------------------------------------------

@dataclass(frozen=True)
class BaselineConfig:
    name: str
    dim: int
    n: int
    m: int
    b: float
    eps: tuple
    method: str
    nrhs: int
    tol: float
    recipe: str
    description: str


CONFIGS = {
    "c1": BaselineConfig("c1", 2, 128, 8, 0.0, (1e-6,), "phif", 1, 1e-12, "iid_log2",
                         "2D 127^2, a=10^(2(2U-1)) iid, m=8, eps 1e-6, PHIF, 1 RHS, tol 1e-12"),
    "c2": BaselineConfig("c2", 2, 512, 8, 0.0, (1e-3,), "phif", 1, 1e-12, "thresh_2d_s4_1e3",
                         "2D 511^2, smoothed-threshold a in {1e-3,1e3} (std 4), m=8, eps 1e-3, PHIF/HIF"),
    "c3": BaselineConfig("c3", 2, 2048, 16, 1e-6, (1e-2, 1e-4), "phif", 8, 1e-12, "thresh_2d_s4_1e4",
                         "2D 2047^2, smoothed-threshold a in {1e-4,1e4} (std 4), b=1e-6, m=16, "
                         "eps 1e-2/1e-4, PHIF, 8 RHS, tol 1e-12"),
    # c3 geometry with the paper's contrast (a in {1e-2, 1e2}): the specified
    # contrast-1e8 field loses positive definiteness at level 1 for eps 1e-2 and 1e-4
    "c3p": BaselineConfig("c3p", 2, 2048, 16, 1e-6, (1e-4,), "phif", 8, 1e-12, "thresh_2d_s4_1e2",
                          "2D 2047^2, smoothed-threshold a in {1e-2,1e2} (std 4), b=1e-6, m=16, eps 1e-4, "
                          "PHIF, 8 RHS, tol 1e-12 (c3 with the paper's contrast)"),
    "c4": BaselineConfig("c4", 3, 64, 4, 0.0, (1e-3,), "phif", 1, 1e-12, "smooth_log3_s2",
                         "3D 63^3, a=10^(3(2Us-1)) Us smoothed uniform (std 2), m=4, eps 1e-3, PHIF"),
    "c5": BaselineConfig("c5", 3, 128, 4, 0.0, (1e-2,), "phif", 32, 1e-10, "thresh_3d_s3_1e3",
                         "3D 127^3, smoothed-threshold a in {1e-3,1e3} (std 3), m=4, eps 1e-2, "
                         "PHIF, 32 RHS, tol 1e-10"),
}


def baseline_field(cfg: BaselineConfig | str, seed: int = 0, n: int | None = None) -> CoefficientField:
    """Coefficient field of a BASELINE config (optionally at a reduced grid size n)."""
    if isinstance(cfg, str):
        cfg = CONFIGS[cfg]
    spec = GridSpec(cfg.dim, n or cfg.n, cfg.m)
    rng = np.random.default_rng(seed)
    shape = spec.shape
    if cfg.recipe == "iid_log2":
        u = rng.random(shape)
        vals, contrast, width = 10.0 ** (2.0 * (2.0 * u - 1.0)), 1e4, 0.0
    elif cfg.recipe.startswith("thresh_"):
        _, _, sig, hi = cfg.recipe.split("_")
        sigma, top = float(sig[1:]), float(hi)
        g = scipy.ndimage.gaussian_filter(rng.standard_normal(shape), sigma=sigma,
                                          mode="reflect", truncate=4.0)
        vals, contrast, width = np.where(g > 0.0, top, 1.0 / top), top * top, sigma
    elif cfg.recipe == "smooth_log3_s2":
        us = scipy.ndimage.gaussian_filter(rng.random(shape), sigma=2.0, mode="reflect", truncate=4.0)
        vals, contrast, width = 10.0 ** (3.0 * (2.0 * us - 1.0)), 1e6, 2.0
    else:
        raise ConfigurationError(f"unknown recipe {cfg.recipe}")
    return CoefficientField(spec, vals, seed, contrast, width)


def baseline_problem(cfg: BaselineConfig | str, seed: int = 0, n: int | None = None):
    """(spec, A, field) for a BASELINE config; A assembled exactly as assemble_operator."""
    if isinstance(cfg, str):
        cfg = CONFIGS[cfg]
    field = baseline_field(cfg, seed, n)
    return field.spec, assemble_operator(field, cfg.b), field


def baseline_rhs(cfg: BaselineConfig | str, N: int, seed: int = 0, nrhs: int | None = None) -> np.ndarray:
    """RHS block f ~ N(0,1) from default_rng([seed, 1]); shape (N, nrhs)."""
    if isinstance(cfg, str):
        cfg = CONFIGS[cfg]
    k = nrhs or cfg.nrhs
    return np.random.default_rng([seed, 1]).standard_normal((N, k))


def write_metadata_json(field: CoefficientField, path):
    with open(path, "w") as fh:
        json.dump(field.metadata(), fh, indent=2)
        fh.write("\n")
