"""Generate golden vectors from the reference's own modules (run in the build container).

    PYTHONPATH=/root/reference/pkg/src python tests/golden/make_golden.py

Calls only the reference's importable primitives (hifsolve.kernels, .hierarchy,
.grid; the factorization/krylov/diagnostics modules do not exist upstream) and
stores their inputs and outputs in tests/golden/reference_golden.npz. The CPU
tests pin the oracle (oracle/dense.py, oracle/hierarchy.py) and the product's
input construction (paper_1808_01364_b200/grid.py) and C++ planner against it.
"""
import os
import sys

import numpy as np

sys.path.insert(0, os.environ.get("HIFSOLVE_SRC", "/root/reference/pkg/src"))
from hifsolve import grid as rgrid, hierarchy as rhier, kernels as rk  # noqa: E402
from hifsolve.errors import NotSpdError  # noqa: E402

out = {}
rng = np.random.default_rng(20260101)


def put(key, arr):
    out[key] = np.asarray(arr)


# ---- cholesky: SPD matrices of hot-path sizes and NotSpd pivots ----
for i, k in enumerate([1, 2, 7, 15, 27, 49]):
    G = rng.standard_normal((k, k))
    S = G @ G.T + k * np.eye(k)
    put(f"chol_{i}_in", S)
    put(f"chol_{i}_out", rk.cholesky(S))
for i, S in enumerate([np.array([[1.0, 2.0], [2.0, 1.0]]), np.diag([3.0, 2.0, -1.0, 4.0]),
                       np.array([[4.0, 2.0, 2.0], [2.0, 1.0, 1.0], [2.0, 1.0, 5.0]])]):
    try:
        rk.cholesky(S)
        piv = -1
    except NotSpdError as e:
        piv = e.pivot
    put(f"chol_bad_{i}_in", S)
    put(f"chol_bad_{i}_pivot", piv)

# ---- tri_solve: all four op/side combinations ----
for i, (trans, side) in enumerate([(False, "left"), (True, "left"), (False, "right"), (True, "right")]):
    k = 9
    L = np.tril(rng.standard_normal((k, k))) + 4 * np.eye(k)
    B = rng.standard_normal((k, 5)) if side == "left" else rng.standard_normal((5, k))
    put(f"tri_{i}_L", L)
    put(f"tri_{i}_B", B)
    put(f"tri_{i}_flags", [int(trans), int(side == "right")])
    put(f"tri_{i}_out", rk.tri_solve(L, B, trans=trans, side=side))

# ---- interpolative_decomposition: hot-path shapes, low rank, wide, ties, zero ----
id_cases = []
for (m, n, r) in [(44, 7, 7), (44, 7, 4), (88, 15, 15), (88, 15, 6), (11, 15, 11), (102, 9, 9),
                  (102, 9, 5), (20, 4, 2), (200, 31, 12), (60, 40, 25)]:
    M = rng.standard_normal((m, r)) @ rng.standard_normal((r, n))
    M += 1e-9 * rng.standard_normal((m, n)) * (r < min(m, n))
    for eps in (1e-2, 1e-6, 0.0):
        id_cases.append((M, eps))
# graded columns (rank revealed by a decaying spectrum)
for (m, n) in [(44, 7), (88, 15), (102, 9)]:
    U, _ = np.linalg.qr(rng.standard_normal((m, n)))
    V, _ = np.linalg.qr(rng.standard_normal((n, n)))
    M = U @ np.diag(np.logspace(0, -12, n)) @ V
    for eps in (1e-2, 1e-4, 1e-6, 1e-8):
        id_cases.append((M, eps))
# exact column-norm ties, duplicated columns, zero matrix, no rows, identity
T = rng.standard_normal((30, 3))
id_cases.append((np.hstack([T, T, T[:, :1] * 2.0]), 1e-6))
id_cases.append((np.array([[1.0, 2.0], [2.0, 4.0]]), 1e-6))
id_cases.append((np.eye(6), 1e-6))
id_cases.append((np.zeros((5, 3)), 1e-6))
id_cases.append((np.zeros((0, 4)), 1e-6))
for i, (M, eps) in enumerate(id_cases):
    res = rk.interpolative_decomposition(M, eps)
    put(f"id_{i}_M", M)
    put(f"id_{i}_eps", eps)
    put(f"id_{i}_skel", res.skeleton)
    put(f"id_{i}_red", res.redundant)
    put(f"id_{i}_T", res.interp)
put("id_count", len(id_cases))

# ---- classify_active: full and random active sets on small grids ----
cls = 0
for (dim, n, m) in [(2, 16, 4), (2, 64, 8), (3, 16, 4), (3, 32, 4)]:
    spec = rgrid.GridSpec(dim, n, m)
    for lev in range(spec.levels + 1):
        for frac in (1.0, 0.4):
            if frac == 1.0:
                act = np.arange(spec.ndofs)
            else:
                act = np.sort(rng.choice(spec.ndofs, int(frac * spec.ndofs), replace=False))
            part = rhier.classify_active(spec, lev, act)
            groups = part.interior_groups + part.precond_groups
            # classify order of the union: re-sort by the reference's own list order
            put(f"cls_{cls}_spec", [dim, n, m, lev])
            put(f"cls_{cls}_active", act)
            put(f"cls_{cls}_interior_sizes", [len(g) for g in part.interior_groups])
            put(f"cls_{cls}_interior", np.concatenate([g.indices for g in part.interior_groups])
                if part.interior_groups else np.zeros(0, np.int64))
            put(f"cls_{cls}_precond_sizes", [len(g) for g in part.precond_groups])
            put(f"cls_{cls}_precond", np.concatenate([g.indices for g in part.precond_groups])
                if part.precond_groups else np.zeros(0, np.int64))
            put(f"cls_{cls}_skeleton_sizes", [len(g) for g in part.skeleton_groups])
            put(f"cls_{cls}_skeleton", np.concatenate([g.indices for g in part.skeleton_groups])
                if part.skeleton_groups else np.zeros(0, np.int64))
            cls += 1
put("cls_count", cls)

# ---- grid: generate_field + assemble_operator ----
for i, (dim, n, m, seed, contrast, width, b) in enumerate([(2, 32, 4, 3, 1e4, 4.0, 0.0), (2, 16, 8, 5, 1e2, 2.0, 1.5),
                                                            (3, 8, 4, 7, 1e4, 1.0, 0.0), (3, 16, 4, 9, 1e6, 2.0, 1e-3)]):
    spec = rgrid.GridSpec(dim, n, m)
    f = rgrid.generate_field(spec, seed, contrast, width)
    A = rgrid.assemble_operator(f, b)
    put(f"grid_{i}_params", [dim, n, m, seed, contrast, width, b])
    put(f"grid_{i}_field", f.values)
    put(f"grid_{i}_indptr", A.csr.indptr)
    put(f"grid_{i}_indices", A.csr.indices)
    put(f"grid_{i}_data", A.csr.data)
put("grid_count", 4)

path = os.path.join(os.path.dirname(os.path.abspath(__file__)), "reference_golden.npz")
np.savez_compressed(path, **out)
print("wrote", path, len(out), "arrays", os.path.getsize(path), "bytes")
