"""PHIF / HIF factorization oracle (restates the absent `factorization` module).

TEST INFRASTRUCTURE ONLY (see oracle/__init__.py).

Algorithm, for l = 0 .. L-1:

1. eliminate_cells: for each interior group I
   in classify order: L = chol(A_II); X = L^-1 A_BI^T; A_BB -= X^T X, where B is
   every active DOF of a group holding a stored block with I. Record
   Eliminate(I, B, L, X).
2. precondition, PHIF only: for each
   non-interior group g: L_g = chol(A_gg); A_hg <- A_hg L_g^-T for every coupled h;
   A_gg <- I. Record Precondition(g, L_g).
3. skeletonize, sequential in
   classify order over edges (2D) / faces (3D): M = A_{R,I} over active rows R
   outside I with a nonzero entry in the current matrix; ID(M, eps) ->
   (skeleton ^I, redundant ~I, T); zeroing update; L~ =
   chol(A~_~I~I); X~ = L~^-1 A~_^I~I^T; A_^I^I -= X~^T X~; drop A_{R,~I}.
   Record Skeletonize(~I, ^I, T, L~, X~).
At level L the single remaining cell's interior is S_L: its elimination record
(empty B) is the root factor B_L.

method = "hif" skips stage 2; method = "exact" is the PHIF pipeline with eps = 0
(full-numerical-rank IDs).

The live matrix is a block store keyed by (group, group) of the current level
(SPEC.md:333), g <= h in classify order; a missing block is structurally zero.
"""

from __future__ import annotations

import time
from dataclasses import dataclass, field

import numpy as np
import scipy.linalg

from .dense import cholesky, interpolative_decomposition, tri_solve
from .errors import NotSpdError
from .hierarchy import classify_active


@dataclass
class Eliminate:
    I: np.ndarray
    B: np.ndarray
    L: np.ndarray
    X: np.ndarray


@dataclass
class Precondition:
    I: np.ndarray
    L: np.ndarray


@dataclass
class Skeletonize:
    redundant: np.ndarray
    skeleton: np.ndarray
    T: np.ndarray
    L: np.ndarray
    X: np.ndarray
    group: int = -1


@dataclass
class LevelRecords:
    level: int
    eliminate: list = field(default_factory=list)
    precondition: list = field(default_factory=list)
    skeletonize: list = field(default_factory=list)


@dataclass
class Factorization:
    method: str
    eps: float
    N: int
    L: int
    levels: list
    root_set: np.ndarray
    stats: dict

    @property
    def root_factor(self):
        return self.levels[-1].eliminate[0].L if self.levels[-1].eliminate else np.zeros((0, 0))

    @property
    def SL(self):
        return len(self.root_set)


class _Store:
    """Dense blocks of the live matrix keyed (g, h), g <= h."""

    def __init__(self, members):
        self.members = [np.asarray(m, dtype=np.int64) for m in members]
        self.blk = {}
        self.adj = [set() for _ in members]

    def get(self, g, h):
        if g <= h:
            b = self.blk.get((g, h))
            return b if b is not None else np.zeros((len(self.members[g]), len(self.members[h])))
        b = self.blk.get((h, g))
        return b.T if b is not None else np.zeros((len(self.members[g]), len(self.members[h])))

    def add(self, g, h, U):
        """block(g, h) += U (U oriented rows g, cols h)."""
        if g > h:
            g, h, U = h, g, U.T
        b = self.blk.get((g, h))
        if b is None:
            self.blk[(g, h)] = np.array(U, dtype=np.float64, copy=True)
            self.adj[g].add(h)
            self.adj[h].add(g)
        else:
            b += U

    def put(self, g, h, V):
        if g > h:
            g, h, V = h, g, V.T
        self.blk[(g, h)] = np.ascontiguousarray(V)
        self.adj[g].add(h)
        self.adj[h].add(g)

    def drop_group(self, g):
        for h in list(self.adj[g]):
            self.blk.pop((min(g, h), max(g, h)), None)
            self.adj[h].discard(g)
        self.adj[g] = set()
        self.members[g] = self.members[g][:0]

    def shrink(self, g, keep):
        """Keep only local positions `keep` of group g in every block touching g."""
        self.members[g] = self.members[g][keep]
        for h in self.adj[g]:
            if h == g:
                self.blk[(g, g)] = np.ascontiguousarray(self.blk[(g, g)][np.ix_(keep, keep)])
            elif g < h:
                self.blk[(g, h)] = np.ascontiguousarray(self.blk[(g, h)][keep, :])
            else:
                self.blk[(h, g)] = np.ascontiguousarray(self.blk[(h, g)][:, keep])

    def neighbours(self, g):
        return sorted(h for h in self.adj[g] if h != g)


def _store_from_csr(csr, groups, N):
    members = [g.indices for g in groups]
    st = _Store(members)
    gid = np.full(N, -1, dtype=np.int64)
    pos = np.full(N, -1, dtype=np.int64)
    for g, mem in enumerate(members):
        gid[mem] = g
        pos[mem] = np.arange(len(mem))
    coo = csr.tocoo()
    r, c, v = coo.row.astype(np.int64), coo.col.astype(np.int64), coo.data
    gi, gj = gid[r], gid[c]
    keep = (gi >= 0) & (gj >= 0) & (gi <= gj) & (v != 0.0)
    r, c, v, gi, gj = r[keep], c[keep], v[keep], gi[keep], gj[keep]
    G = len(members)
    pk = gi * G + gj
    order = np.argsort(pk, kind="stable")
    pk, r, c, v = pk[order], r[order], c[order], v[order]
    cuts = np.flatnonzero(np.diff(pk)) + 1
    for a, b in zip(np.concatenate([[0], cuts]), np.concatenate([cuts, [len(pk)]])):
        g, h = divmod(int(pk[a]), G)
        blk = np.zeros((len(members[g]), len(members[h])))
        blk[pos[r[a:b]], pos[c[a:b]]] = v[a:b]
        st.put(g, h, blk)
    return st


def _regroup(old: _Store, groups, N):
    """Carry the live matrix to the next level's grouping (level transition)."""
    new = _Store([g.indices for g in groups])
    gid = np.full(N, -1, dtype=np.int64)
    pos = np.full(N, -1, dtype=np.int64)
    for G, mem in enumerate(new.members):
        gid[mem] = G
        pos[mem] = np.arange(len(mem))
    target = []
    for g, mem in enumerate(old.members):
        if len(mem) == 0:
            target.append(-1)
            continue
        t = np.unique(gid[mem])
        if len(t) != 1 or t[0] < 0:
            raise AssertionError("an old group split across new groups")
        target.append(int(t[0]))
    acc = {}

    def slot(A, B):
        d = acc.get((A, B))
        if d is None:
            d = acc[(A, B)] = np.zeros((len(new.members[A]), len(new.members[B])))
        return d

    for (g, h), blk in old.blk.items():
        G, H = target[g], target[h]
        if G < 0 or H < 0:
            continue
        pg, ph = pos[old.members[g]], pos[old.members[h]]
        if G < H:
            slot(G, H)[np.ix_(pg, ph)] = blk
        elif G > H:
            slot(H, G)[np.ix_(ph, pg)] = blk.T
        else:
            d = slot(G, G)
            d[np.ix_(pg, ph)] = blk
            if g != h:
                d[np.ix_(ph, pg)] = blk.T
    for (A, B), blk in acc.items():
        new.put(A, B, blk)
    return new


def store_from_dense(A, groups):
    """Block store of a dense symmetric matrix for the given index groups (test helper)."""
    A = np.asarray(A, dtype=np.float64)
    st = _Store([np.asarray(g, dtype=np.int64) for g in groups])
    for g in range(len(groups)):
        for h in range(g, len(groups)):
            blk = A[np.ix_(st.members[g], st.members[h])]
            if np.any(blk != 0.0) or g == h:
                st.put(g, h, blk.copy())
    return st


def store_to_dense(st, N):
    """Dense live matrix (eliminated DOFs appear as identity rows/cols)."""
    D = np.eye(N)
    alive = np.concatenate([m for m in st.members if len(m)]) if any(len(m) for m in st.members) else []
    D[np.ix_(alive, alive)] = 0.0
    for (g, h), blk in st.blk.items():
        D[np.ix_(st.members[g], st.members[h])] = blk
        D[np.ix_(st.members[h], st.members[g])] = blk.T
    return D


def eliminate_cells(store, interior, level=None, stage="eliminate", stats=None):
    """Stage 1: block elimination of each interior group, in order."""
    recs = []
    for t, gi in enumerate(interior):
        nb = store.neighbours(gi)
        Aii = store.get(gi, gi)
        Abt = np.hstack([store.get(gi, h) for h in nb]) if nb else np.zeros((len(Aii), 0))
        try:
            Lc = cholesky(Aii)
        except NotSpdError as e:
            raise NotSpdError(e.pivot, level, stage, t, stats) from None
        X = tri_solve(Lc, Abt)
        off = np.cumsum([0] + [len(store.members[h]) for h in nb])
        for a, ha in enumerate(nb):
            Xa = X[:, off[a]:off[a + 1]]
            for b in range(a, len(nb)):
                store.add(ha, nb[b], -(Xa.T @ X[:, off[b]:off[b + 1]]))
        Bidx = np.concatenate([store.members[h] for h in nb]) if nb else np.zeros(0, np.int64)
        recs.append(Eliminate(store.members[gi].copy(), Bidx, Lc, X))
        store.drop_group(gi)
    return recs


def precondition_blocks(store, groups, level=None, stats=None):
    """Stage 2: two-sided block-Jacobi scaling, A_gg -> I."""
    recs = []
    for t, g in enumerate(groups):
        try:
            Lg = cholesky(store.get(g, g))
        except NotSpdError as e:
            raise NotSpdError(e.pivot, level, "precondition", t, stats) from None
        for h in store.neighbours(g):
            if g < h:
                store.blk[(g, h)] = scipy.linalg.solve_triangular(Lg, store.blk[(g, h)], lower=True)
            else:
                store.blk[(h, g)] = scipy.linalg.solve_triangular(Lg, store.blk[(h, g)].T, lower=True).T
        store.put(g, g, np.eye(len(Lg)))
        recs.append(Precondition(store.members[g].copy(), Lg))
    return recs


def skeletonize_separators(store, groups, eps, level=None, stats=None):
    """Stage 3: sequential ID + zeroing + elimination of ~I."""
    recs, ranks = [], []
    for t, g in enumerate(groups):
        nb = store.neighbours(g)
        k = len(store.members[g])
        M = np.vstack([store.get(h, g) for h in nb]) if nb else np.zeros((0, k))
        M = M[np.any(M != 0.0, axis=1)]
        idr = interpolative_decomposition(M, eps)
        sk, rd, T = idr.skeleton, idr.redundant, idr.interp
        ranks.append(len(sk))
        if len(rd) == 0:
            continue
        Agg = store.get(g, g)
        Arr = Agg[np.ix_(rd, rd)]
        Asr = Agg[np.ix_(sk, rd)]
        Ass = Agg[np.ix_(sk, sk)]
        Att = Arr - T.T @ Asr - Asr.T @ T + T.T @ Ass @ T
        Ast = Asr - Ass @ T
        try:
            Lt = cholesky(Att)
        except NotSpdError as e:
            raise NotSpdError(e.pivot, level, "skeletonize", t, stats) from None
        Xt = tri_solve(Lt, Ast.T)
        mem = store.members[g]
        recs.append(Skeletonize(mem[rd].copy(), mem[sk].copy(), T, Lt, Xt, t))
        Anew = Ass - Xt.T @ Xt
        store.put(g, g, np.zeros((k, k)))
        store.shrink(g, sk)
        store.put(g, g, Anew)
    return recs, ranks


def factorize(A, spec, eps: float, method: str = "phif") -> Factorization:
    """Oracle factorization (see module docstring). A: object with `.csr` or a scipy matrix."""
    method = method.lower()
    if method not in ("hif", "phif", "exact"):
        raise ValueError(f"unknown method {method!r}")
    if method == "exact":
        eps = 0.0
    csr = getattr(A, "csr", A).tocsr()
    dim, n, m = spec.dim, spec.n, spec.m
    Lmax = (n // m).bit_length() - 1
    N = csr.shape[0]
    active = np.arange(N, dtype=np.int64)
    levels, stats_levels = [], []
    stats = {"method": method, "eps": eps, "N": N, "levels": stats_levels}
    store = None
    for lev in range(Lmax + 1):
        part = classify_active(dim, n, m, lev, active)
        t0 = time.perf_counter()
        store = _store_from_csr(csr, part.groups, N) if lev == 0 else _regroup(store, part.groups, N)
        recs = LevelRecords(lev)
        st = {"level": lev, "S": int(len(active)), "p": part.p, "q": part.q, "r": part.r,
              "t_regroup": time.perf_counter() - t0}
        t0 = time.perf_counter()
        recs.eliminate = eliminate_cells(store, part.interior, lev, "root" if lev == Lmax else "eliminate", stats)
        st["t_eliminate"] = time.perf_counter() - t0
        if lev == Lmax:
            levels.append(recs)
            stats_levels.append(st)
            break
        t0 = time.perf_counter()
        if method != "hif":
            recs.precondition = precondition_blocks(store, part.precond, lev, stats)
        st["t_precondition"] = time.perf_counter() - t0
        t0 = time.perf_counter()
        recs.skeletonize, ranks = skeletonize_separators(store, part.skeleton, eps, lev, stats)
        st["t_skeletonize"] = time.perf_counter() - t0
        st["rho_max"] = int(max(ranks)) if ranks else 0
        st["rho_mean"] = float(np.mean(ranks)) if ranks else 0.0
        levels.append(recs)
        stats_levels.append(st)
        active = np.sort(np.concatenate([mm for mm in store.members if len(mm)]))
    root = levels[-1].eliminate[0].I if levels[-1].eliminate else np.zeros(0, np.int64)
    stats["SL"] = int(len(root))
    stats["mem_bytes"] = int(_record_bytes(levels))
    return Factorization(method, eps, N, Lmax, levels, root, stats)


def _record_bytes(levels):
    tot = 0
    for lv in levels:
        for r in lv.eliminate:
            tot += r.L.nbytes + r.X.nbytes
        for r in lv.precondition:
            tot += r.L.nbytes
        for r in lv.skeletonize:
            tot += r.T.nbytes + r.L.nbytes + r.X.nbytes
    return tot


# ---------------------------------------------------------------------------
# Record replay
# ---------------------------------------------------------------------------

def _solve_l(L, y, trans=False):
    if L.shape[0] == 0:
        return y
    return scipy.linalg.solve_triangular(L, y, lower=True, trans="T" if trans else "N")


def _up(F, x):
    """x <- R_{L-1}^T ... R_0^T x, then B_L^-1 on the root set (G^-1 x)."""
    for lv in F.levels:
        for r in lv.eliminate:
            y = _solve_l(r.L, x[r.I])
            if len(r.B):
                x[r.B] -= r.X.T @ y
            x[r.I] = y
        for r in lv.precondition:
            x[r.I] = _solve_l(r.L, x[r.I])
        for r in lv.skeletonize:
            if len(r.skeleton):
                x[r.redundant] -= r.T.T @ x[r.skeleton]
            y = _solve_l(r.L, x[r.redundant])
            if len(r.skeleton):
                x[r.skeleton] -= r.X.T @ y
            x[r.redundant] = y
    return x


def _down(F, x):
    """x <- R_0 ... R_{L-1} B_L^-T x (G^-T x)."""
    for lv in reversed(F.levels):
        for r in lv.skeletonize:
            t = x[r.redundant]
            if len(r.skeleton):
                t = t - r.X @ x[r.skeleton]
            x[r.redundant] = _solve_l(r.L, t, trans=True)
            if len(r.skeleton):
                x[r.skeleton] -= r.T @ x[r.redundant]
        for r in lv.precondition:
            x[r.I] = _solve_l(r.L, x[r.I], trans=True)
        for r in lv.eliminate:
            t = x[r.I]
            if len(r.B):
                t = t - r.X @ x[r.B]
            x[r.I] = _solve_l(r.L, t, trans=True)
    return x


def _as2d(b):
    b = np.asarray(b, dtype=np.float64)
    return (b.reshape(-1, 1).copy(), True) if b.ndim == 1 else (b.copy(), False)


def apply_inverse(F, b):
    """F^-1 b = G^-T G^-1 b (PAPER.md eq. eqAinv)."""
    x, flat = _as2d(b)
    x = _down(F, _up(F, x))
    return x[:, 0] if flat else x


def apply_ginv(F, b):
    x, flat = _as2d(b)
    x = _up(F, x)
    return x[:, 0] if flat else x


def apply_ginv_t(F, b):
    x, flat = _as2d(b)
    x = _down(F, x)
    return x[:, 0] if flat else x


def _gt(F, x):
    """x <- G^T x = B_L^T R_{L-1}^-1 ... R_0^-1 x."""
    for lv in F.levels:
        for r in lv.eliminate:
            xi = r.L.T @ x[r.I]
            if len(r.B):
                xi = xi + r.X @ x[r.B]
            x[r.I] = xi
        for r in lv.precondition:
            x[r.I] = r.L.T @ x[r.I]
        for r in lv.skeletonize:
            if len(r.skeleton):
                x[r.skeleton] += r.T @ x[r.redundant]
            xr = r.L.T @ x[r.redundant]
            if len(r.skeleton):
                xr = xr + r.X @ x[r.skeleton]
            x[r.redundant] = xr
    return x


def _g(F, x):
    """x <- G x = R_0^-T ... R_{L-1}^-T B_L x."""
    for lv in reversed(F.levels):
        for r in lv.skeletonize:
            if len(r.skeleton):
                x[r.skeleton] += r.X.T @ x[r.redundant]
            x[r.redundant] = r.L @ x[r.redundant]
            if len(r.skeleton):
                x[r.redundant] += r.T.T @ x[r.skeleton]
        for r in lv.precondition:
            x[r.I] = r.L @ x[r.I]
        for r in lv.eliminate:
            if len(r.B):
                x[r.B] += r.X.T @ x[r.I]
            x[r.I] = r.L @ x[r.I]
    return x


def apply(F, x):
    """F x = G G^T x (PAPER.md eq. eqA)."""
    y, flat = _as2d(x)
    y = _g(F, _gt(F, y))
    return y[:, 0] if flat else y


def root_condition(F):
    Lr = F.root_factor
    if Lr.shape[0] == 0:
        return 1.0
    s = np.linalg.svd(Lr, compute_uv=False)
    return float((s[0] / s[-1]) ** 2)
