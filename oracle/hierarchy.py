"""Level grouping of active DOFs (restates reference hierarchy.py:80-168).

TEST INFRASTRUCTURE ONLY (see oracle/__init__.py).

Level l tiles the grid with cells of side s = 2^l m. A DOF's lattice coords
(x fastest, grid.py:67-80) give q = coords // s and on_line = coords % s == 0;
the group key is (q_x, q_y[, q_z], bits) with bits = sum(on_line_d << d),
ordered x-major with the kind bits last (hierarchy.py:124-133); members are
ascending global ids (hierarchy.py:145). Kind = number of on-line axes:
2D {0 interior, 1 edge, 2 corner}; 3D {0 interior, 1 face, 2 edge, 3 corner}.
Interior groups are eliminated, every other group is preconditioned, and
edges (2D) / faces (3D) are skeletonized (hierarchy.py:150-155).
"""

from __future__ import annotations

from dataclasses import dataclass, field

import numpy as np

KINDS = {2: ("interior", "edge", "corner"), 3: ("interior", "face", "edge", "corner")}


@dataclass
class Group:
    kind: str
    level: int
    indices: np.ndarray
    owner: tuple
    key: tuple


@dataclass
class Partition:
    level: int
    groups: list = field(default_factory=list)      # all groups, key order
    interior: list = field(default_factory=list)    # indices into groups
    precond: list = field(default_factory=list)
    skeleton: list = field(default_factory=list)

    @property
    def p(self):
        return len(self.interior)

    @property
    def q(self):
        return len(self.skeleton)

    @property
    def r(self):
        return len(self.precond)


def lattice_coords(dim, n, ids):
    ids = np.asarray(ids, dtype=np.int64)
    side = n - 1
    return np.stack([(ids // side ** d) % side + 1 for d in range(dim)], axis=-1)


def _owner(kind, dim, q, bits):
    if kind in ("interior", "corner"):
        return (kind, tuple(int(v) for v in q))
    axes = tuple(d for d in range(dim) if bits >> d & 1)
    free = tuple(d for d in range(dim) if not bits >> d & 1)
    return (kind, axes, tuple(int(q[d]) for d in axes), tuple(int(q[d]) for d in free))


def classify_active(dim, n, m, level, active) -> Partition:
    active = np.asarray(active, dtype=np.int64)
    part = Partition(level)
    if active.size == 0:
        return part
    s = m << level
    per = n // s
    xyz = lattice_coords(dim, n, active)
    if xyz.min() < 1 or xyz.max() > n - 1:
        raise ValueError("active DOF outside the domain")
    q = xyz // s
    bits = ((xyz % s == 0).astype(np.int64) << np.arange(dim)).sum(axis=1)
    key = np.zeros(len(active), dtype=np.int64)
    for d in range(dim):
        key = key * per + q[:, d]
    key = key * (1 << dim) + bits
    order = np.argsort(key, kind="stable")
    skey = key[order]
    cuts = np.flatnonzero(np.diff(skey)) + 1
    starts = np.concatenate([[0], cuts])
    ends = np.concatenate([cuts, [len(skey)]])
    names = KINDS[dim]
    sep = "edge" if dim == 2 else "face"
    for a, b in zip(starts, ends):
        first = order[a]
        bb = int(bits[first])
        kind = names[bin(bb).count("1")]
        g = Group(kind, level, np.sort(active[order[a:b]]),
                  _owner(kind, dim, q[first], bb), tuple(int(v) for v in q[first]) + (bb,))
        idx = len(part.groups)
        part.groups.append(g)
        if kind == "interior":
            part.interior.append(idx)
        else:
            part.precond.append(idx)
            if kind == sep:
                part.skeleton.append(idx)
    return part
