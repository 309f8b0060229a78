"""classify_active through the B200 engine's C++ planner (hierarchy.py:102-156 semantics).

The planner groups active DOFs by level-l cell geometry: key (x-major cell index,
kind bits), members ascending. This wrapper exists so the grouping the engine uses
can be checked against the reference's own `classify_active` (tests/test_planner.py).
"""

from __future__ import annotations

from dataclasses import dataclass

import numpy as np

from . import _lib

KINDS = {2: ("interior", "edge", "corner"), 3: ("interior", "face", "edge", "corner")}


@dataclass
class DofGroup:
    kind: str
    level: int
    indices: np.ndarray


@dataclass
class LevelPartition:
    level: int
    interior_groups: list
    skeleton_groups: list
    precond_groups: list

    @property
    def p(self):
        return len(self.interior_groups)

    @property
    def q(self):
        return len(self.skeleton_groups)

    @property
    def r(self):
        return len(self.precond_groups)


def classify_active(spec, level, active) -> LevelPartition:
    act = np.ascontiguousarray(np.asarray(active, dtype=np.int32))
    gof = np.zeros(max(len(act), 1), dtype=np.int32)
    kinds = np.zeros(max(len(act), 1), dtype=np.int32)
    G = _lib.lib().phif_classify(spec.dim, spec.n, spec.m, level, _lib.ptr(act), len(act), _lib.ptr(gof),
                                 _lib.ptr(kinds), len(kinds))
    if G < 0:
        raise ValueError("classify failed (DOF outside the domain?)")
    order = np.argsort(gof[:len(act)], kind="stable")
    cuts = np.searchsorted(gof[:len(act)][order], np.arange(G + 1))
    names = KINDS[spec.dim]
    interior, skeleton, precond = [], [], []
    for g in range(G):
        mem = np.sort(act[order[cuts[g]:cuts[g + 1]]].astype(np.int64))
        kind = names[int(kinds[g])]
        grp = DofGroup(kind, level, mem)
        if kind == "interior":
            interior.append(grp)
        else:
            precond.append(grp)
            if int(kinds[g]) == 1:
                skeleton.append(grp)
    return LevelPartition(level, interior, skeleton, precond)
