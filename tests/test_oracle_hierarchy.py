"""Oracle classify_active vs golden outputs of the reference's hierarchy.py."""
import numpy as np

from oracle.hierarchy import classify_active


def _split(flat, sizes):
    out, a = [], 0
    for s in sizes:
        out.append(flat[a:a + s])
        a += s
    return out


def test_classify_golden(golden):
    for i in range(int(golden["cls_count"])):
        dim, n, m, lev = (int(v) for v in golden[f"cls_{i}_spec"])
        part = classify_active(dim, n, m, lev, golden[f"cls_{i}_active"])
        for name, idx in (("interior", part.interior), ("precond", part.precond), ("skeleton", part.skeleton)):
            ref = _split(golden[f"cls_{i}_{name}"], golden[f"cls_{i}_{name}_sizes"])
            got = [part.groups[j].indices for j in idx]
            assert len(ref) == len(got), (i, name)
            assert all(np.array_equal(a, b) for a, b in zip(ref, got)), (i, name)
