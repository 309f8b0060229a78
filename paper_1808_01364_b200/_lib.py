"""ctypes binding of the C-ABI in include/phif_b200.h (the drop-in boundary).

Loads the in-tree `libphif_b200.so` (built by `__graft_entry__.build()` /
`csrc/build.sh`). There is no CPU fallback: if the library is missing or no
CUDA device is present, every compute call raises.
"""

from __future__ import annotations

import ctypes as C
import os

import numpy as np

_HERE = os.path.dirname(os.path.abspath(__file__))
LIB_PATH = os.path.join(_HERE, "libphif_b200.so")


class phif_error(C.Structure):
    _fields_ = [("code", C.c_int), ("pivot", C.c_int), ("level", C.c_int), ("stage", C.c_int),
                ("group", C.c_int), ("message", C.c_char * 512)]


OK, ERROR, NOT_SPD, BREAKDOWN = 0, 1, 2, 3
METHODS = {"hif": 0, "phif": 1, "exact": 2}
STAGES = {0: "eliminate", 1: "precondition", 2: "skeletonize", 3: "root"}

_lib = None

EXPORTS = ("phif_version", "phif_launch_count", "phif_matrix_create", "phif_matrix_free", "phif_matrix_from_field",
           "phif_matrix_csr", "phif_matrix_apply", "phif_factorize", "phif_factor_free",
           "phif_apply", "phif_pcg", "phif_solve_error", "phif_apply_error", "phif_root_factor", "phif_stats_json",
           "phif_skeleton_sets",
           "phif_num_levels", "phif_last_partial_stats", "phif_plan_check", "phif_classify", "phif_plan_dryrun")


def lib():
    """The loaded library (raises if the CUDA extension was not built)."""
    global _lib
    if _lib is not None:
        return _lib
    if not os.path.exists(LIB_PATH):
        raise RuntimeError(f"B200 engine not built: {LIB_PATH} missing (run __graft_entry__.build())")
    L = C.CDLL(LIB_PATH)
    P, D, I64, I = C.c_void_p, C.POINTER(C.c_double), C.c_int64, C.c_int
    L.phif_version.restype = I
    L.phif_launch_count.restype = C.c_longlong
    L.phif_matrix_create.argtypes = [P, P, P, I64, P, C.POINTER(P), C.POINTER(phif_error)]
    L.phif_matrix_create.restype = I
    L.phif_matrix_free.argtypes = [P]
    L.phif_matrix_from_field.argtypes = [I, I, P, P, I, C.c_double, C.c_double, C.c_double, P, C.POINTER(P),
                                         C.POINTER(phif_error)]
    L.phif_matrix_from_field.restype = I
    L.phif_matrix_csr.argtypes = [P, C.POINTER(C.c_int64), P, P, P, P]
    L.phif_matrix_csr.restype = I
    L.phif_matrix_apply.argtypes = [P, P, P, I, I, C.POINTER(phif_error)]
    L.phif_matrix_apply.restype = I
    L.phif_factorize.argtypes = [P, I, I, I, C.c_double, I, P, I, C.POINTER(P), C.POINTER(phif_error)]
    L.phif_factorize.restype = I
    L.phif_factor_free.argtypes = [P]
    L.phif_apply.argtypes = [P, P, I, I, C.POINTER(phif_error)]
    L.phif_apply.restype = I
    L.phif_pcg.argtypes = [P, P, P, P, I, C.c_double, I, P, P, P, P, P, C.POINTER(I), C.POINTER(phif_error)]
    L.phif_pcg.restype = I
    L.phif_solve_error.argtypes = [P, P, P, C.c_double, I, D, C.POINTER(I), C.POINTER(I), D,
                                   C.POINTER(phif_error)]
    L.phif_solve_error.restype = I
    L.phif_apply_error.argtypes = [P, P, P, C.c_double, I, D, C.POINTER(I), C.POINTER(I), D,
                                   C.POINTER(phif_error)]
    L.phif_apply_error.restype = I
    L.phif_root_factor.argtypes = [P, P, C.POINTER(I), C.POINTER(phif_error)]
    L.phif_root_factor.restype = I
    L.phif_stats_json.argtypes = [P, C.c_char_p, C.c_size_t]
    L.phif_stats_json.restype = C.c_size_t
    L.phif_skeleton_sets.argtypes = [P, I, P, P, P, P, P]
    L.phif_skeleton_sets.restype = I
    L.phif_num_levels.argtypes = [P]
    L.phif_num_levels.restype = I
    L.phif_last_partial_stats.argtypes = [C.c_char_p, C.c_size_t]
    L.phif_last_partial_stats.restype = C.c_size_t
    L.phif_plan_check.argtypes = [P, I, I, I, C.c_char_p, C.c_size_t]
    L.phif_plan_check.restype = I
    L.phif_classify.argtypes = [I, I, I, I, P, I64, P, P, I64]
    L.phif_classify.restype = I64
    L.phif_plan_dryrun.argtypes = [I, I, I, P, P, I, C.c_char_p, C.c_size_t]
    L.phif_plan_dryrun.restype = C.c_size_t
    _lib = L
    return L


def ptr(a: np.ndarray):
    return C.c_void_p(a.ctypes.data)


def last_partial_stats():
    """Statistics of the levels completed before the last NotSpd failure (None if unavailable)."""
    import json
    L = lib()
    n = L.phif_last_partial_stats(None, 0)
    if n == 0:
        return None
    buf = C.create_string_buffer(n + 1)
    L.phif_last_partial_stats(buf, n + 1)
    try:
        return json.loads(buf.value.decode())
    except ValueError:
        return None


def raise_for(rc: int, err: phif_error, partial_stats=None):
    from .errors import BreakdownError, NotSpdError
    if rc == OK:
        return
    if rc == NOT_SPD:
        if partial_stats is None:
            partial_stats = last_partial_stats()
        raise NotSpdError(err.pivot, err.level, STAGES.get(err.stage, err.stage), err.group, partial_stats)
    if rc == BREAKDOWN:
        raise BreakdownError(f"non-finite PCG recurrence value at iteration {err.group}")
    raise RuntimeError(f"phif engine error: {err.message.decode(errors='replace')}")
