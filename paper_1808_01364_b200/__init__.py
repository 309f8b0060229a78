"""B200-native PHIF (arXiv 1808.01364): factorize / apply-inverse / PCG on sm_100a.

Drop-in for the reference's hot-path entry points (reference
package `hifsolve`): the same names, argument meaning and error types, backed by
the C-ABI library libphif_b200.so (C++ level planner + batched FP64 CUDA kernels).
"""

from .errors import (BreakdownError, ConfigurationError, ConsistencyError, EstimationError,  # noqa: F401
                     NotSpdError)
from .grid import (CONFIGS, CoefficientField, GridSpec, SymSparseMatrix, assemble_operator,  # noqa: F401
                   baseline_field, baseline_problem, baseline_rhs, generate_field)

__all__ = ["GridSpec", "SymSparseMatrix", "CoefficientField", "generate_field", "assemble_operator",
           "factorize", "apply_inverse", "apply_ginv", "apply_ginv_t", "apply", "root_condition", "pcg", "power_norm",
           "estimate_solve_error", "estimate_apply_error", "NotSpdError", "ConfigurationError", "BreakdownError", "EstimationError"]


def __getattr__(name):
    # lazy: importing the package must not require the CUDA library (CPU tests)
    if name in ("factorize", "apply_inverse", "apply_ginv", "apply_ginv_t", "apply", "root_condition", "Factorization"):
        from . import factorization
        return getattr(factorization, name)
    if name in ("pcg", "SolveReport"):
        from . import krylov
        return getattr(krylov, name)
    if name in ("power_norm", "estimate_solve_error", "estimate_apply_error", "NormEstimate"):
        from . import diagnostics
        return getattr(diagnostics, name)
    raise AttributeError(name)
