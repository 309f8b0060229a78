"""Oracle-side exception types (TEST INFRASTRUCTURE ONLY).

Same classes and fields as the reference's errors.py:4-42; kept separate from
the product package so the oracle never imports product code.
"""


class NotSpdError(ArithmeticError):
    def __init__(self, pivot, level=None, stage=None, group=None, partial_stats=None):
        self.pivot = pivot
        self.level = level
        self.stage = stage
        self.group = group
        self.partial_stats = partial_stats
        msg = f"matrix not positive definite at pivot {pivot}"
        if level is not None:
            msg += f" (level {level}, stage {stage}, group {group})"
        super().__init__(msg)


class BreakdownError(ArithmeticError):
    pass


class EstimationError(RuntimeError):
    def __init__(self, message, partial=None):
        self.partial = partial
        super().__init__(message)
