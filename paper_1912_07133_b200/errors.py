"""Exception taxonomy mirrored from the reference (errors.py:8-37) for the
parts the hot path can raise."""


class FilterError(Exception):
    """Base class for numerical/design failures (errors.py:8)."""


class StabilityError(FilterError):
    """A recursion was asked to run with poles on or outside the unit circle
    (errors.py:32)."""


class SplitError(FilterError):
    """A denominator cannot be split into forward/backward factors: a root
    within tolerance of the unit circle, or a non-mirrored root set
    (errors.py:16)."""


class DecompositionError(FilterError):
    """The three-part numerator system is singular or inconsistent
    (errors.py:24)."""


class DesignError(FilterError):
    """A filter design's constraint system is unsolvable or ill-conditioned
    (errors.py:28)."""
