"""Exception taxonomy mirrored from the reference (errors.py:8-37) for the
parts the hot path can raise."""


class FilterError(Exception):
    """Base class for numerical/design failures (errors.py:8)."""


class StabilityError(FilterError):
    """A recursion was asked to run with poles on or outside the unit circle
    (errors.py:32)."""
