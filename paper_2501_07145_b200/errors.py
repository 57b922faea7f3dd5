"""Exception types raised at the boundary (reference: sigkern/errors.py:4-27).

The host layer re-raises the reference's exception classes with the
reference's messages, so callers' `except` clauses and the reference tests'
`match=` strings keep working.
"""


class SigkernError(Exception):
    """Base class for errors raised by this package (errors.py:4)."""


class ConfigError(SigkernError, ValueError):
    """Invalid run configuration (errors.py:18)."""


class NumericError(SigkernError, ArithmeticError):
    """Numerically degenerate computation (errors.py:22)."""


class NativeError(SigkernError, RuntimeError):
    """The CUDA library reported a failure (launch error, workspace, ...)."""


class ParseError(SigkernError, ValueError):
    """Malformed input file (errors.py:8-15): the text is prefixed with
    "line N: " and `.line` holds N when the offending line is known."""

    def __init__(self, message, line=None):
        self.line = line
        super().__init__(message if line is None else "line %d: %s" % (line, message))
