"""Error types of the host API (mirror of pipepath/errors.py:1-21).

``ValidationError`` is a ``ValueError`` that appends the offending matrix coordinates to its
message (errors.py:10-17); ``InfeasibleError`` is a ``RuntimeError`` raised when no
schedule or path satisfies the constraints.  The CLI maps them to exit codes 1 and 2
(SPEC.md:511).
"""

from __future__ import annotations


class ValidationError(ValueError):
    """Malformed input: bad matrix, inconsistent sizes, out-of-range ids."""

    def __init__(self, message, row=None, col=None):
        where = []
        if row is not None:
            where.append(f"row {row}")
            if col is not None:
                where.append(f"col {col}")
        if where:
            message = f"{message} ({', '.join(where)})"
        super().__init__(message)
        self.row = row
        self.col = col


class InfeasibleError(RuntimeError):
    """No schedule / path exists under the given constraints."""
