"""Exception types, mirroring ``pathfield/errors.py:1-37``.

Argument validation happens in Python before any launch so the exception
types raised by the device path are the reference's.  When the reference
package ``pathfield`` is importable (drop-in mode) its
own classes are re-exported, so ``pytest.raises(pathfield.errors.X)`` in the
reference's tests catches errors raised here.
"""

from __future__ import annotations

try:  # drop-in mode: share the reference's exception classes
    from pathfield.errors import (BudgetExceededError, ConfigError,  # type: ignore
                                  DegenerateGeometryError,
                                  DivergenceDomainError, FactorizationError,
                                  InvalidTargetError, MeshFormatError,
                                  MeshTopologyError, PathfieldError)
except Exception:  # standalone: same hierarchy, same names
    class PathfieldError(Exception):
        """Base class for all errors raised by this package."""

    class MeshFormatError(PathfieldError):
        """A mesh file could not be parsed."""

    class MeshTopologyError(PathfieldError):
        """The triangulation is not a valid manifold planar mesh."""

    class DegenerateGeometryError(PathfieldError):
        """A triangle has (numerically) zero area or a 0/pi angle."""

    class FactorizationError(PathfieldError):
        """The interior Laplacian block could not be factorized."""

    class InvalidTargetError(PathfieldError):
        """The requested source/target vertex is not admissible."""

    class BudgetExceededError(PathfieldError):
        """The mesh is too large for a dense pseudo-inverse computation."""

    class DivergenceDomainError(PathfieldError):
        """A divergence hit a zero denominator and clamping is disabled."""

    class ConfigError(PathfieldError):
        """A configuration file or value is invalid."""


class NativeError(PathfieldError):
    """A call into libpathfield_b200.so returned a non-zero status."""

    def __init__(self, code: int, message: str):
        super().__init__(f"[{code}] {message}")
        self.code = code


__all__ = [
    "PathfieldError", "MeshFormatError", "MeshTopologyError",
    "DegenerateGeometryError", "FactorizationError", "InvalidTargetError",
    "BudgetExceededError", "DivergenceDomainError", "ConfigError", "NativeError",
]
