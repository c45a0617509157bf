"""Data contracts of the hot path, mirroring ``pathfield/solvers.py``.

* :class:`ScalarField` (``solvers.py:47-65``) — the output of every field
  function: read-only ``values``, ``kind``, ``target``, ``params``, ``sign``,
  ``residual``, ``precision_flags``.
* :class:`PoissonKernel` (``solvers.py:229-275``) — the input: ``dense``
  (n x k row-stochastic FP64, read-only), sorted ``boundary`` columns, and
  the optional sparse/log views that :func:`sparsify` adds.

Both accept duck-typed reference objects everywhere they are consumed; the
device path only reads attributes.
"""

from __future__ import annotations

from dataclasses import dataclass, field as dc_field

import numpy as np

from .errors import InvalidTargetError

try:  # drop-in mode: the reference's warning class (solvers.py:43-44)
    from pathfield.solvers import PrecisionWarning  # type: ignore
except Exception:
    class PrecisionWarning(UserWarning):
        """A numerical result is less accurate than requested (solvers.py:43)."""


@dataclass(frozen=True)
class ScalarField:
    """Per-vertex distance-like values with the target as global minimum."""

    values: np.ndarray
    kind: str
    target: int
    params: dict = dc_field(default_factory=dict)
    sign: int = 1
    residual: float | None = None
    precision_flags: tuple[str, ...] = ()

    def __post_init__(self):
        self.values.setflags(write=False)

    @property
    def raw(self) -> np.ndarray:
        return self.sign * self.values


@dataclass(frozen=True, eq=False)
class PoissonKernel:
    """Row-stochastic matrix of boundary harmonic measures (n x k, FP64).

    ``sparse`` is a CSR view ``(data, indices, indptr)``-compatible object
    (scipy ``csr_matrix`` when scipy built it, or :class:`CsrView` when the
    device built it); ``log_sparse`` the logs of its data with the same
    pattern; ``log_dense`` the logs of every clamped entry.
    """

    dense: np.ndarray
    boundary: np.ndarray
    residual: float
    row_sum_error: float
    threshold: float | None = None
    sparse: object | None = None
    log_sparse: object | None = None
    log_dense: np.ndarray | None = None
    dropped_mass: np.ndarray | None = None
    row_cut: float | None = None
    sparsity_percent: float | None = None

    def __post_init__(self):
        self.dense.setflags(write=False)

    @property
    def n(self) -> int:
        return self.dense.shape[0]

    @property
    def k(self) -> int:
        return self.dense.shape[1]

    def column_of(self, vertex: int) -> int:
        c = int(np.searchsorted(self.boundary, vertex))
        if c >= self.k or self.boundary[c] != vertex:
            raise InvalidTargetError(f"vertex {vertex} is not a boundary vertex")
        return c

    def sparsity_report(self) -> dict:
        return {
            "threshold": self.threshold,
            "sparsity_percent": self.sparsity_percent,
            "max_dropped_row_mass": (
                float(self.dropped_mass.max()) if self.dropped_mass is not None else None
            ),
        }


@dataclass(frozen=True, eq=False)
class CsrView:
    """Minimal CSR container with scipy's attribute names.

    Produced by the device ``sparsify`` (the pattern is bit-identical to
    ``scipy.sparse.csr_matrix`` + ``eliminate_zeros``, divergence.py:220-223).
    ``tocsr()`` converts to scipy when scipy is present.
    """

    data: np.ndarray
    indices: np.ndarray
    indptr: np.ndarray
    shape: tuple

    @property
    def nnz(self) -> int:
        return int(self.indptr[-1])

    def tocsr(self):
        import scipy.sparse as sp
        return sp.csr_matrix((self.data, self.indices, self.indptr), shape=self.shape)

    def toarray(self) -> np.ndarray:
        out = np.zeros(self.shape)
        rows = np.repeat(np.arange(self.shape[0]), np.diff(self.indptr))
        out[rows, self.indices] = self.data
        return out

    def sum(self, axis=None):
        if axis == 1:
            return np.add.reduceat(self.data, self.indptr[:-1]) * (np.diff(self.indptr) > 0)
        return float(self.data.sum())
