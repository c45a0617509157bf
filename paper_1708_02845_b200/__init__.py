"""B200-native divergence-distance hot path of arXiv 1708.02845 (reference: ``pathfield``).

Drop-in mirror of the reference package's hot-path API
(``pathfield/__init__.py:4-17``): the same names, signatures and return
types, computed by hand-written sm_100a CUDA kernels behind the C ABI in
``include/pathfield_b200.h``.  There is no CPU fallback.
"""

from .config import DEFAULTS, Settings
from .divergence import (FDivergence, builtin_f, dv_at, dv_field, dv_field_batch,
                         dv_field_device, dv_field_sparse, dv_pair,
                         dv_pair_sparse, dv_pair_sparse_stats, sparsify)
from .mesh import TriMesh
from .paths import (TracedPath, edge_descent, edge_descent_batch, find_local_minima,
                    path_hausdorff, path_hausdorff_batch, resample_polyline,
                    triangle_descent, triangle_descent_batch, triangle_gradient)
from .errors import (DivergenceDomainError, InvalidTargetError, NativeError,
                     PathfieldError)
from .solvers import PoissonKernel, ScalarField

__version__ = "0.1.0"

__all__ = [
    "DEFAULTS", "Settings", "FDivergence", "builtin_f", "dv_at", "dv_field", "dv_field_batch",
    "dv_field_device", "dv_pair", "sparsify", "dv_pair_sparse", "dv_pair_sparse_stats",
    "dv_field_sparse", "TriMesh", "TracedPath", "triangle_descent", "triangle_descent_batch",
    "triangle_gradient", "edge_descent", "edge_descent_batch", "find_local_minima",
    "path_hausdorff", "path_hausdorff_batch", "resample_polyline",
    "DivergenceDomainError", "InvalidTargetError",
    "NativeError", "PathfieldError", "PoissonKernel", "ScalarField",
]
