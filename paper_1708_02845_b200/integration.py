"""Drop-in routing of the reference package ``pathfield`` to the B200 path.

``install()`` rebinds the reference's hot-path functions at every binding
site listed in SURVEY §8b (the names are imported with ``from ... import``,
so each site is patched explicitly):

    pathfield.divergence.{dv_field, dv_at, dv_pair, sparsify,
                          dv_pair_sparse, dv_pair_sparse_stats}
    pathfield.{dv_field, dv_pair, dv_pair_sparse, sparsify,
               triangle_descent, triangle_gradient}          (__init__.py:4-13)
    pathfield.domain.{dv_field, sparsify, triangle_descent}  (domain.py:17-22)
    pathfield.bench.{dv_at, dv_field, dv_pair_sparse_stats}  (bench.py:25)
    pathfield.paths.{triangle_descent, triangle_gradient, edge_descent,
                     find_local_minima, path_hausdorff, resample_polyline}
    (domain.py also binds edge_descent, find_local_minima, path_hausdorff)
    pathfield.fileio.{field_to_csv, field_to_json, path_to_csv}   (fileio.py:37-75)
    pathfield.service.app.field_to_csv                            (app.py:18, 114)
    pathfield.{solvers, domain, bench, ""}.poisson_kernel         (solvers.py:278-303;
        DomainContext.kernel, domain.py:54-61, builds P on the GPU and keeps it resident)

Results are converted to the reference's own dataclasses (``ScalarField``,
``TracedPath``), and the reference's ``PoissonKernel`` objects are accepted
as-is (the device cache keys on ``pk.dense``), so ``DomainContext``, the
service and the CLI run unchanged on the GPU.  Exceptions keep the
reference's types: ``errors.py`` re-exports ``pathfield.errors`` whenever the
reference is importable, and argument validation precedes every launch.

Call ``install()`` before importing modules that bind these names with
``from pathfield... import`` (e.g. from a pytest plugin or a conftest), as
the SURVEY's patch-point list notes.
"""

from __future__ import annotations

import importlib

from . import divergence as _div
from . import fileio as _fileio
from . import paths as _paths

_ORIGINAL: dict = {}


def _ref_types(pathfield):
    solvers = importlib.import_module(pathfield.__name__ + ".solvers")
    paths = importlib.import_module(pathfield.__name__ + ".paths")
    return solvers.ScalarField, paths.TracedPath


def _wrap(pathfield):
    from .config import DEFAULTS as DEFAULTS_
    RefField, RefPath = _ref_types(pathfield)

    def to_field(f):
        return RefField(f.values, f.kind, f.target, f.params, f.sign, f.residual,
                        f.precision_flags)

    def to_path(p):
        return RefPath(p.points, p.locations, p.source, p.target, p.status, p.stuck_vertex)

    def dv_field(pk, fd, p, swap_order=False, clamp=None):
        return to_field(_div.dv_field(pk, fd, p, swap_order=swap_order, clamp=clamp))

    solvers = importlib.import_module(pathfield.__name__ + ".solvers")

    def poisson_kernel(ls, settings=None):
        from . import laplacian as _lap
        return _lap.poisson_kernel(ls, settings, kernel_type=solvers.PoissonKernel)

    def triangle_descent(mesh, field, source, settings=None):
        from .config import DEFAULTS
        return to_path(_paths.triangle_descent(mesh, field, source, settings or DEFAULTS))

    return {
        "dv_field": dv_field,
        "dv_at": _div.dv_at,
        "dv_pair": _div.dv_pair,
        "sparsify": _div.sparsify,
        "dv_pair_sparse": _div.dv_pair_sparse,
        "dv_pair_sparse_stats": _div.dv_pair_sparse_stats,
        "triangle_descent": triangle_descent,
        "triangle_gradient": _paths.triangle_gradient,
        "edge_descent": lambda mesh, field, source, settings=None: to_path(
            _paths.edge_descent(mesh, field, source, settings or DEFAULTS_)),
        "find_local_minima": _paths.find_local_minima,
        "path_hausdorff": _paths.path_hausdorff,
        "resample_polyline": _paths.resample_polyline,
        "field_to_csv": _fileio.field_to_csv,
        "field_to_json": _fileio.field_to_json,
        "path_to_csv": _fileio.path_to_csv,
        "poisson_kernel": poisson_kernel,
    }


SITES = {
    "divergence": ("dv_field", "dv_at", "dv_pair", "sparsify", "dv_pair_sparse",
                   "dv_pair_sparse_stats"),
    "": ("dv_field", "dv_pair", "dv_pair_sparse", "sparsify", "triangle_descent",
         "triangle_gradient", "edge_descent", "find_local_minima", "path_hausdorff",
         "poisson_kernel"),
    "domain": ("dv_field", "sparsify", "triangle_descent", "edge_descent", "find_local_minima",
               "path_hausdorff", "poisson_kernel"),
    "bench": ("dv_at", "dv_field", "dv_pair_sparse_stats", "poisson_kernel"),
    "solvers": ("poisson_kernel",),
    "paths": ("triangle_descent", "triangle_gradient", "edge_descent", "find_local_minima",
              "path_hausdorff", "resample_polyline"),
    "fileio": ("field_to_csv", "field_to_json", "path_to_csv"),
    "service.app": ("field_to_csv",),
}


def install(pathfield=None) -> dict:
    """Patch the reference's binding sites; returns {site: [names]} patched."""
    if pathfield is None:
        pathfield = importlib.import_module("pathfield")
    repl = _wrap(pathfield)
    done = {}
    for sub, names in SITES.items():
        try:
            mod = importlib.import_module(pathfield.__name__ + ("." + sub if sub else ""))
        except Exception:  # e.g. bench needs jsonschema; skip what cannot import
            continue
        for name in names:
            if hasattr(mod, name):
                _ORIGINAL.setdefault((mod.__name__, name), getattr(mod, name))
                setattr(mod, name, repl[name])
                done.setdefault(mod.__name__, []).append(name)
    return done


def uninstall() -> None:
    """Restore every binding ``install`` replaced."""
    for (modname, name), fn in list(_ORIGINAL.items()):
        setattr(importlib.import_module(modname), name, fn)
    _ORIGINAL.clear()
