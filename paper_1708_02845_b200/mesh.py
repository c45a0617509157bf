"""Mesh input contract of the tracer and its device form.

* :class:`TriMesh` mirrors the parts of ``pathfield/mesh.py:23-172`` the hot
  path reads — CCW normalisation, |signed area| per triangle, boundary /
  interior classification, sorted ``neighbors`` and ``vertex_triangles``,
  ``edge_adjacency`` and ``bbox_diagonal`` — with the same array semantics
  (so the tracer is bit-identical whichever object it is given).  A reference
  ``pathfield.TriMesh`` is accepted everywhere in its place.
* :class:`DeviceMesh` flattens any such mesh into the device CSR topology of
  ``pf_mesh_t`` (include/pathfield_b200.h), cached per mesh.
"""

from __future__ import annotations

import ctypes
import threading
import weakref

import numpy as np

from . import _device as dev
from . import _native as nat
from .errors import DegenerateGeometryError, MeshFormatError, MeshTopologyError

_AREA_EPS = 1e-14  # mesh.py:20


def _signed_areas(v, t):
    # mesh.py:244-247
    p0, p1, p2 = v[t[:, 0]], v[t[:, 1]], v[t[:, 2]]
    u, w = p1 - p0, p2 - p0
    return 0.5 * (u[:, 0] * w[:, 1] - u[:, 1] * w[:, 0])


def topology(triangles: np.ndarray, n: int):
    """Vectorised (vt_ptr, vt_idx, nb_ptr, nb_idx, tri_nbr) — ascending lists as in
    mesh.py:113-157 (vertex_triangles, neighbors, edge_adjacency)."""
    t = np.asarray(triangles, dtype=np.int64)
    nt = len(t)
    v = t.ravel()
    tid = np.repeat(np.arange(nt, dtype=np.int64), 3)
    order = np.lexsort((tid, v))
    vt_idx = tid[order]
    vt_ptr = np.zeros(n + 1, dtype=np.int64)
    np.cumsum(np.bincount(v, minlength=n), out=vt_ptr[1:])
    e = np.concatenate([t[:, [0, 1]], t[:, [1, 2]], t[:, [2, 0]]])
    e = np.concatenate([e, e[:, ::-1]])
    key = np.unique(e[:, 0] * n + e[:, 1])
    src = key // n
    nb_idx = key % n
    nb_ptr = np.zeros(n + 1, dtype=np.int64)
    np.cumsum(np.bincount(src, minlength=n), out=nb_ptr[1:])
    slot = np.tile(np.arange(3), nt)
    i = t[tid, (slot + 1) % 3]
    j = t[tid, (slot + 2) % 3]
    k = np.minimum(i, j) * n + np.maximum(i, j)
    o = np.argsort(k, kind="stable")
    ks = k[o]
    cnt = np.diff(np.concatenate([[0], np.flatnonzero(ks[1:] != ks[:-1]) + 1, [len(ks)]]))
    if cnt.size and cnt.max() > 2:
        raise MeshTopologyError("non-manifold edge with more than 2 triangles")
    tri_nbr = -np.ones((nt, 3), dtype=np.int64)
    same = np.flatnonzero(ks[1:] == ks[:-1])
    a, b = o[same], o[same + 1]
    tri_nbr[tid[a], slot[a]] = tid[b]
    tri_nbr[tid[b], slot[b]] = tid[a]
    return vt_ptr, vt_idx, nb_ptr, nb_idx, tri_nbr


class TriMesh:
    """Planar triangle mesh (mirror of mesh.py:23-172 for the hot path)."""

    def __init__(self, vertices, triangles):
        v = np.ascontiguousarray(np.asarray(vertices, dtype=float))
        t = np.ascontiguousarray(np.asarray(triangles, dtype=np.int64)).copy()
        if v.ndim != 2 or v.shape[1] != 2:
            raise MeshFormatError(f"vertices must be (n, 2), got {v.shape}")
        if t.ndim != 2 or t.shape[1] != 3:
            raise MeshFormatError(f"triangles must be (nt, 3), got {t.shape}")
        if t.shape[0] < 1:
            raise MeshFormatError("mesh needs at least one triangle")
        if t.min() < 0 or t.max() >= len(v):
            raise MeshFormatError("triangle index out of range")
        self.vertices = v
        scale2 = max(np.ptp(v, axis=0).max() ** 2, 1e-30)
        signed = _signed_areas(v, t)
        flip = signed < 0
        t[flip] = t[flip][:, ::-1]
        signed = np.abs(signed)
        if np.any(signed <= _AREA_EPS * scale2):
            bad = int(np.argmin(signed))
            raise DegenerateGeometryError(f"triangle {bad} has (near) zero area {signed[bad]:.3e}")
        self.triangles = t
        self.triangle_areas = signed
        self._topo = topology(t, len(v))
        tri_nbr = self._topo[4]
        bmask = np.zeros(len(v), dtype=bool)
        tid, slot = np.nonzero(tri_nbr < 0)
        bmask[t[tid, (slot + 1) % 3]] = True
        bmask[t[tid, (slot + 2) % 3]] = True
        if not bmask.any():
            raise MeshTopologyError("mesh has no boundary (closed surface?)")
        self.is_boundary = bmask
        self.boundary_vertices = np.flatnonzero(bmask)
        self.interior_vertices = np.flatnonzero(~bmask)
        for arr in (self.vertices, self.triangles, self.triangle_areas,
                    self.boundary_vertices, self.interior_vertices):
            arr.setflags(write=False)

    @property
    def n(self) -> int:
        return len(self.vertices)

    @property
    def k(self) -> int:
        return len(self.boundary_vertices)

    @property
    def m(self) -> int:
        return len(self.interior_vertices)

    @property
    def bbox(self):
        return self.vertices.min(axis=0), self.vertices.max(axis=0)

    @property
    def bbox_diagonal(self) -> float:
        lo, hi = self.bbox
        return float(np.hypot(*(hi - lo)))

    @property
    def neighbors(self):
        vp, _, nbp, nbi, _ = self._topo
        return [nbi[nbp[i]:nbp[i + 1]] for i in range(self.n)]

    @property
    def vertex_triangles(self):
        vp, vi = self._topo[0], self._topo[1]
        return [vi[vp[i]:vp[i + 1]] for i in range(self.n)]

    @property
    def edge_adjacency(self):
        t, tri_nbr = self.triangles, self._topo[4]
        out = {}
        for ti in range(len(t)):
            for s in range(3):
                i, j = int(t[ti, (s + 1) % 3]), int(t[ti, (s + 2) % 3])
                key = (min(i, j), max(i, j))
                if key not in out:
                    o = int(tri_nbr[ti, s])
                    out[key] = (ti,) if o < 0 else tuple(sorted((ti, o)))
        return out

    def edge_lengths(self) -> np.ndarray:
        vp, _, nbp, nbi, _ = self._topo
        src = np.repeat(np.arange(self.n), np.diff(nbp))
        keep = src < nbi
        d = self.vertices[src[keep]] - self.vertices[nbi[keep]]
        return np.hypot(d[:, 0], d[:, 1])

    def mean_edge_length(self) -> float:
        return float(self.edge_lengths().mean())

    def min_edge_length(self) -> float:
        return float(self.edge_lengths().min())


def grid_mesh(nx: int, ny: int, lx: float = 1.0, ly: float = 1.0) -> TriMesh:
    """Structured (nx+1) x (ny+1) vertex grid on [0,lx]x[0,ly], each cell split
    along its diagonal: a synthetic benchmark mesh of any size (no Delaunay)."""
    xs = np.linspace(0.0, lx, nx + 1)
    ys = np.linspace(0.0, ly, ny + 1)
    X, Y = np.meshgrid(xs, ys)
    V = np.column_stack([X.ravel(), Y.ravel()])
    i, j = np.meshgrid(np.arange(nx), np.arange(ny))
    a = (j * (nx + 1) + i).ravel()
    b, c, d = a + 1, a + nx + 2, a + nx + 1
    T = np.concatenate([np.column_stack([a, b, c]), np.column_stack([a, c, d])])
    return TriMesh(V, T)


# --------------------------------------------------------------- device --
class PfMesh(ctypes.Structure):
    _fields_ = [("vertices", ctypes.c_void_p), ("triangles", ctypes.c_void_p),
                ("areas", ctypes.c_void_p), ("tri_nbr", ctypes.c_void_p),
                ("vt_ptr", ctypes.c_void_p), ("vt_idx", ctypes.c_void_p),
                ("nb_ptr", ctypes.c_void_p), ("nb_idx", ctypes.c_void_p),
                ("n", ctypes.c_int64), ("nt", ctypes.c_int64), ("eps_prog", ctypes.c_double),
                ("G", ctypes.c_void_p), ("pack", ctypes.c_void_p)]


class DeviceMesh:
    """pf_mesh_t arrays in HBM (vertices FP64, triangles/topology int32/int64)."""

    def __init__(self, mesh, device=None):
        t = dev.require_cuda()
        self.device = (t.device(device) if device is not None
                       else t.device("cuda", t.cuda.current_device()))
        V = np.ascontiguousarray(mesh.vertices, dtype=np.float64)
        T = np.ascontiguousarray(mesh.triangles, dtype=np.int64)
        topo = getattr(mesh, "_topo", None) or topology(T, len(V))
        vt_ptr, vt_idx, nb_ptr, nb_idx, tri_nbr = topo
        to = lambda a, dt: t.from_numpy(np.array(a, dtype=dt)).to(self.device)  # noqa: E731
        self.V = to(V, np.float64)
        self.T = to(T, np.int32)
        self.A = to(np.asarray(mesh.triangle_areas), np.float64)
        self.tri_nbr = to(tri_nbr, np.int32)
        self.vt_ptr = to(vt_ptr, np.int64)
        self.vt_idx = to(vt_idx, np.int32)
        self.nb_ptr = to(nb_ptr, np.int64)
        self.nb_idx = to(nb_idx, np.int32)
        self.n, self.nt = len(V), len(T)
        # paths.py:143: eps_prog = 1e-14 * mesh.bbox_diagonal (host property of the mesh)
        self.eps_prog = 1e-14 * float(mesh.bbox_diagonal)
        self.struct = PfMesh(self.V.data_ptr(), self.T.data_ptr(), self.A.data_ptr(),
                             self.tri_nbr.data_ptr(), self.vt_ptr.data_ptr(),
                             self.vt_idx.data_ptr(), self.nb_ptr.data_ptr(),
                             self.nb_idx.data_ptr(), self.n, self.nt, self.eps_prog, None,
                             None)
        # per-triangle barycentric gradients, computed once on the device with
        # the tracer's own arithmetic (bitwise what it would recompute per visit)
        self.G = t.empty((self.nt, 6), dtype=t.float64, device=self.device)
        nat.call("pf_mesh_geometry_f64", ctypes.addressof(self.struct), self.G.data_ptr(),
                 t.cuda.current_stream(self.device).cuda_stream)
        self.struct.G = self.G.data_ptr()
        # packed 128-byte triangle records: one round trip per tracer step
        self.pack = t.empty((self.nt, 16), dtype=t.float64, device=self.device)
        nat.call("pf_mesh_pack_f64", ctypes.addressof(self.struct), self.pack.data_ptr(),
                 t.cuda.current_stream(self.device).cuda_stream)
        self.struct.pack = self.pack.data_ptr()


_cache: dict[int, tuple[weakref.ref, DeviceMesh]] = {}
_lock = threading.Lock()


def device_mesh(mesh) -> DeviceMesh:
    """Device topology of `mesh`, built once and cached while the mesh lives."""
    key = id(mesh.triangles)
    with _lock:
        hit = _cache.get(key)
        if hit is not None and hit[0]() is mesh.triangles:
            return hit[1]
    dm = DeviceMesh(mesh)

    def _drop(_r, key=key):
        with _lock:
            ent = _cache.get(key)
            if ent is not None and ent[0]() is None:
                del _cache[key]

    with _lock:
        _cache[key] = (weakref.ref(mesh.triangles, _drop), dm)
    return dm
