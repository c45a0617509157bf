"""Workload inputs: the reference's mesh generators and the benchmark configs.

INPUT GENERATION for bench.py and tests/ (not product code, not the
oracle): the GPU box has no /root/reference, so the meshes the reference
would build for SURVEY Appendix B's configs are rebuilt here with the same
numpy / qhull calls — bitwise the reference's vertices and CCW triangles
(the golden fixtures pin sha256 digests of the reference's own arrays;
tests/test_oracle.py).  The product package never imports this module; the
Poisson kernel P of a workload is built on the device by the product
(laplacian.DevicePoisson) or, for parity, by the oracle's SuperLU
restatement (oracle/inputs.py).

Restated from /root/reference/pkg/src/pathfield:
  mesh.py:244-247 _signed_areas; :57-68 CCW normalisation; :113-157 edges /
  boundary / neighbours / vertex_triangles; :370-388 generate_disk_mesh;
  :391-405 generate_rectangle_mesh; :424-457 generate_holes_mesh;
  :460-470 _polygon_points; :486-505 _staggered_interior;
  :580-600 _delaunay_raw/_prune; domain.py:155-165 default_endpoints.
"""

from __future__ import annotations

import hashlib
import math
from dataclasses import dataclass

import numpy as np
from scipy.spatial import Delaunay


def sha(a: np.ndarray) -> str:
    a = np.ascontiguousarray(a)
    return hashlib.sha256(a.view(np.uint8).tobytes() + str(a.dtype).encode()
                          + str(a.shape).encode()).hexdigest()


@dataclass
class Mesh:
    """Plain arrays of a TriMesh after the reference's normalisation."""
    vertices: np.ndarray      # (n, 2) float64
    triangles: np.ndarray     # (nt, 3) int64, CCW
    areas: np.ndarray         # (nt,) float64, |signed area|
    _bmask: np.ndarray | None = None   # cached boundary mask (the arrays are not mutated)

    @property
    def n(self):
        return len(self.vertices)

    def boundary_mask(self) -> np.ndarray:
        if self._bmask is None:
            self._bmask = self._boundary_mask()
        return self._bmask

    def _boundary_mask(self) -> np.ndarray:
        # mesh.py:128-144: vertices on an edge with exactly one triangle
        t = self.triangles
        e = np.concatenate([t[:, [0, 1]], t[:, [1, 2]], t[:, [2, 0]]])
        e.sort(axis=1)
        key = e[:, 0] * self.n + e[:, 1]
        uniq, cnt = np.unique(key, return_counts=True)
        bnd = uniq[cnt == 1]
        mask = np.zeros(self.n, dtype=bool)
        mask[bnd // self.n] = True
        mask[bnd % self.n] = True
        return mask

    @property
    def boundary_vertices(self):
        return np.flatnonzero(self.boundary_mask())

    @property
    def interior_vertices(self):
        return np.flatnonzero(~self.boundary_mask())

    @property
    def bbox_diagonal(self) -> float:
        lo, hi = self.vertices.min(axis=0), self.vertices.max(axis=0)
        return float(np.hypot(*(hi - lo)))


def _signed_areas(v, t):
    p0, p1, p2 = v[t[:, 0]], v[t[:, 1]], v[t[:, 2]]
    u, w = p1 - p0, p2 - p0
    return 0.5 * (u[:, 0] * w[:, 1] - u[:, 1] * w[:, 0])


def make_mesh(vertices, triangles) -> Mesh:
    v = np.ascontiguousarray(np.asarray(vertices, dtype=float))
    t = np.ascontiguousarray(np.asarray(triangles, dtype=np.int64)).copy()
    signed = _signed_areas(v, t)
    flip = signed < 0
    t[flip] = t[flip][:, ::-1]
    return Mesh(v, t, np.abs(signed))


def _polygon_points(corners, spacing):
    corners = [np.asarray(c, dtype=float) for c in corners]
    pts = []
    for a, b in zip(corners, corners[1:] + corners[:1]):
        seg = b - a
        cnt = max(1, int(round(np.hypot(*seg) / spacing)))
        for i in range(cnt):
            pts.append(a + seg * (i / cnt))
    return np.array(pts)


def _staggered_interior(x0, x1, y0, y1, spacing, seed, jitter=0.08):
    rng = np.random.default_rng(seed)
    dy = spacing * math.sqrt(3.0) / 2.0
    rows = []
    j = 0
    y = y0 + dy
    while y < y1:
        off = 0.5 * spacing if j % 2 else 0.0
        xs = np.arange(x0 + spacing + off, x1 - 0.25 * spacing, spacing)
        if len(xs):
            pts = np.column_stack([xs, np.full(len(xs), y)])
            pts += (rng.random(pts.shape) - 0.5) * (jitter * spacing)
            rows.append(pts)
        y += dy
        j += 1
    if not rows:
        return np.empty((0, 2))
    return np.vstack(rows)


def _delaunay_raw(points):
    tri = Delaunay(points)
    tris = tri.simplices.astype(np.int64)
    areas = np.abs(_signed_areas(points, tris))
    scale2 = np.ptp(points, axis=0).max() ** 2
    return points, tris[areas > 1e-12 * scale2]


def _prune(points, tris) -> Mesh:
    used = np.zeros(len(points), dtype=bool)
    used[tris.ravel()] = True
    remap = np.cumsum(used) - 1
    return make_mesh(points[used], remap[tris])


def disk_mesh(rings: int) -> Mesh:
    pts = [(0.0, 0.0)]
    for j in range(1, rings + 1):
        r = j / rings
        cnt = 6 * j
        ang = 2.0 * np.pi * np.arange(cnt) / cnt
        pts.extend(zip(r * np.cos(ang), r * np.sin(ang)))
    return _prune(*_delaunay_raw(np.array(pts)))


def rectangle_mesh(length, width, spacing, seed=0, jitter=0.08) -> Mesh:
    boundary = _polygon_points([(0, 0), (length, 0), (length, width), (0, width)], spacing)
    interior = _staggered_interior(0, length, 0, width, spacing, seed, jitter)
    keep = (interior[:, 0] > 0.45 * spacing) & (interior[:, 0] < length - 0.45 * spacing) \
        & (interior[:, 1] > 0.45 * spacing) & (interior[:, 1] < width - 0.45 * spacing)
    return _prune(*_delaunay_raw(np.vstack([boundary, interior[keep]])))


def holes_mesh(spacing, size=(2.0, 1.25),
               holes=((0.55, 0.42, 0.21), (1.42, 0.78, 0.23), (1.05, 0.3, 0.13)),
               seed=0, jitter=0.08) -> Mesh:
    w, h = size
    boundary = _polygon_points([(0, 0), (w, 0), (w, h), (0, h)], spacing)
    rings = []
    for cx, cy, r in holes:
        cnt = max(8, int(round(2 * np.pi * r / (0.9 * spacing))))
        ang = 2 * np.pi * np.arange(cnt) / cnt
        rings.append(np.column_stack([cx + r * np.cos(ang), cy + r * np.sin(ang)]))
    interior = _staggered_interior(0, w, 0, h, spacing, seed, jitter)
    keep = (interior[:, 0] > 0.45 * spacing) & (interior[:, 0] < w - 0.45 * spacing) \
        & (interior[:, 1] > 0.45 * spacing) & (interior[:, 1] < h - 0.45 * spacing)
    for cx, cy, r in holes:
        keep &= np.hypot(interior[:, 0] - cx, interior[:, 1] - cy) > r + 0.45 * spacing
    pts, tris = _delaunay_raw(np.vstack([boundary] + rings + [interior[keep]]))
    cen = pts[tris].mean(axis=1)
    drop = np.zeros(len(tris), dtype=bool)
    for cx, cy, r in holes:
        drop |= np.hypot(cen[:, 0] - cx, cen[:, 1] - cy) < r
    return _prune(pts, tris[~drop])


def square_hole_mesh(spacing=0.0235, lo=0.4, hi=0.6, seed=0, jitter=0.08) -> Mesh:
    """C1: unit square minus the square [lo,hi]^2.

    The holes-mesh recipe with a square obstacle: boundary points on both
    squares at `spacing`, staggered interior kept at 0.45*spacing from the
    outer walls and outside the obstacle grown by 0.45*spacing, Delaunay,
    drop triangles whose centroid lies inside the obstacle, prune.
    """
    boundary = _polygon_points([(0, 0), (1, 0), (1, 1), (0, 1)], spacing)
    hole = _polygon_points([(lo, lo), (hi, lo), (hi, hi), (lo, hi)], spacing)
    interior = _staggered_interior(0, 1, 0, 1, spacing, seed, jitter)
    g = 0.45 * spacing
    keep = (interior[:, 0] > g) & (interior[:, 0] < 1 - g) \
        & (interior[:, 1] > g) & (interior[:, 1] < 1 - g)
    inside_grown = (interior[:, 0] > lo - g) & (interior[:, 0] < hi + g) \
        & (interior[:, 1] > lo - g) & (interior[:, 1] < hi + g)
    keep &= ~inside_grown
    pts, tris = _delaunay_raw(np.vstack([boundary, hole, interior[keep]]))
    cen = pts[tris].mean(axis=1)
    drop = (cen[:, 0] > lo) & (cen[:, 0] < hi) & (cen[:, 1] > lo) & (cen[:, 1] < hi)
    return _prune(pts, tris[~drop])


def default_endpoints(mesh: Mesh) -> tuple[int, int]:
    """domain.py:155-165."""
    interior = mesh.interior_vertices
    center = mesh.vertices.mean(axis=0)
    d = np.hypot(*(mesh.vertices[interior] - center).T)
    target = int(interior[np.argmin(d)])
    dt = np.hypot(*(mesh.vertices[interior] - mesh.vertices[target]).T)
    source = int(interior[np.argmax(dt)])
    return source, target


def synthetic_kernel(n: int, k: int, seed: int = 0) -> np.ndarray:
    """Random row-stochastic P (softmax of N(0,1) rows), SURVEY §8d 'Synthetic'."""
    rng = np.random.default_rng(seed)
    x = rng.standard_normal((n, k))
    x = np.exp(x - x.max(axis=1, keepdims=True))
    return x / x.sum(axis=1, keepdims=True)


BUILDERS = {
    "disk": disk_mesh,
    "rectangle": rectangle_mesh,
    "holes": holes_mesh,
    "square_hole": square_hole_mesh,
}


def build(spec: dict) -> Mesh:
    """Build a mesh from a JSON-able spec {"gen": name, **kwargs}."""
    spec = dict(spec)
    gen = BUILDERS[spec.pop("gen")]
    if "holes" in spec:
        spec["holes"] = tuple(tuple(h) for h in spec["holes"])
    if "size" in spec:
        spec["size"] = tuple(spec["size"])
    return gen(**spec)


# ---------------------------------------------------------------------------
# SURVEY Appendix B / §8d config recipes
# ---------------------------------------------------------------------------

SPECS = {
    # C1: square + square obstacle, 2,104 x 208 (reference CPU config)
    "c1": {"gen": "square_hole", "spacing": 0.0235},
    # C2 / C3: 50:1 corridor, 102,104 x 4,250 (the reference's maze stand-in)
    "c2": {"gen": "rectangle", "length": 50.0, "width": 1.0, "spacing": 0.024},
    # C2': literal 100K x ~1K shape, 106,030 x 1,234
    "c2p": {"gen": "rectangle", "length": 1.5, "width": 1.0, "spacing": 0.00405},
    # C4 / C5: 20 circular obstacles on a 5 x 4 grid, 1,000,386 x 4,102
    "c4": {"gen": "holes", "spacing": 0.0017, "size": [2.0, 1.25],
           "holes": [[0.2 + 0.4 * i, 0.16 + 0.31 * j, 0.0034]
                     for i in range(5) for j in range(4)]},
}


def c4_targets(mesh: Mesh, count: int = 8) -> np.ndarray:
    """SURVEY §8d C4 targets: default_endpoints' target plus count-1 more from
    np.random.default_rng(0).choice(interior, count)."""
    _, t0 = default_endpoints(mesh)
    more = np.random.default_rng(0).choice(mesh.interior_vertices, count)
    out = [t0] + [int(x) for x in more if int(x) != t0]
    return np.array(out[:count], dtype=np.int64)


def c5_jobs(mesh: Mesh, targets: int = 1024, paths: int = 10_000):
    """T targets rng(0).choice(interior, T, replace=False); sources
    rng(1).choice(interior, paths), source i paired with target i % T, pairs
    with source == target skipped.  Returns (targets, sources, field_of)."""
    interior = mesh.interior_vertices
    tg = np.random.default_rng(0).choice(interior, targets, replace=False).astype(np.int64)
    src = np.random.default_rng(1).choice(interior, paths).astype(np.int64)
    fo = np.arange(paths, dtype=np.int64) % targets
    keep = src != tg[fo]
    return tg, src[keep], fo[keep]
