"""Test-input builders: meshes and Poisson kernels, restating the reference.

TEST INFRASTRUCTURE (see oracle/__init__.py).  Produces the same vertices,
CCW triangles and Poisson kernel P as the reference generators so that the
GPU box (which has no /root/reference) can rebuild real inputs; the golden
fixtures carry sha256 digests of the reference's own arrays so a test can
tell whether the rebuilt input is bitwise the reference's.

Restated from /root/reference/pkg/src/pathfield:
  mesh.py:244-247 _signed_areas; :57-68 CCW normalisation; :113-157 edges /
  boundary / neighbours / vertex_triangles; :370-388 generate_disk_mesh;
  :391-405 generate_rectangle_mesh; :424-457 generate_holes_mesh;
  :460-470 _polygon_points; :486-505 _staggered_interior;
  :580-600 _delaunay_raw/_prune; laplacian.py:91-134 assemble_cotan;
  laplacian.py:29-61 InteriorFactor; solvers.py:278-303 poisson_kernel.
"""

from __future__ import annotations

import hashlib
import math
from dataclasses import dataclass

import numpy as np
import scipy.sparse as sp
from scipy.sparse.linalg import splu
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

    @property
    def n(self):
        return len(self.vertices)

    def boundary_mask(self) -> np.ndarray:
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


def cotan_laplacian(mesh: Mesh) -> sp.csr_matrix:
    """laplacian.py:91-134 (same COO construction, so identical duplicate sums)."""
    v, t, n = mesh.vertices, mesh.triangles, mesh.n
    rows, cols, vals = [], [], []
    for c0, c1, c2 in ((0, 1, 2), (1, 2, 0), (2, 0, 1)):
        pk, pi, pj = v[t[:, c0]], v[t[:, c1]], v[t[:, c2]]
        u, w = pi - pk, pj - pk
        cross = u[:, 0] * w[:, 1] - u[:, 1] * w[:, 0]
        cot = (u * w).sum(axis=1) / np.abs(cross)
        half = 0.5 * cot
        rows += [t[:, c1], t[:, c2]]
        cols += [t[:, c2], t[:, c1]]
        vals += [half, half]
    off = sp.coo_matrix((np.concatenate(vals), (np.concatenate(rows), np.concatenate(cols))),
                        shape=(n, n)).tocsr()
    diag = -np.asarray(off.sum(axis=1)).ravel()
    return (off + sp.diags(diag)).tocsr()


def poisson_kernel(mesh: Mesh, col_chunk: int | None = None) -> tuple[np.ndarray, np.ndarray]:
    """solvers.py:278-303: P_IB = -Lc_II^{-1} Lc_IB; boundary rows are indicators.

    Returns (dense, boundary).  ``col_chunk`` solves in column chunks (needed
    at 1M vertices; not bitwise equal to the all-columns solve).
    """
    lc = cotan_laplacian(mesh)
    bmask = mesh.boundary_mask()
    boundary = np.flatnonzero(bmask)
    interior = np.flatnonzero(~bmask)
    n, k = mesh.n, boundary.size
    dense = np.zeros((n, k))
    dense[boundary, np.arange(k)] = 1.0
    if interior.size:
        lc_i = lc[interior]
        lc_ii = lc_i[:, interior]
        lc_ib = lc_i[:, boundary]
        lu = splu((-lc_ii).tocsc())
        if col_chunk is None:
            p_ib = lu.solve(np.asarray(lc_ib.toarray(), dtype=float))
        else:
            p_ib = np.empty((interior.size, k))
            for a in range(0, k, col_chunk):
                b = min(k, a + col_chunk)
                p_ib[:, a:b] = lu.solve(np.asarray(lc_ib[:, a:b].toarray(), dtype=float))
        tiny = (p_ib > -1e-12) & (p_ib < 0.0)
        p_ib[tiny] = 0.0
        dense[interior] = p_ib
    return dense, boundary


def _solve_cols(args):
    """Worker: factor -L_II once, solve a column range of -L_IB into shared memory."""
    shm_name, shape, interior_size, cols, lc_ii, lc_ib = args
    from multiprocessing import shared_memory
    try:  # one BLAS thread per worker: the workers are the parallelism
        from threadpoolctl import threadpool_limits
        threadpool_limits(1)
    except Exception:
        pass
    shm = shared_memory.SharedMemory(name=shm_name)
    try:
        out = np.ndarray(shape, dtype=np.float64, buffer=shm.buf)
        lu = splu((-lc_ii).tocsc())
        a, b = cols
        for c0 in range(a, b, 64):
            c1 = min(b, c0 + 64)
            x = lu.solve(np.asarray(lc_ib[:, c0:c1].toarray(), dtype=float))
            tiny = (x > -1e-12) & (x < 0.0)
            x[tiny] = 0.0
            out[:, c0:c1] = x
    finally:
        shm.close()
    return cols


def poisson_kernel_parallel(mesh: Mesh, workers: int = 8):
    """poisson_kernel for large meshes: `workers` processes each factor -L_II
    (SuperLU, as solvers.py:278-303) and solve a column range in 64-column
    chunks into shared memory.  Column-chunked solves differ from the
    all-columns solve by ~1e-17 absolute; there is no reference
    P at this size to compare against, so the returned P is the shared input."""
    from concurrent.futures import ProcessPoolExecutor
    from multiprocessing import get_context, shared_memory
    lc = cotan_laplacian(mesh)
    bmask = mesh.boundary_mask()
    boundary = np.flatnonzero(bmask)
    interior = np.flatnonzero(~bmask)
    n, k = mesh.n, boundary.size
    lc_i = lc[interior]
    lc_ii = lc_i[:, interior].tocsr()
    lc_ib = lc_i[:, boundary].tocsc()
    shm = shared_memory.SharedMemory(create=True, size=max(8, interior.size * k * 8))
    try:
        shape = (interior.size, k)
        bounds = np.linspace(0, k, workers + 1).astype(int)
        jobs = [(shm.name, shape, interior.size, (int(a), int(b)), lc_ii, lc_ib)
                for a, b in zip(bounds[:-1], bounds[1:]) if b > a]
        with ProcessPoolExecutor(len(jobs), mp_context=get_context("fork")) as ex:
            list(ex.map(_solve_cols, jobs))
        p_ib = np.ndarray(shape, dtype=np.float64, buffer=shm.buf)
        dense = np.zeros((n, k))
        dense[boundary, np.arange(k)] = 1.0
        dense[interior] = p_ib
    finally:
        shm.close()
        shm.unlink()
    return dense, boundary


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
