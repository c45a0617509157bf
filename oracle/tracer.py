"""triangle_descent restatement — TEST INFRASTRUCTURE (see oracle/__init__.py).

Follows /root/reference/pkg/src/pathfield/paths.py:101-307 step for step,
with the same numpy primitives (np.hypot, 3x2 matmuls, elementwise ops), so on
the host that produced the goldens it reproduces the reference bitwise
(tests/test_oracle.py).  Topology (vertex_triangles, neighbors, the triangle
across each edge) is rebuilt from the triangle array exactly as
mesh.py:113-157 orders it (ascending indices).

Also exports :func:`topology`, the array form the device tracer consumes, so
tests can check the product's own topology builder against it.
"""

from __future__ import annotations

import numpy as np

REACHED, STUCK, MAX_STEPS = "reached", "stuck", "max-steps-exceeded"


def topology(triangles: np.ndarray, n: int):
    """(vt_ptr, vt_idx, nb_ptr, nb_idx, tri_nbr) with ascending per-vertex lists."""
    t = np.asarray(triangles, dtype=np.int64)
    nt = len(t)
    # vertex -> incident triangles (mesh.py:152-157)
    v = t.ravel()
    ti = np.repeat(np.arange(nt), 3)
    order = np.lexsort((ti, v))
    vt_idx = ti[order]
    vt_ptr = np.zeros(n + 1, dtype=np.int64)
    np.cumsum(np.bincount(v, minlength=n), out=vt_ptr[1:])
    # neighbours (mesh.py:146-151)
    e = np.concatenate([t[:, [0, 1]], t[:, [1, 2]], t[:, [2, 0]]])
    e = np.concatenate([e, e[:, ::-1]])
    key = np.unique(e[:, 0] * n + e[:, 1])
    a, b = key // n, key % n
    nb_idx = b
    nb_ptr = np.zeros(n + 1, dtype=np.int64)
    np.cumsum(np.bincount(a, minlength=n), out=nb_ptr[1:])
    # triangle across the edge opposite each slot (edge_adjacency, mesh.py:113-126)
    tri_nbr = -np.ones((nt, 3), dtype=np.int64)
    slots = np.tile(np.arange(3), nt)
    tis = np.repeat(np.arange(nt), 3)
    i = t[tis, (slots + 1) % 3]
    j = t[tis, (slots + 2) % 3]
    k = np.minimum(i, j) * n + np.maximum(i, j)
    o = np.argsort(k, kind="stable")
    ks = k[o]
    same = np.flatnonzero(ks[1:] == ks[:-1])
    for x, y in ((o[same], o[same + 1]), (o[same + 1], o[same])):
        tri_nbr[tis[x], slots[x]] = tis[y]
    return vt_ptr, vt_idx, nb_ptr, nb_idx, tri_nbr


class Tracer:
    """paths.py:137-289 with array topology."""

    def __init__(self, V, T, areas, bbox_diagonal, vals, target, source, cap, topo):
        self.V, self.T, self.areas = V, T, areas
        self.vals = vals
        self.target = target
        self.cap = cap
        self.eps_prog = 1e-14 * bbox_diagonal
        self.pts = [V[source].copy()]
        self.locs = [("vertex", source)]
        self.source = source
        self.vt_ptr, self.vt_idx, self.nb_ptr, self.nb_idx, self.tri_nbr = topo

    def grads(self, ti):
        a, b, c = self.T[ti]
        pa, pb, pc = self.V[a], self.V[b], self.V[c]
        area2 = 2.0 * self.areas[ti]
        perp = lambda v: np.array([-v[1], v[0]])  # noqa: E731
        return np.array([perp(pc - pb), perp(pa - pc), perp(pb - pa)]) / area2

    def gradient(self, ti):
        return self.vals[self.T[ti]] @ self.grads(ti)

    def emit(self, status, stuck=None):
        return dict(points=np.array(self.pts), locations=self.locs, source=self.source,
                    target=self.target, status=status, stuck_vertex=stuck)

    def append_vertex(self, v):
        self.pts.append(self.V[v].copy())
        self.locs.append(("vertex", int(v)))

    def step_from_vertex(self, v):
        if v == self.target:
            return self.emit(REACHED)
        best = None
        for ti in self.vt_idx[self.vt_ptr[v]:self.vt_ptr[v + 1]]:
            g = self.gradient(ti)
            norm = float(np.hypot(*g))
            if norm <= 0.0:
                continue
            d = -g / norm
            tri = self.T[ti]
            slot = int(np.flatnonzero(tri == v)[0])
            dlam = self.grads(ti) @ d
            others = [s for s in range(3) if s != slot]
            scale = np.abs(dlam).max() + 1e-300
            if dlam[others[0]] > 1e-12 * scale and dlam[others[1]] > 1e-12 * scale:
                if best is None or norm > best[0]:
                    best = (norm, int(ti))
        if best is not None:
            return ("tri", best[1], self.V[v].copy(), self.vals[v])
        nbrs = self.nb_idx[self.nb_ptr[v]:self.nb_ptr[v + 1]]
        diffs = self.vals[v] - self.vals[nbrs]
        lens = np.hypot(*(self.V[nbrs] - self.V[v]).T)
        slopes = diffs / lens
        bi = int(np.argmax(slopes))
        if slopes[bi] <= 0.0:
            return self.emit(STUCK, stuck=int(v))
        u = int(nbrs[bi])
        self.append_vertex(u)
        return ("vertex", u)

    def step_through_triangle(self, ti, x, cur_val):
        tri = self.T[ti]
        g = self.gradient(ti)
        norm = float(np.hypot(*g))
        if norm <= 0.0:
            return self.slide_to_best_vertex(tri, cur_val)
        d = -g / norm
        a, b, c = tri
        pa, pb, pc = self.V[a], self.V[b], self.V[c]
        area2 = 2.0 * self.areas[ti]
        cr = lambda u, w: u[0] * w[1] - u[1] * w[0]  # noqa: E731
        la = cr(pc - pb, x - pb) / area2
        lb = cr(pa - pc, x - pc) / area2
        lam = np.clip(np.array([la, lb, 1.0 - la - lb]), 0.0, None)
        lam /= lam.sum()
        dlam = self.grads(ti) @ d
        scale = np.abs(dlam).max() + 1e-300
        s_exit, slot_exit = np.inf, -1
        for s in range(3):
            if dlam[s] < -1e-14 * scale and lam[s] > 0.0:
                cand = lam[s] / -dlam[s]
                if cand < s_exit:
                    s_exit, slot_exit = cand, s
        if not np.isfinite(s_exit):
            return self.slide_to_best_vertex(tri, cur_val)
        le = lam + s_exit * dlam
        le[slot_exit] = 0.0
        le = np.clip(le, 0.0, None)
        le /= le.sum()
        hi = int(np.argmax(le))
        if le[hi] > 1.0 - 1e-12:
            w = int(tri[hi])
            if not self.progress_ok(self.V[w]):
                return self.emit(STUCK, stuck=self.nearest_vertex(x))
            self.append_vertex(w)
            return ("vertex", w)
        others = [s for s in range(3) if s != slot_exit]
        i, j = int(tri[others[0]]), int(tri[others[1]])
        if i > j:
            i, j = j, i
            others = others[::-1]
        t_param = float(le[others[1]])
        xe = le @ self.V[tri]
        if not self.progress_ok(xe):
            return self.emit(STUCK, stuck=self.nearest_vertex(x))
        self.pts.append(np.asarray(xe, dtype=float))
        self.locs.append(("edge", i, j, t_param))
        val_exit = float(le @ self.vals[tri])
        if self.target in (i, j):
            self.append_vertex(self.target)
            return self.emit(REACHED)
        nt = int(self.tri_nbr[ti, slot_exit])
        if nt < 0:
            return self.slide_along_edge(i, j, val_exit, x)
        if self.enters(nt, (i, j)):
            return ("tri", nt, xe, val_exit)
        return self.slide_along_edge(i, j, val_exit, xe)

    def enters(self, ti, edge):
        g = self.gradient(ti)
        norm = float(np.hypot(*g))
        if norm <= 0.0:
            return False
        d = -g / norm
        tri = self.T[ti]
        (slot_opp,) = [s for s in range(3) if tri[s] not in edge]
        dlam = self.grads(ti) @ d
        scale = np.abs(dlam).max() + 1e-300
        return dlam[slot_opp] > 1e-12 * scale

    def slide_along_edge(self, i, j, cur_val, x):
        w = min((i, j), key=lambda u: (self.vals[u], u))
        if self.vals[w] >= cur_val:
            return self.emit(STUCK, stuck=self.nearest_vertex(x))
        self.append_vertex(w)
        return ("vertex", w)

    def slide_to_best_vertex(self, tri, cur_val):
        w = min((int(u) for u in tri), key=lambda u: (self.vals[u], u))
        if self.vals[w] >= cur_val:
            return self.emit(STUCK, stuck=w)
        self.append_vertex(w)
        return ("vertex", w)

    def progress_ok(self, xnew):
        return float(np.hypot(*(xnew - self.pts[-1]))) >= self.eps_prog

    def nearest_vertex(self, x):
        d = self.V - x
        return int(np.argmin(np.hypot(d[:, 0], d[:, 1])))


def triangle_descent(V, T, areas, bbox_diagonal, vals, target, source, step_cap_factor=50,
                     topo=None):
    """paths.py:292-307; returns a dict with the TracedPath fields."""
    if source == target:
        raise ValueError("source equals target")
    topo = topo if topo is not None else topology(T, len(V))
    tr = Tracer(V, T, areas, bbox_diagonal, vals, target, source, step_cap_factor * len(V), topo)
    state = ("vertex", source)
    for _ in range(tr.cap):
        if state[0] == "vertex":
            state = tr.step_from_vertex(state[1])
        else:
            _, ti, x, cur_val = state
            state = tr.step_through_triangle(ti, x, cur_val)
        if isinstance(state, dict):
            return state
    return tr.emit(MAX_STEPS)


# ---------------------------------------------------------------------------
# Path metric (paths.py:326-368): resampling + symmetric Hausdorff distance
# ---------------------------------------------------------------------------

def resample_polyline(points, step: float) -> np.ndarray:
    """paths.py:326-340 (np.hypot segments, sequential cumsum, np.linspace,
    np.interp) — the same numpy calls, so bitwise the reference."""
    pts = np.asarray(points, dtype=float)
    if len(pts) < 2:
        return pts.reshape(-1, 2)
    d = np.diff(pts, axis=0)
    seg = np.hypot(d[:, 0], d[:, 1])
    arc = np.concatenate([[0.0], np.cumsum(seg)])
    total = arc[-1]
    if total <= 0:
        return pts[:1]
    cnt = max(2, int(np.ceil(total / step)) + 1)
    s = np.linspace(0.0, total, cnt)
    return np.column_stack([np.interp(s, arc, pts[:, 0]), np.interp(s, arc, pts[:, 1])])


def default_step(pa, pb) -> float:
    """paths.py:355-363: a quarter of the shortest positive segment, else 1."""
    segs = []
    for p in (pa, pb):
        if len(p) > 1:
            d = np.diff(p, axis=0)
            s = np.hypot(d[:, 0], d[:, 1])
            s = s[s > 0]
            if len(s):
                segs.append(s.min())
    return min(segs) / 4.0 if segs else 1.0


def directed_sq(ra, rb) -> float:
    """max over ra of min over rb of (dx*dx) + (dy*dy): the squared distance in
    scipy cKDTree's order for 2-D points (sqeuclidean: 0 + dx^2, then + dy^2),
    brute force instead of the tree (the nearest distance is the same value)."""
    best = 0.0
    chunk = max(1, (1 << 22) // max(1, len(rb)))
    for a in range(0, len(ra), chunk):
        x = ra[a:a + chunk]
        dx = x[:, None, 0] - rb[None, :, 0]
        dy = x[:, None, 1] - rb[None, :, 1]
        best = max(best, float(((dx * dx) + (dy * dy)).min(axis=1).max()))
    return best


def path_hausdorff(pa, pb, step=None) -> float:
    """paths.py:343-368 with the cKDTree queries replaced by brute force."""
    pa = np.asarray(pa, dtype=float)
    pb = np.asarray(pb, dtype=float)
    if len(pa) == 0 or len(pb) == 0:
        raise ValueError("paths must be nonempty")
    if step is None:
        step = default_step(pa, pb)
    ra = resample_polyline(pa, step)
    rb = resample_polyline(pb, step)
    return float(np.sqrt(max(directed_sq(ra, rb), directed_sq(rb, ra))))
