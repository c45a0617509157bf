"""Triangle-descent path tracing on the B200 — mirror of ``pathfield/paths.py``.

* :func:`triangle_descent` (paths.py:292-307): same signature, same
  :class:`TracedPath` (points, locations, source, target, status,
  stuck_vertex), same statuses; runs the K8 kernel for one source.
* :func:`triangle_descent_batch` (additive): many sources, one
  or many fields, one launch; equal to per-source ``triangle_descent``.
* :func:`triangle_gradient` (paths.py:113-121) on the device.

The location sequence is bit-identical to the reference given the same field
(the kernel follows numpy's rounding, see csrc/trace.cu).
"""

from __future__ import annotations

import ctypes
import threading
from dataclasses import dataclass

import numpy as np

from . import _device as dev
from . import _native as nat
from .config import DEFAULTS, Settings
from .errors import DegenerateGeometryError, InvalidTargetError
from .mesh import device_mesh
from .solvers import ScalarField

STATUS_REACHED = "reached"
STATUS_STUCK = "stuck"
STATUS_MAX_STEPS = "max-steps-exceeded"
_STATUS = {0: STATUS_REACHED, 1: STATUS_STUCK, 2: STATUS_MAX_STEPS}


@dataclass(frozen=True)
class TracedPath:
    """A polyline of mesh-located points from source toward target (paths.py:32-55)."""

    points: np.ndarray
    locations: list
    source: int
    target: int
    status: str
    stuck_vertex: int | None = None

    def __post_init__(self):
        self.points.setflags(write=False)

    @property
    def length(self) -> float:
        if len(self.points) < 2:
            return 0.0
        d = np.diff(self.points, axis=0)
        return float(np.hypot(d[:, 0], d[:, 1]).sum())

    @property
    def reached(self) -> bool:
        return self.status == STATUS_REACHED


class PfPaths(ctypes.Structure):
    _fields_ = [("kind", ctypes.c_void_p), ("i", ctypes.c_void_p), ("j", ctypes.c_void_p),
                ("t", ctypes.c_void_p), ("x", ctypes.c_void_p), ("y", ctypes.c_void_p),
                ("cap", ctypes.c_int64), ("count", ctypes.c_void_p),
                ("status", ctypes.c_void_p), ("stuck", ctypes.c_void_p),
                ("qx", ctypes.c_void_p), ("qy", ctypes.c_void_p)]


def _byref(s):
    return ctypes.addressof(s)


class PathBuffers:
    """Device output of one tracer launch (pf_paths_t) and its host copy."""

    def reshape(self, cap: int) -> None:
        """Reuse the same storage with a different per-path capacity."""
        self.cap = cap
        self.struct.cap = cap

    def __init__(self, t, npaths: int, cap: int, device):
        self.npaths, self.cap_total = npaths, npaths * cap
        self.cap = cap
        tot = max(npaths * cap, 1)
        self.kind = t.empty(tot, dtype=t.int8, device=device)
        self.i = t.empty(tot, dtype=t.int32, device=device)
        self.j = t.empty(tot, dtype=t.int32, device=device)
        self.t = t.empty(tot, dtype=t.float64, device=device)
        self.x = t.empty(tot, dtype=t.float64, device=device)
        self.y = t.empty(tot, dtype=t.float64, device=device)
        self.count = t.empty(max(npaths, 1), dtype=t.int64, device=device)
        self.status = t.empty(max(npaths, 1), dtype=t.int32, device=device)
        self.stuck = t.empty(max(npaths, 1), dtype=t.int64, device=device)
        self.q = t.empty((2, max(npaths, 1)), dtype=t.float64, device=device)
        self.struct = PfPaths(self.kind.data_ptr(), self.i.data_ptr(), self.j.data_ptr(),
                              self.t.data_ptr(), self.x.data_ptr(), self.y.data_ptr(), cap,
                              self.count.data_ptr(), self.status.data_ptr(),
                              self.stuck.data_ptr(), self.q[0].data_ptr(), self.q[1].data_ptr())


_ws_lock = threading.Lock()
_workspaces: dict = {}


def _workspace(t, npaths: int, cap: int, device, slot: str) -> PathBuffers:
    """Per-(thread, device, slot) path output buffers, grown on demand and reused:
    a 10,000-path launch needs ~2.7 GB of location buffers, and fresh device
    allocations of that size cost more than the trace itself."""
    key = (threading.get_ident(), str(device), slot)
    with _ws_lock:
        ws = _workspaces.get(key)
    if ws is None or ws.npaths < npaths or ws.cap_total < npaths * cap:
        ws = PathBuffers(t, max(npaths, 1), cap, device)
        ws.npaths, ws.cap_total = max(npaths, 1), max(npaths, 1) * cap
        with _ws_lock:
            _workspaces[key] = ws
    else:
        ws.reshape(cap)
    return ws


def _fields_to_device(t, fields, n, device):
    """Stack field values (numpy or device tensors) into an (F, n) FP64 device tensor."""
    vals = []
    for f in fields:
        v = f if isinstance(f, t.Tensor) else (f.values if hasattr(f, "values") else f)
        if isinstance(v, np.ndarray):   # a field dv_field returned: its device copy
            mirror = dev.field_mirror(v)
            if mirror is not None and mirror.device == device and mirror.numel() >= n:
                v = mirror
        if isinstance(v, t.Tensor):
            vals.append(v.to(device=device, dtype=t.float64).reshape(-1)[:n])
        else:
            vals.append(t.from_numpy(np.array(v, dtype=np.float64)).to(device))
    return t.stack(vals) if len(vals) > 1 else vals[0].reshape(1, -1).contiguous()


def trace_arrays(mesh, fields, targets, sources, field_of=None, settings: Settings = DEFAULTS,
                 cap: int | None = None, entry: str = "pf_trace_batch_f64", layout=None):
    """Launch K8 and return the raw device outputs (PathBuffers), rerunning overflows.

    `fields` is a list of field values (numpy or device tensors) or an (F, n)
    device tensor, `targets` their targets, `sources` the start vertices,
    `field_of[p]` the field of path p.  With `layout = (field_ld, vertex_ld)`
    `fields` is a device FP64 tensor read in place as field f, vertex v at
    ``fields[f * field_ld + v * vertex_ld]`` (e.g. the (n, T) batched-KL
    output: (1, T)).  The returned buffers are a per-thread workspace: valid
    until the next call from the same thread.
    """
    t = dev.require_cuda()
    dm = device_mesh(mesh)
    sources = np.asarray(sources, dtype=np.int64)
    npaths = sources.size
    targets = np.asarray(targets, dtype=np.int64)
    fo = None if field_of is None else np.asarray(field_of, dtype=np.int32)
    step_cap = int(settings.step_cap_factor) * dm.n
    if layout is not None:
        if fields.dtype != t.float64 or fields.device != dm.device:
            raise ValueError("strided fields must be an FP64 tensor on the mesh device")
        F = fields
        fld_ld, vtx_ld = int(layout[0]), int(layout[1])
        call = lambda src, fo_, cnt, out: nat.call(  # noqa: E731
            "pf_trace_fields_f64", _byref(dm.struct), F.data_ptr(), fld_ld, vtx_ld,
            tgt_d.data_ptr(), src, fo_, cnt, step_cap, _byref(out), s)
    else:
        if isinstance(fields, t.Tensor) and fields.dim() == 2:   # (F, n) device block
            F = fields.to(device=dm.device, dtype=t.float64).contiguous()
        else:
            F = _fields_to_device(t, fields, dm.n, dm.device)
        call = lambda src, fo_, cnt, out: nat.call(  # noqa: E731
            entry, _byref(dm.struct), F.data_ptr(), tgt_d.data_ptr(), src, fo_, cnt, step_cap,
            _byref(out), s)
    src_d = t.from_numpy(sources).to(dm.device)
    tgt_d = t.from_numpy(targets).to(dm.device)
    fo_d = None if fo is None else t.from_numpy(fo).to(dm.device)
    s = t.cuda.current_stream(dm.device).cuda_stream
    if cap is None:
        cap = int(min(step_cap + 2, max(64, 8 * int(np.sqrt(dm.n)) + 64)))
    buf = _workspace(t, npaths, cap, dm.device, "main")
    if npaths:
        call(src_d.data_ptr(), nat.ptr(fo_d), npaths, buf.struct)
    counts = buf.count[:npaths].cpu().numpy()
    over = np.flatnonzero(counts > cap)
    extra = None
    if over.size:
        cap2 = int(counts[over].max())
        sub_src = t.from_numpy(sources[over]).to(dm.device)
        sub_fo = None if fo is None else t.from_numpy(fo[over]).to(dm.device)
        extra = _workspace(t, over.size, cap2, dm.device, "overflow")
        call(sub_src.data_ptr(), nat.ptr(sub_fo), over.size, extra.struct)
    return buf, counts, over, extra


def trace_fields_status(mesh, fields, field_ld: int, vertex_ld: int, targets, sources,
                        field_of=None, settings: Settings = DEFAULTS):
    """:func:`trace_fields` without building the host TracedPath objects:
    returns (status codes (0 reached, 1 stuck, 2 max steps), location counts)
    as numpy arrays — the per-path result summary a batched caller needs."""
    sources = np.asarray(sources, dtype=np.int64).reshape(-1)
    targets = np.asarray(targets, dtype=np.int64).reshape(-1)
    fo = None if field_of is None else np.asarray(field_of, dtype=np.int64).reshape(-1)
    if sources.size == 0:
        return np.zeros(0, np.int32), np.zeros(0, np.int64)
    buf, counts, over, extra = trace_arrays(mesh, fields, targets, sources, fo, settings,
                                            layout=(field_ld, vertex_ld))
    return buf.status[:sources.size].cpu().numpy().astype(np.int32), counts


def trace_fields(mesh, fields, field_ld: int, vertex_ld: int, targets, sources, field_of=None,
                 settings: Settings = DEFAULTS) -> list[TracedPath]:
    """:func:`triangle_descent_batch` over device-resident fields in any 2-D
    layout (field f's value at vertex v is ``fields[f * field_ld + v * vertex_ld]``),
    without copying them: the multi-GPU tracers (parallel.py) trace straight
    from a gathered field or from a rank's (n, T) batched-KL columns.
    `targets[f]` is field f's target; path p descends field ``field_of[p]``
    (0 if None).  Validation (source == target) is the caller's."""
    sources = np.asarray(sources, dtype=np.int64).reshape(-1)
    targets = np.asarray(targets, dtype=np.int64).reshape(-1)
    fo = None if field_of is None else np.asarray(field_of, dtype=np.int64).reshape(-1)
    if sources.size == 0:
        return []
    buf, counts, over, extra = trace_arrays(mesh, fields, targets, sources, fo, settings,
                                            layout=(field_ld, vertex_ld))
    return _host_paths(buf, counts, over, extra, sources, targets, fo)


def _host_paths(buf, counts, over, extra, sources, targets, field_of):
    kind = buf.kind.cpu().numpy()
    ii = buf.i.cpu().numpy()
    jj = buf.j.cpu().numpy()
    tt = buf.t.cpu().numpy()
    xx = buf.x.cpu().numpy()
    yy = buf.y.cpu().numpy()
    status = buf.status.cpu().numpy()
    stuck = buf.stuck.cpu().numpy()
    where = {int(p): r for r, p in enumerate(over)}
    if extra is not None:
        ek, ei, ej = extra.kind.cpu().numpy(), extra.i.cpu().numpy(), extra.j.cpu().numpy()
        et, ex, ey = extra.t.cpu().numpy(), extra.x.cpu().numpy(), extra.y.cpu().numpy()
    out = []
    for p in range(len(sources)):
        c = int(counts[p])
        if p in where:
            r = where[p]
            a = r * extra.cap
            K, I_, J, T_, X, Y = ek[a:a + c], ei[a:a + c], ej[a:a + c], et[a:a + c], ex[a:a + c], ey[a:a + c]
        else:
            a = p * buf.cap
            K, I_, J, T_, X, Y = kind[a:a + c], ii[a:a + c], jj[a:a + c], tt[a:a + c], xx[a:a + c], yy[a:a + c]
        locs = [("vertex", int(I_[q])) if K[q] == 0 else ("edge", int(I_[q]), int(J[q]), float(T_[q]))
                for q in range(c)]
        pts = np.column_stack([X, Y]).astype(np.float64, copy=True)
        fi = 0 if field_of is None else int(field_of[p])
        st = _STATUS[int(status[p])]
        sv = int(stuck[p]) if st == STATUS_STUCK else None
        out.append(TracedPath(pts, locs, int(sources[p]), int(targets[fi]), st, sv))
    return out


def _batch(mesh, fields, sources, settings, field_of, entry):
    if isinstance(fields, ScalarField) or hasattr(fields, "target"):
        fields = [fields]
    fields = list(fields)
    targets = np.array([int(f.target) for f in fields], dtype=np.int64)
    sources = np.asarray(sources, dtype=np.int64).reshape(-1)
    fo = None if field_of is None else np.asarray(field_of, dtype=np.int64).reshape(-1)
    ft = targets[fo] if fo is not None else np.full(sources.size, targets[0])
    if np.any(sources == ft):
        raise InvalidTargetError("source equals target")
    n = len(mesh.vertices)
    if sources.size and (sources.min() < 0 or sources.max() >= n):
        raise InvalidTargetError("source out of range")
    buf, counts, over, extra = trace_arrays(mesh, fields, targets, sources, fo, settings,
                                            entry=entry)
    return _host_paths(buf, counts, over, extra, sources, targets, fo)


def triangle_descent_batch(mesh, fields, sources, settings: Settings = DEFAULTS,
                           field_of=None) -> list[TracedPath]:
    """Trace many sources in one launch; path p descends fields[field_of[p]].

    ``fields`` is one ScalarField or a list of them (their ``target`` is the
    destination); ``field_of`` defaults to field 0 for every path.  Equal to
    ``[triangle_descent(mesh, fields[field_of[p]], sources[p]) for p]``.
    """
    return _batch(mesh, fields, sources, settings, field_of, "pf_trace_batch_f64")


def edge_descent_batch(mesh, fields, sources, settings: Settings = DEFAULTS,
                       field_of=None) -> list[TracedPath]:
    """Vertex walks (paths.py:71-94) for many sources in one launch."""
    return _batch(mesh, fields, sources, settings, field_of, "pf_edge_descent_batch_f64")


def edge_descent(mesh, field: ScalarField, source: int,
                 settings: Settings = DEFAULTS) -> TracedPath:
    """Vertex walk choosing the neighbour with the largest value drop (paths.py:71-94)."""
    if source == field.target:
        raise InvalidTargetError("source equals target")
    return edge_descent_batch(mesh, [field], [int(source)], settings)[0]


def find_local_minima(mesh, field: ScalarField) -> list[int]:
    """Vertices (excluding the target) strictly below every neighbour (paths.py:314-324)."""
    t = dev.require_cuda()
    dm = device_mesh(mesh)
    F = _fields_to_device(t, [field], dm.n, dm.device)
    out = t.empty(dm.n, dtype=t.uint8, device=dm.device)
    nat.call("pf_local_minima_f64", _byref(dm.struct), F.data_ptr(), int(field.target),
             out.data_ptr(), t.cuda.current_stream(dm.device).cuda_stream)
    return [int(v) for v in t.nonzero(out).flatten().cpu().numpy()]


def triangle_descent(mesh, field: ScalarField, source: int,
                     settings: Settings = DEFAULTS) -> TracedPath:
    """Trace the negative interpolant gradient through triangle interiors (paths.py:292-307)."""
    if source == field.target:
        raise InvalidTargetError("source equals target")
    return triangle_descent_batch(mesh, [field], [int(source)], settings)[0]


def triangle_gradient(mesh, field_values, ti: int) -> np.ndarray:
    """Gradient of the linear interpolant on triangle ti (paths.py:113-121), on the device."""
    if mesh.triangle_areas[ti] <= 0:
        raise DegenerateGeometryError(f"triangle {ti} is degenerate")
    t = dev.require_cuda()
    dm = device_mesh(mesh)
    vals = field_values.values if isinstance(field_values, ScalarField) else field_values
    F = _fields_to_device(t, [vals], dm.n, dm.device)
    tri = t.tensor([int(ti)], dtype=t.int64, device=dm.device)
    out = t.empty(2, dtype=t.float64, device=dm.device)
    nat.call("pf_triangle_gradient_f64", _byref(dm.struct), F.data_ptr(), tri.data_ptr(), 1,
             out.data_ptr(), t.cuda.current_stream(dm.device).cuda_stream)
    return out.cpu().numpy()


def np_hypot_device(x, y) -> np.ndarray:
    """The tracer's hypot (glibc non-FMA kernel) evaluated on the device (testing aid)."""
    t = dev.require_cuda()
    xd = t.from_numpy(np.ascontiguousarray(x, dtype=np.float64)).cuda()
    yd = t.from_numpy(np.ascontiguousarray(y, dtype=np.float64)).cuda()
    out = t.empty_like(xd)
    nat.call("pf_np_hypot_f64", xd.data_ptr(), yd.data_ptr(), xd.numel(), out.data_ptr(),
             t.cuda.current_stream().cuda_stream)
    return out.cpu().numpy()


# ---------------------------------------------------------------------------
# Path metric (paths.py:326-368)
# ---------------------------------------------------------------------------

_MAX_RESAMPLED = 1 << 31  # resampled points per call (16 B each on the device)


def _points_of(x) -> np.ndarray:
    """paths.py:352-353: a TracedPath's points, else the array as float."""
    pts = x.points if hasattr(x, "points") and hasattr(x, "locations") else x
    return np.asarray(pts, dtype=float)


def _resample_device(sources):
    """Upload the source polylines and run the arc-length kernel: returns the
    device points and arcs, host offsets / lengths / totals / shortest
    positive segments."""
    t = dev.require_cuda()
    device = t.device("cuda", t.cuda.current_device())
    s = t.cuda.current_stream(device).cuda_stream
    lens = np.array([len(p) for p in sources], dtype=np.int64)
    offs = np.zeros(len(sources) + 1, dtype=np.int64)
    np.cumsum(lens, out=offs[1:])
    flat = np.concatenate([p.reshape(-1, 2) for p in sources]) if offs[-1] else np.zeros((0, 2))
    pts = t.from_numpy(np.ascontiguousarray(flat, dtype=np.float64)).to(device)
    src_off = t.from_numpy(offs[:-1].copy()).to(device)
    src_len = t.from_numpy(lens).to(device)
    arc = t.empty(max(int(offs[-1]), 1), dtype=t.float64, device=device)
    segmin = t.empty(len(sources), dtype=t.float64, device=device)
    nat.call("pf_polyline_arc_f64", pts.data_ptr(), src_off.data_ptr(), src_len.data_ptr(),
             len(sources), arc.data_ptr(), segmin.data_ptr(), s)
    arc_h = arc.cpu().numpy()
    seg_h = segmin.cpu().numpy()
    totals = np.array([arc_h[offs[i] + lens[i] - 1] if lens[i] else 0.0
                       for i in range(len(sources))])
    return t, device, s, pts, arc, offs, lens, totals, seg_h


def _counts(lens, totals, inst_src, inst_step):
    """Resampled point count per instance exactly as paths.py:327-339 decides it
    (0: copied input, -1: first point only) and the number of output points."""
    cnt = np.empty(len(inst_src), dtype=np.int64)
    nout = np.empty(len(inst_src), dtype=np.int64)
    for q, (si, st) in enumerate(zip(inst_src, inst_step)):
        L, total = int(lens[si]), float(totals[si])
        if L < 2:
            cnt[q], nout[q] = 0, L
        elif total <= 0:
            cnt[q], nout[q] = -1, 1
        else:
            c = max(2, int(np.ceil(total / st)) + 1)
            cnt[q], nout[q] = c, c
    return cnt, nout


def _launch_resample(t, device, s, pts, arc, offs, lens, inst_src, cnt, nout):
    out_off = np.zeros(len(inst_src) + 1, dtype=np.int64)
    np.cumsum(nout, out=out_off[1:])
    total_out = int(out_off[-1])
    if total_out > _MAX_RESAMPLED:
        raise MemoryError(f"resampling needs {total_out} points (step too small)")
    d_src = t.from_numpy(offs[np.asarray(inst_src, dtype=np.int64)].copy()).to(device)
    d_len = t.from_numpy(lens[np.asarray(inst_src, dtype=np.int64)].copy()).to(device)
    d_cnt = t.from_numpy(cnt).to(device)
    d_off = t.from_numpy(out_off).to(device)
    rp = t.empty((max(total_out, 1), 2), dtype=t.float64, device=device)
    nat.call("pf_polyline_resample_f64", pts.data_ptr(), d_src.data_ptr(), d_len.data_ptr(),
             arc.data_ptr(), d_cnt.data_ptr(), d_off.data_ptr(), len(inst_src), total_out,
             rp.data_ptr(), s)
    return rp, d_off, out_off, (d_src, d_len, d_cnt)


def resample_polyline(points, step: float) -> np.ndarray:
    """paths.py:326-340 on the device (bitwise the reference's numpy result)."""
    pts = np.asarray(points, dtype=float)
    if len(pts) < 2:
        return pts.reshape(-1, 2)
    t, device, s, dpts, arc, offs, lens, totals, _ = _resample_device([pts.reshape(-1, 2)])
    cnt, nout = _counts(lens, totals, [0], [float(step)])
    rp, _, out_off, _ = _launch_resample(t, device, s, dpts, arc, offs, lens, [0], cnt, nout)
    return rp[:int(out_off[-1])].cpu().numpy()


def path_hausdorff_batch(pairs, step: float | None = None) -> np.ndarray:
    """``[path_hausdorff(a, b, step) for a, b in pairs]`` in one pass on the device.

    Every pair is resampled with ``step`` (default: a quarter of the shortest
    positive segment of the pair, paths.py:355-363) and its symmetric
    Hausdorff distance evaluated exhaustively on the GPU — bitwise the
    reference's cKDTree result (same squared-distance arithmetic; the nearest
    point is the nearest point).
    """
    pairs = list(pairs)
    if not pairs:
        return np.zeros(0)
    sources, index, inst_src = [], {}, []
    for a, b in pairs:
        for x in (a, b):
            pts = _points_of(x)
            if len(pts) == 0:
                raise ValueError("paths must be nonempty")
            key = id(x)
            if key not in index:
                index[key] = len(sources)
                sources.append(pts.reshape(-1, 2))
            inst_src.append(index[key])
    t, device, s, dpts, arc, offs, lens, totals, segmin = _resample_device(sources)
    inst_step = []
    for q in range(len(pairs)):
        if step is None:
            m = min(segmin[inst_src[2 * q]], segmin[inst_src[2 * q + 1]])
            st = float(m) / 4.0 if np.isfinite(m) else 1.0
        else:
            st = float(step)
        inst_step += [st, st]
    cnt, nout = _counts(lens, totals, inst_src, inst_step)
    rp, d_off, _, (d_src, d_len, d_cnt) = _launch_resample(t, device, s, dpts, arc, offs, lens,
                                                           inst_src, cnt, nout)
    res = np.empty(len(pairs))
    for c0 in range(0, len(pairs), 32767):
        c1 = min(len(pairs), c0 + 32767)
        ia = t.arange(2 * c0, 2 * c1, 2, dtype=t.int64, device=device)
        ib = ia + 1
        best = t.empty(c1 - c0, dtype=t.int64, device=device)
        nat.call("pf_hausdorff_pairs_f64", dpts.data_ptr(), arc.data_ptr(), d_src.data_ptr(),
                 d_len.data_ptr(), d_cnt.data_ptr(), rp.data_ptr(), d_off.data_ptr(),
                 ia.data_ptr(), ib.data_ptr(), c1 - c0, int(nout[2 * c0:2 * c1].max()),
                 best.data_ptr(), s)
        res[c0:c1] = np.sqrt(best.cpu().numpy().view(np.float64))
    return res


def path_hausdorff(a, b, step: float | None = None) -> float:
    """Symmetric Hausdorff distance between two densely resampled polylines
    (paths.py:343-368), on the device."""
    return float(path_hausdorff_batch([(a, b)], step)[0])
