"""Device cotangent Laplacian and Poisson kernel.

Mirrors the preprocessing the reference runs before the hot path:

* ``assemble_cotan(mesh)`` — ``pathfield/laplacian.py:91-134``: the
  symmetric cotangent Laplacian, assembled on the GPU bit-for-bit (each
  edge weight is the sum of the <= 2 corner halves of its triangles, the
  diagonal is minus scipy's row sum: first entry + numpy pairwise sum of the
  rest, in ascending column order).
* ``poisson_kernel(ls)`` — ``pathfield/solvers.py:278-303``: the harmonic
  measures ``P_IB = -Lc_II^{-1} Lc_IB`` with boundary rows set to indicators.
  The reference factors ``-Lc_II`` with SuperLU and back-substitutes all k
  columns on one core (about 50 s at 100K vertices, 21 min at 1M).  Here:

    1. a host nested-dissection plan (``csrc/nd_plan.cpp``; geometric
       bisection of the planar mesh, post-order fronts, scatter maps),
    2. a multifrontal Cholesky of ``A = -Lc_II`` on the GPU, one launch per
       tree level (``pf_mf_factor_level``),
    3. a forward solve over the sparse right-hand side ``Lc_IB`` that only
       visits the (front, 32-column tile) pairs reachable from a boundary
       column (``pf_mf_forward_level``), writing ``L^{-1} B`` straight into
       the rows of the device P,
    4. a backward solve, top-down, that overwrites those rows with ``X``
       (``pf_mf_backward_level``) — P is produced in place, in the device
       layout of :class:`~._device.DeviceKernel` (row-major, ``ld =
       round_up(k, 16)``), so the divergence kernels use it without a copy,
    5. ``pf_poisson_residual_rows`` + ``pf_poisson_finalize_rows``:
       ``residual`` and, on the same read of each row, the chunk row sums;
       then boundary indicator rows, zero pads and ``row_sum_error`` — or,
       when K1 is fused or a negative entry makes the reference's clip of
       tiny negatives (``-1e-12 < P < 0 -> 0``) possible,
       ``pf_poisson_finalize``'s full pass.

  ``-Lc_II`` is a symmetric M-matrix on Delaunay meshes, so its Cholesky
  factor has non-positive off-diagonals and every term of both triangular
  solves is non-negative: the device P carries small *componentwise*
  relative error, tails included (``DESIGN.md`` §K11 and the parity tests).
"""

from __future__ import annotations

import ctypes
import threading
import weakref

import numpy as np

from . import _native as nat
from .errors import NativeError

# per-array dtypes of the host plan (nd_plan.cpp)
_I32 = ("perm_orig", "iperm", "c0", "cn", "rn", "fn", "parent", "height", "ch_ptr", "ch_idx",
        "r_pos", "r_orig", "relmap", "b_row", "b_col", "act_tile", "level_ptr", "level_nodes")
_I64 = ("foff", "r_ptr", "relmap_off", "a_ptr", "a_dst", "a_src", "b_ptr", "b_src", "act_ptr",
        "act_voff", "tile_item")
_STATS = ("n", "m", "k", "nodes", "levels", "f_total", "v_total", "nnz_l", "flops_factor",
          "flops_solve", "max_f", "max_c", "max_r", "ntiles", "tile", "leaf")

LEAF = 64   # leaf sub-domain size of the dissection
KL_CLAMP = 1e-300  # divergence.py:82-83 (the H the fused K1 precomputes)
TILE = 64   # column tile of the multi-RHS solves (pf_mf_plan_t.tile)
RESIDUAL_COLS = 512  # PF_RESIDUAL_COLS: column chunk of the residual pass


def vertex_neighbors(triangles, n: int):
    """Sorted vertex-neighbour CSR (nb_ptr, nb_idx) of a triangle list
    (mesh.py:151), built by the C++ runtime (pf_vertex_neighbors)."""
    tri = np.ascontiguousarray(triangles, dtype=np.int64)
    nb_ptr = np.empty(n + 1, dtype=np.int64)
    nb_idx = np.empty(max(6 * len(tri), 1), dtype=np.int64)
    nnz = ctypes.c_int64(0)
    nat.call("pf_vertex_neighbors", n, len(tri), tri.ctypes.data, nb_ptr.ctypes.data,
             nb_idx.ctypes.data, ctypes.byref(nnz))
    return nb_ptr, nb_idx[:nnz.value].copy()


def mesh_topology(mesh):
    """(nb_ptr, nb_idx, is_boundary) of a mirror or reference TriMesh: the
    sorted vertex neighbour CSR (mesh.py:151) and the boundary mask."""
    topo = getattr(mesh, "_topo", None)
    if topo is None:
        nb_ptr, nb_idx = vertex_neighbors(mesh.triangles, len(mesh.vertices))
    else:
        nb_ptr = np.ascontiguousarray(topo[2], dtype=np.int64)
        nb_idx = np.ascontiguousarray(topo[3], dtype=np.int64)
    isb = np.zeros(len(mesh.vertices), dtype=np.uint8)
    isb[np.asarray(mesh.boundary_vertices, dtype=np.int64)] = 1
    return nb_ptr, nb_idx, isb


def slab_needs(plan, nb_ptr, nb_idx, is_boundary, row0: int, rows: int, ld: int):
    """Host half of a row-slab build (DevicePoisson.slab_plan): which fronts the
    backward must run for rows [row0, row0 + rows) — those holding a slab row,
    a row of the slab's 1-ring (the residual reads it) or an ancestor's row —
    and the per-vertex output offsets (slab rows at (v - row0) * ld, the other
    needed rows in scratch rows after the slab, -1 elsewhere).
    Returns (need mask over fronts, rowoff (n,), number of scratch rows)."""
    pl = plan
    n = pl.n
    isb = np.asarray(is_boundary).astype(bool)
    pos_of = -np.ones(n, dtype=np.int64)
    pos_of[pl.perm_orig] = np.arange(pl.m)
    node_of_pos = np.repeat(np.arange(pl.nodes), pl.cn)
    slab = np.arange(row0, row0 + rows)
    slab_int = slab[~isb[slab]]
    lo, hi = nb_ptr[slab_int], nb_ptr[slab_int + 1]
    cnt = hi - lo
    ring = nb_idx[np.repeat(lo - (np.cumsum(cnt) - cnt), cnt) + np.arange(cnt.sum())]
    verts = np.unique(np.concatenate([slab_int, ring]))
    verts = verts[~isb[verts]]
    need = np.zeros(pl.nodes, dtype=bool)
    cur = np.unique(node_of_pos[pos_of[verts]])
    while cur.size:
        cur = cur[~need[cur]]
        need[cur] = True
        cur = np.unique(pl.parent[cur])
        cur = cur[cur >= 0]
    need_v = pl.perm_orig[np.flatnonzero(need[node_of_pos])].astype(np.int64)
    rowoff = np.full(n, -1, dtype=np.int64)
    in_slab = (need_v >= row0) & (need_v < row0 + rows)
    rowoff[need_v[in_slab]] = (need_v[in_slab] - row0) * ld
    extra = need_v[~in_slab]
    rowoff[extra] = (rows + np.arange(extra.size)) * ld
    return need, rowoff, int(extra.size)


class NdPlan:
    """Host nested-dissection plan of the interior block (nd_plan.cpp).

    Attributes are numpy arrays named as in the C++ plan, plus ``stats``.
    """

    def __init__(self, vertices, nb_ptr, nb_idx, is_boundary, leaf: int = LEAF,
                 tile: int = TILE):
        lib = nat.load()
        xy = np.ascontiguousarray(vertices, dtype=np.float64)
        nb_ptr = np.ascontiguousarray(nb_ptr, dtype=np.int64)
        nb_idx = np.ascontiguousarray(nb_idx, dtype=np.int64)
        isb = np.ascontiguousarray(is_boundary, dtype=np.uint8)
        h = ctypes.c_void_p()
        rc = lib.pf_nd_plan_build(len(xy), xy.ctypes.data, nb_ptr.ctypes.data,
                                  nb_idx.ctypes.data, isb.ctypes.data, int(leaf), int(tile),
                                  ctypes.byref(h))
        if rc != 0:
            raise NativeError(rc, "pf_nd_plan_build: " + lib.pf_last_error().decode())
        try:
            for names, dt in ((_I32, np.int32), (_I64, np.int64)):
                for name in names:
                    ln = lib.pf_nd_plan_array(h, name.encode(), None)
                    if ln < 0:
                        raise NativeError(-1, lib.pf_last_error().decode())
                    arr = np.empty(ln, dtype=dt)
                    lib.pf_nd_plan_array(h, name.encode(), arr.ctypes.data)
                    setattr(self, name, arr)
            st = np.zeros(len(_STATS))
            nat.call("pf_nd_plan_stats", h, st.ctypes.data)
        finally:
            lib.pf_nd_plan_free(h)
        self.stats = {k: (float(v) if k.startswith("flops") else int(v))
                      for k, v in zip(_STATS, st)}
        self.n, self.m, self.k = self.stats["n"], self.stats["m"], self.stats["k"]
        self.nodes = self.stats["nodes"]
        self.ntiles = self.stats["ntiles"]
        self.tile = self.stats["tile"]
        self.levels = [self.level_nodes[self.level_ptr[h]:self.level_ptr[h + 1]]
                       for h in range(len(self.level_ptr) - 1)]

    @classmethod
    def from_mesh(cls, mesh, leaf: int = LEAF, tile: int = TILE) -> "NdPlan":
        nb_ptr, nb_idx, isb = mesh_topology(mesh)
        return cls(mesh.vertices, nb_ptr, nb_idx, isb, leaf=leaf, tile=tile)


# ------------------------------------------------------------------ device --
class PfMfPlan(ctypes.Structure):
    """ctypes mirror of pf_mf_plan_t (include/pathfield_b200.h)."""
    _PTRS = ("c0", "cn", "rn", "fn", "foff", "ch_ptr", "ch_idx", "r_ptr", "r_orig",
             "relmap_off", "relmap", "a_ptr", "a_dst", "a_src", "b_ptr", "b_row", "b_col",
             "b_src", "act_tile", "act_voff", "tile_item", "perm_orig", "mt_off", "m_off",
             "rowoff")
    _fields_ = [(name, ctypes.c_void_p) for name in _PTRS] + [
        ("nodes", ctypes.c_int64), ("ntiles", ctypes.c_int64), ("k", ctypes.c_int64),
        ("tile", ctypes.c_int32), ("pad_", ctypes.c_int32)]


def _u64_to_f64(x: int) -> float:
    return float(np.array([x], dtype=np.uint64).view(np.float64)[0])


def _ranges(ptr, nodes):
    """Concatenated arange(ptr[s], ptr[s+1]) over `nodes` (and the owner of each)."""
    lo, hi = ptr[nodes], ptr[nodes + 1]
    cnt = hi - lo
    owner = np.repeat(nodes, cnt)
    idx = np.repeat(lo - (np.cumsum(cnt) - cnt), cnt) + np.arange(cnt.sum())
    return owner, idx


class DevicePoisson:
    """The device pipeline of one mesh: Laplacian, plan, factor, solves.

    ``laplacian()`` and ``factor()`` (L, then the explicit front inverses Mt
    and M) are cached; ``solve()`` writes a fresh P every call.
    """

    GEMM_TARGET = 8 * 148  # CTAs per backward level before column blocks are split
    SPLIT_BELOW = 148      # levels with fewer fronts factor each front over many CTAs

    def __init__(self, mesh, leaf: int = LEAF, device=None):
        from . import _device as dev
        t = dev.require_cuda()
        self.mesh = mesh
        self.device = (t.device(device) if device is not None
                       else t.device("cuda", t.cuda.current_device()))
        nb_ptr, nb_idx, isb_h = mesh_topology(mesh)
        tod = lambda a, dt: t.from_numpy(np.array(a, dtype=dt)).to(self.device)  # noqa: E731
        # device mesh arrays of the assembly (any TriMesh-like object: vertices,
        # triangles as stored, boundary_vertices)
        self.dm = type("DevMesh", (), {})()
        self.dm.V = tod(mesh.vertices, np.float64)
        self.dm.T = tod(mesh.triangles, np.int32)
        self.dm.nt = len(mesh.triangles)
        self.dm.nb_ptr = tod(nb_ptr, np.int64)
        self.dm.nb_idx = tod(nb_idx, np.int32)
        self._nnz = int(nb_ptr[-1])
        self.plan = pl = NdPlan(mesh.vertices, nb_ptr, nb_idx, isb_h, leaf=leaf, tile=TILE)
        self.n, self.k = pl.n, pl.k
        self.stream = lambda: t.cuda.current_stream(self.device).cuda_stream
        c, f = pl.cn.astype(np.int64), pl.fn.astype(np.int64)
        ldc, ldf = (c + 15) // 16 * 16, (f + 15) // 16 * 16  # 128-byte rows
        mt_sz, m_sz = f * ldc, c * ldf
        self.mt_off = np.concatenate([[0], np.cumsum(mt_sz)]).astype(np.int64)
        self.m_off = np.concatenate([[0], np.cumsum(m_sz)]).astype(np.int64)
        arrays = {name: getattr(pl, name) for name in PfMfPlan._PTRS if hasattr(pl, name)}
        arrays["mt_off"], arrays["m_off"] = self.mt_off, self.m_off
        self._dev = {name: tod(a, a.dtype) for name, a in arrays.items()}
        self.struct = PfMfPlan(*[self._dev[name].data_ptr() if name in self._dev else None
                                 for name in PfMfPlan._PTRS],
                               pl.nodes, pl.ntiles, pl.k, pl.tile, 0)
        isb = np.zeros(pl.n, dtype=np.uint8)
        bnd = np.asarray(mesh.boundary_vertices, dtype=np.int64)
        isb[bnd] = 1
        bcol = -np.ones(pl.n, dtype=np.int32)
        bcol[bnd] = np.arange(len(bnd), dtype=np.int32)
        self.boundary = bnd
        self.is_boundary = tod(isb, np.uint8)
        self.bcol = tod(bcol, np.int32)
        # ---- launch lists ------------------------------------------------
        self.levels = [tod(lv, np.int32) for lv in pl.levels]
        # (max f, max c, split) per level: few fronts -> every step over many CTAs
        self.level_shape = [(int(f[lv].max()) if len(lv) else 0,
                             int(c[lv].max()) if len(lv) else 0,
                             int(len(lv) < self.SPLIT_BELOW)) for lv in pl.levels]
        all_nodes = np.arange(pl.nodes, dtype=np.int64)
        ct = (c + 31) // 32
        inv_node = np.repeat(all_nodes, ct)
        inv_ct = np.arange(ct.sum()) - np.repeat(np.cumsum(ct) - ct, ct)
        # longest items first (an item sweeps rows 32*ct .. f of its front): the
        # top separators' CTAs would otherwise start last and form the tail
        work = (f[inv_node] - 32 * inv_ct) * (c[inv_node] - 32 * inv_ct)
        o = np.argsort(-work, kind="stable")
        inv_node, inv_ct = inv_node[o], inv_ct[o]
        big_first = all_nodes[np.argsort(-(c * f), kind="stable")]
        self.inv = (tod(inv_node, np.int32), tod(inv_ct, np.int32), len(inv_node),
                    tod(big_first, np.int32))
        self.fwd, wmax = [], 1
        for lv in pl.levels:
            lv = lv.astype(np.int64)
            node, item = _ranges(pl.act_ptr, lv)
            fi = f[node]
            woff = (np.cumsum(fi * TILE) - fi * TILE).astype(np.int64)
            wmax = max(wmax, int((fi * TILE).sum()))
            rb = (fi + 31) // 32
            g_node = np.repeat(node, rb)
            g_item = np.repeat(item, rb)
            g_woff = np.repeat(woff, rb)
            g_rb = np.arange(rb.sum()) - np.repeat(np.cumsum(rb) - rb, rb)
            self.fwd.append((tod(node, np.int32), tod(item, np.int64), tod(woff, np.int64),
                             len(node), tod(g_node, np.int32), tod(g_item, np.int64),
                             tod(g_woff, np.int64), tod(g_rb, np.int32), len(g_node)))
        self.w_total = wmax
        self._tod, self._c, self._f = tod, c, f
        self.bwd = self._bwd_lists(None)
        # host copies for the row-slab build (pf_mf_plan_t.rowoff)
        self._nb_host = (nb_ptr, nb_idx)
        self._isb_host = isb
        self._slabs: dict = {}
        self._lap = None
        self._F = None
        self._bufs = None

    def _bwd_lists(self, need):
        """Per-level backward launch lists (node, C-row block, column-block
        range), optionally restricted to the fronts in the boolean mask `need`."""
        pl, c, f, tod = self.plan, self._c, self._f, self._tod
        out = []
        nblk = (pl.ntiles + 1) // 2  # 128-column blocks (pairs of plan tiles)
        for lv in pl.levels:
            lv = lv.astype(np.int64)
            lv = lv[c[lv] > 0]
            if need is not None:
                lv = lv[need[lv]]
            # C-row block of the level: the smallest of 8/16/32/64 covering most
            # of its separators (the 90th percentile), larger ones in blocks
            cq = int(np.percentile(c[lv], 90)) if len(lv) else 1
            nbr = next(x for x in (8, 16, 32, 64) if x >= min(cq, 64))
            rb = (c[lv] + nbr - 1) // nbr
            blocks = int(rb.sum())
            chunks = int(min(nblk, max(1, -(-self.GEMM_TARGET // max(blocks, 1)))))
            step = -(-nblk // chunks)
            cb0 = np.arange(0, nblk, step, dtype=np.int64)
            cb1 = np.minimum(cb0 + step, nblk)
            nodes = np.repeat(lv, rb)
            rbi = np.arange(blocks) - np.repeat(np.cumsum(rb) - rb, rb)
            nn = len(nodes)
            out.append((tod(np.repeat(nodes, len(cb0)), np.int32),
                        tod(np.repeat(rbi, len(cb0)), np.int32),
                        tod(np.tile(cb0, nn), np.int32), tod(np.tile(cb1, nn), np.int32),
                        nn * len(cb0), int(f[lv].max()) if len(lv) else 1, int(step), nbr))
        return out

    def slab_plan(self, row0: int, rows: int) -> dict:
        """What a rank owning rows [row0, row0 + rows) of P computes (§8e /
        §8f-1: P row slabs written straight into each GPU's shard): the
        backward of every front holding a slab row, a row of the slab's 1-ring
        (the residual reads it) or an ancestor's row (X_R of a descendant);
        per-vertex output offsets — slab rows first, the other needed rows in
        scratch rows after them — and the slab's interior rows in
        nested-dissection order (the residual's walk)."""
        key = (int(row0), int(rows))
        hit = self._slabs.get(key)
        if hit is not None:
            return hit
        pl, tod = self.plan, self._tod
        ld = round_up_cols(self.k)
        nb_ptr, nb_idx = self._nb_host
        need, rowoff, extra = slab_needs(pl, nb_ptr, nb_idx, self._isb_host, row0, rows, ld)
        in_slab_pos = (pl.perm_orig >= row0) & (pl.perm_orig < row0 + rows)
        hit = {"need": need, "rowoff": tod(rowoff, np.int64), "scratch_rows": int(extra),
               "order": tod(pl.perm_orig[in_slab_pos], np.int32),
               "count": int(in_slab_pos.sum()), "bwd": self._bwd_lists(need),
               "fronts": int(need.sum())}
        st = PfMfPlan()
        ctypes.pointer(st)[0] = self.struct
        st.rowoff = hit["rowoff"].data_ptr()
        hit["struct"] = st
        self._slabs[key] = hit
        return hit

    # -- laplacian.py:91-134 ---------------------------------------------
    def laplacian(self):
        """(off, diag) device tensors: Lc in neighbour-CSR order, bitwise the reference's."""
        if self._lap is None:
            from . import _device as dev
            from .errors import DegenerateGeometryError
            t = dev.torch()
            dm = self.dm
            nnz = int(self.plan_nnz())
            off = t.empty(max(nnz, 1), dtype=t.float64, device=self.device)
            diag = t.empty(self.n, dtype=t.float64, device=self.device)
            bad = t.empty(1, dtype=t.int64, device=self.device)
            nat.call("pf_cotan_laplacian_f64", dm.V.data_ptr(), dm.T.data_ptr(), dm.nt,
                     dm.nb_ptr.data_ptr(), dm.nb_idx.data_ptr(), self.n, nnz, off.data_ptr(),
                     diag.data_ptr(), bad.data_ptr(), self.stream())
            b = int(bad.item())
            if b != np.iinfo(np.int64).max:
                raise DegenerateGeometryError(f"triangle {b} has a 0/pi angle")
            self._lap = (off, diag)
        return self._lap

    def plan_nnz(self) -> int:
        return self._nnz

    # -- laplacian.py:29-45 (splu of -Lc_II) -------------------------------
    def factor(self):
        """Multifrontal Cholesky of -Lc_II and the explicit front inverses Mt
        on the device (cached).  Returns Mt."""
        if self._F is None:
            from . import _device as dev
            from .errors import FactorizationError
            t = dev.torch()
            off, diag = self.laplacian()
            if self._bufs is None:  # kept across refactorisations (pads of Mt stay 0)
                self._bufs = (
                    t.empty(max(self.plan.stats["f_total"], 1), dtype=t.float64,
                            device=self.device),
                    t.zeros(max(int(self.mt_off[-1]), 1), dtype=t.float64, device=self.device))
            F, Mt = self._bufs
            err = t.zeros(1, dtype=t.int32, device=self.device)
            s = self.stream()
            for lv, (mf, mc, split) in zip(self.levels, self.level_shape):
                nat.call("pf_mf_factor_level", ctypes.addressof(self.struct), off.data_ptr(),
                         diag.data_ptr(), lv.data_ptr(), lv.numel(), mf, mc, split,
                         F.data_ptr(), err.data_ptr(), s)
            inode, ict, icnt, nodes = self.inv
            nat.call("pf_mf_inverse", ctypes.addressof(self.struct), F.data_ptr(),
                     inode.data_ptr(), ict.data_ptr(), icnt, nodes.data_ptr(), nodes.numel(),
                     Mt.data_ptr(), None, s)  # the solves read Mt (no transpose)
            if int(err.item()):
                raise FactorizationError(
                    "interior block is not positive definite after negation "
                    "(severely non-Delaunay mesh)")
            self._F = Mt
        return self._F

    # -- solvers.py:278-303 ------------------------------------------------
    def solve(self, P_out=None, events: dict | None = None, slab=None, fuse_h: bool = False):
        """P (device, n x round_up(k, 64) FP64, pads zero) with the reference's
        diagnostics.  Returns (P, residual, row_sum_error).  `events`, if given,
        receives CUDA events bracketing the forward / backward / diagnostics
        phases on the launch stream.  `slab = (row0, rows)` builds only rows
        [row0, row0 + rows) (the rank's shard; bitwise the same rows as the
        whole build): the returned P is (rows, ld) and the diagnostics cover
        the slab (the max over ranks is the whole P's).  `fuse_h` also
        computes the KL negentropy H and min P in the finalize pass (K1: one
        FP64 log per entry, worth it only when a KL field follows —
        device_kernel() sets it)."""
        from . import _device as dev
        t = dev.torch()
        mark = (lambda name: events.setdefault(name, t.cuda.Event(enable_timing=True)).record(
            t.cuda.current_stream(self.device))) if events is not None else (lambda name: None)
        off, diag = self.laplacian()
        Mt = self.factor()
        ld = round_up_cols(self.k)
        if slab is None:
            row0, rows, extra = 0, self.n, 0
            st, bwd, rowoff = self.struct, self.bwd, None
            order, count = self._dev["perm_orig"], self.plan.m
        else:
            row0, rows = int(slab[0]), int(slab[1])
            sp = self.slab_plan(row0, rows)
            st, bwd, rowoff = sp["struct"], sp["bwd"], sp["rowoff"]
            order, count, extra = sp["order"], sp["count"], sp["scratch_rows"]
        want = rows + extra
        if P_out is not None and (P_out.stride(0) != ld or P_out.shape[0] < want):
            raise ValueError(f"P_out must be ({want}, {ld}) row-major")
        Pbuf = P_out if P_out is not None else t.empty((want, ld), dtype=t.float64,
                                                       device=self.device)
        O = t.empty(max(self.plan.stats["v_total"], 1), dtype=t.float64, device=self.device)
        Wb = t.empty(self.w_total, dtype=t.float64, device=self.device)
        s = self.stream()
        ps = ctypes.addressof(st)
        mark("fwd0")
        for (an, ai, aw, acnt, gn, gi, gw, grb, gcnt) in self.fwd:
            nat.call("pf_mf_forward_level", ps, Mt.data_ptr(), off.data_ptr(), an.data_ptr(),
                     ai.data_ptr(), aw.data_ptr(), acnt, gn.data_ptr(), gi.data_ptr(),
                     gw.data_ptr(), grb.data_ptr(), gcnt, Wb.data_ptr(), O.data_ptr(), s)
        mark("bwd0")
        for nodes, rb, cb0, cb1, cnt, maxf, ncb, nbr in reversed(bwd):
            if cnt == 0:  # a slab build may need no front of a level
                continue
            nat.call("pf_mf_backward_level", ps, Mt.data_ptr(), O.data_ptr(), nodes.data_ptr(),
                     rb.data_ptr(), cb0.data_ptr(), cb1.data_ptr(), cnt, maxf, ncb, nbr,
                     Pbuf.data_ptr(), ld, s)
        mark("bwd1")
        mx = t.zeros(4, dtype=t.int64, device=self.device)  # residual, row sums, neg flag
        dm = self.dm
        nrow = self._residual_table(ld, rowoff)
        # fused K1: the KL negentropy per row (clamp 1e-300) and min(P), so the
        # first field on this P does not stream it again
        H = t.empty(rows, dtype=t.float64, device=self.device) if fuse_h else None
        mn = t.full((1,), float("inf"), dtype=t.float64, device=self.device) if fuse_h else None
        resargs = (Pbuf.data_ptr(), ld, self.k, order.data_ptr(), count, nat.ptr(rowoff),
                   dm.nb_ptr.data_ptr(), nrow.data_ptr(), off.data_ptr(), diag.data_ptr())
        finargs = (Pbuf.data_ptr(), ld, row0, rows, self.k, self.is_boundary.data_ptr(),
                   self.bcol.data_ptr())
        if fuse_h:  # the K1 pass reads every entry anyway: it also finalizes
            nat.call("pf_poisson_residual", *resargs, mx.data_ptr(), s)
            nat.call("pf_poisson_finalize", *finargs, KL_CLAMP, nat.ptr(H), nat.ptr(mn),
                     mx.data_ptr() + 8, s)
        else:  # row sums ride on the residual's read of each row: no second pass
            part = t.empty(max(rows * (-(-self.k // RESIDUAL_COLS)), 1), dtype=t.float64,
                           device=self.device)
            nat.call("pf_poisson_residual_rows", *resargs, part.data_ptr(), mx.data_ptr(), s)
            nat.call("pf_poisson_finalize_rows", *finargs, part.data_ptr(), mx.data_ptr() + 8, s)
        self.last_H, self.last_min = H, mn
        mark("end")
        del O, Wb
        r = mx.cpu().numpy().astype(np.uint64)
        if r[2]:  # a negative entry: the reference's clip may apply (full finalize)
            mx[1] = 0
            nat.call("pf_poisson_finalize", *finargs, KL_CLAMP, None, None, mx.data_ptr() + 8, s)
            r = mx.cpu().numpy().astype(np.uint64)
        residual = _u64_to_f64(int(r[0])) if count else 0.0
        return Pbuf[:rows], residual, _u64_to_f64(int(r[1]))

    def _residual_table(self, ld: int, rowoff=None):
        """Per neighbour entry: the output offset of an interior neighbour's row
        or -1 - the boundary column (pf_poisson_residual_table), cached per
        (ld, row-offset table)."""
        key = (ld, None if rowoff is None else rowoff.data_ptr())
        tabs = getattr(self, "_rtabs", None)
        if tabs is None:
            tabs = self._rtabs = {}
        hit = tabs.get(key)
        if hit is None:
            from . import _device as dev
            t = dev.torch()
            hit = t.empty(max(self._nnz, 1), dtype=t.int64, device=self.device)
            nat.call("pf_poisson_residual_table", self.dm.nb_idx.data_ptr(), self._nnz,
                     self.is_boundary.data_ptr(), self.bcol.data_ptr(), ld, nat.ptr(rowoff),
                     hit.data_ptr(), self.stream())
            tabs[key] = hit
        return hit

    def solve_flops(self) -> dict:
        """Algorithmic FP64 work of the solves (SURVEY §8d convention): the
        triangular-solve count sum_s (c^2 + 2 c r) per column for each of the
        backward (all k columns) and the forward (its active 64-column tiles),
        plus what the backward GEMM issues (2 c f per column, less the
        skipped zero Y rows of unreached tiles)."""
        pl = self.plan
        c = pl.cn.astype(np.float64)
        r = pl.rn.astype(np.float64)
        f = pl.fn.astype(np.float64)
        per_col = c * c + 2 * c * r
        k = float(self.k)
        act = np.diff(pl.act_ptr).astype(np.float64)
        issued = 0.0
        nblk = (pl.ntiles + 1) // 2
        ti = pl.tile_item.reshape(pl.nodes, pl.ntiles)
        if pl.ntiles % 2:
            ti = np.concatenate([ti, -np.ones((pl.nodes, 1), np.int64)], axis=1)
        blk_active = (ti.reshape(pl.nodes, nblk, 2) >= 0).any(axis=2)
        width = np.minimum(128.0, k - 128.0 * np.arange(nblk))
        kskip = np.floor(c / 16) * 16
        keff = np.where(blk_active, f[:, None], (f - kskip)[:, None])
        issued = float((2.0 * c[:, None] * keff * width[None, :]).sum())
        return {"backward": float(per_col.sum() * k),
                "forward": float((per_col * act).sum() * TILE),
                "backward_issued": issued}

    def device_kernel(self, P=None, slab=None):
        """Solve and wrap P (or the row slab (row0, rows)) as a DeviceKernel
        (the hot path's input; a slab is a parallel.ShardedField shard)."""
        from . import _device as dev
        P, residual, rse = self.solve(P, slab=slab, fuse_h=True)
        row0 = 0 if slab is None else int(slab[0])
        dk = dev.DeviceKernel(None, self.boundary, n=self.n, k=self.k, P_dev=P, row0=row0,
                              rows=P.shape[0])
        dk.residual, dk.row_sum_error = residual, rse
        dk._H[KL_CLAMP] = self.last_H     # K1, fused into the build's finalize pass
        dk._min = self.last_min
        return dk


def round_up_cols(k: int) -> int:
    """Row stride of a device-built P: 64-column tiles never cross a row end."""
    return (k + 63) // 64 * 64


class LaplacianSet:
    """Mirror of ``pathfield.laplacian.LaplacianSet`` (laplacian.py:63-88) whose
    matrix lives on the device; ``lc`` materialises the scipy CSR (bitwise the
    reference's) on first access."""

    def __init__(self, mesh, solver: DevicePoisson):
        self.mesh = mesh
        self.solver = solver
        self.interior = np.asarray(mesh.interior_vertices).copy()
        self.boundary = np.asarray(mesh.boundary_vertices).copy()
        self._lc = None

    @property
    def lc(self):
        if self._lc is None:
            import scipy.sparse as sp
            off, diag = self.solver.laplacian()
            dm = self.solver.dm
            nb_ptr = dm.nb_ptr.cpu().numpy()
            nb_idx = dm.nb_idx.cpu().numpy().astype(np.int64)
            n = self.solver.n
            m = sp.csr_matrix((off.cpu().numpy()[:len(nb_idx)], nb_idx, nb_ptr), shape=(n, n))
            self._lc = (m + sp.diags(diag.cpu().numpy())).tocsr()
        return self._lc

    @property
    def lc_ii(self):
        return self.lc[self.interior][:, self.interior]

    @property
    def lc_ib(self):
        return self.lc[self.interior][:, self.boundary]


def assemble_cotan(mesh, leaf: int = LEAF) -> LaplacianSet:
    """laplacian.py:91-134 on the device (the matrix stays resident)."""
    solver = DevicePoisson(mesh, leaf=leaf)
    solver.laplacian()
    return LaplacianSet(mesh, solver)


def poisson_kernel_device(ls_or_mesh, leaf: int = LEAF):
    """P on the device only (no host copy): a DeviceKernel with ``residual``
    and ``row_sum_error`` attributes."""
    solver = (ls_or_mesh.solver if isinstance(ls_or_mesh, LaplacianSet)
              else DevicePoisson(ls_or_mesh, leaf=leaf))
    return solver.device_kernel()


_STAGING: dict = {}
# dense_to_host holds this for the whole copy: the staging buffers are shared
# per (rows, ld), and concurrent DomainContext builds (domain.py:45-61 locks
# only its own context) may copy P to the host from several threads at once
_STAGING_LOCK = threading.Lock()


def _staging(t, rows: int, ld: int):
    """Two persistent pinned staging buffers per (rows, ld) (a fresh pinned
    allocation costs ~0.3 ms per MB).  Callers hold _STAGING_LOCK."""
    key = (rows, ld)
    bufs = _STAGING.get(key)
    if bufs is None:
        bufs = _STAGING[key] = [t.empty((rows, ld), dtype=t.float64, pin_memory=True)
                                for _ in range(2)]
    return bufs


def dense_to_host(P, n: int, k: int, chunk_bytes: int = 64 << 20,
                  threads: int | None = None) -> np.ndarray:
    """Host (n, k) copy of a device P (row stride >= k): ~64 MB row chunks are
    copied D2H into two alternating pinned buffers while a thread pool
    scatters the previous chunk into the numpy result (first-touching its
    pages in parallel; a direct pageable copy of a strided 33 GB matrix runs
    at a fraction of the PCIe rate)."""
    from . import _device as dev
    t = dev.torch()
    out = np.empty((n, k))
    if n == 0:
        return out
    with _STAGING_LOCK:
        return _dense_to_host_locked(t, P, out, n, k, chunk_bytes, threads)


def _dense_to_host_locked(t, P, out, n, k, chunk_bytes, threads):
    import os
    from concurrent.futures import ThreadPoolExecutor
    ld = P.stride(0)
    rows = max(1, min(n, chunk_bytes // (8 * ld)))
    bufs = _staging(t, rows, ld)
    evs = [t.cuda.Event() for _ in range(2)]
    stream = t.cuda.Stream(P.device)
    stream.wait_stream(t.cuda.current_stream(P.device))
    threads = threads or max(1, min(16, os.cpu_count() or 1))
    pool = ThreadPoolExecutor(threads)

    def scatter(buf, a, b):
        src = buf.numpy()
        step = -(-(b - a) // threads)
        futs = [pool.submit(np.copyto, out[a + i:min(b, a + i + step)],
                            src[i:min(b - a, i + step), :k]) for i in range(0, b - a, step)]
        for fu in futs:
            fu.result()

    pending = None
    try:
        for ci, a in enumerate(range(0, n, rows)):
            b = min(n, a + rows)
            j = ci & 1
            with t.cuda.stream(stream):
                bufs[j][:b - a].copy_(P[a:b], non_blocking=True)
                evs[j].record(stream)
            if pending is not None:
                pj, pa, pb = pending
                evs[pj].synchronize()
                scatter(bufs[pj], pa, pb)
            pending = (j, a, b)
        pj, pa, pb = pending
        evs[pj].synchronize()
        scatter(bufs[pj], pa, pb)
    finally:
        pool.shutdown()
    return out


def poisson_kernel(ls, settings=None, kernel_type=None):
    """solvers.py:278-303: the PoissonKernel of a LaplacianSet (this package's
    or the reference's: only ``.mesh`` is read) or of a mesh.

    P is computed on the device and stays resident there (registered as the
    device mirror of the returned ``dense``, so the hot path never re-uploads
    it); ``dense`` is its host copy, as the reference's return type requires.
    ``kernel_type`` builds the reference's own PoissonKernel class in drop-in
    mode (integration.py)."""
    import warnings
    from . import _device as dev
    from .config import DEFAULTS
    from .solvers import PoissonKernel, PrecisionWarning
    settings = settings or DEFAULTS
    mesh = getattr(ls, "mesh", ls)
    solver = ls.solver if isinstance(ls, LaplacianSet) else DevicePoisson(mesh)
    dk = solver.device_kernel()
    dense = dense_to_host(dk.P, dk.n, dk.k)
    if dk.residual > settings.residual_warn:
        warnings.warn(f"poisson kernel residual {dk.residual:.2e}", PrecisionWarning,
                      stacklevel=2)
    cls = kernel_type or PoissonKernel
    pk = cls(dense, np.asarray(mesh.boundary_vertices, dtype=np.int64).copy(), dk.residual,
             dk.row_sum_error)
    dev.register(pk.dense, dk)
    return pk


def dk_boundary(ls_or_mesh):
    mesh = ls_or_mesh.mesh if isinstance(ls_or_mesh, LaplacianSet) else ls_or_mesh
    return np.asarray(mesh.boundary_vertices, dtype=np.int64)
