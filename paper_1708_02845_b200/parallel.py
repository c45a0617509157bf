"""Row-sharded multi-GPU evaluation: one process per GPU.

Every output row q of a divergence field depends only on row q of P and on
the target row, so the GPUs of one box own contiguous row slabs
(dense: balanced by row count; CSR: balanced by nnz) and evaluate them with
the single-GPU kernels unchanged — the N-GPU field is bitwise the 1-GPU
field.  The data path has exactly two exchanges, both NCCL over NVLink,
issued through the C ABI (``pf_nccl_*``, :class:`NcclComm`) on the launch
stream:

* the target row P[t, :] (k FP64) is broadcast from its owner rank
  (33 KB at k = 4,102);
* the finished field slabs are all-gathered (n FP64) only when a tracer on
  every rank needs the whole field (:meth:`ShardedField.trace`).

plus two word-sized reductions that keep the single-process contract of
``dv_field`` (``divergence.py:157-183``) on every rank: the ``clamped`` flag
word is max-reduced (an interior row of ANY slab can fire it) and, for
``clamp <= 0``, the slab minima are min-reduced before the domain check, so
every rank raises :class:`DivergenceDomainError` or none does.

Batched targets (K7) come in both layouts the survey
names: :meth:`ShardedField.field_batch` keeps P row-sharded and assembles
the T target rows with one all-reduce (each row is its owner's values plus
zeros: exact), then every rank contracts its slab; :func:`field_batch_by_targets`
replicates P (32.8 GB at C4 fits one B200) and partitions the targets, with
no data-path collective at all, and :func:`trace_batch` traces each path on
the rank that owns its target's column (C5: no field exchange either).

``torch.distributed`` is the control plane only (rendezvous, the NCCL unique
id, barriers); on CPU tensors (the gloo tests of tests/test_parallel.py) the
same host logic runs over the process group (:class:`GroupComm`), with the
slab computation swapped for the oracle inside those tests only — the
product's slab computation is always the CUDA kernels.
"""

from __future__ import annotations

import ctypes

import numpy as np

from . import _device as dev
from .errors import DivergenceDomainError, InvalidTargetError


def partition_rows(n: int, world: int) -> list[tuple[int, int]]:
    """Contiguous, balanced row slabs [r0, r1) for `world` ranks (sizes differ by <= 1)."""
    base, extra = divmod(n, world)
    out, r0 = [], 0
    for r in range(world):
        r1 = r0 + base + (1 if r < extra else 0)
        out.append((r0, r1))
        r0 = r1
    return out


def partition_by_weight(weights, world: int) -> list[tuple[int, int]]:
    """Contiguous slabs balanced by a per-row weight (CSR: nnz per row + 1 per row)."""
    w = np.asarray(weights, dtype=np.float64) + 1.0
    cum = np.concatenate([[0.0], np.cumsum(w)])
    total = cum[-1]
    cuts = [0]
    for r in range(1, world):
        cuts.append(int(np.searchsorted(cum, total * r / world, side="left")))
    cuts.append(len(w))
    cuts = np.maximum.accumulate(np.array(cuts))
    return [(int(cuts[r]), int(cuts[r + 1])) for r in range(world)]


def owner_of(row: int, bounds: list[tuple[int, int]]) -> int:
    """Rank whose slab holds global row `row` (InvalidTargetError outside every slab)."""
    for r, (a, b) in enumerate(bounds):
        if a <= row < b:
            return r
    raise InvalidTargetError(f"target {row} out of range")


# ---------------------------------------------------------------------------
# Collectives
# ---------------------------------------------------------------------------

_PF_T = {"torch.uint8": 0, "torch.int32": 1, "torch.int64": 2, "torch.float64": 3}
_PF_OP = {"sum": 0, "max": 1, "min": 2}


class NcclComm:
    """NCCL communicator of the GPU data plane, driven through the C ABI.

    Rank 0 draws the unique id (``pf_nccl_unique_id``) and the control-plane
    process group ``dist`` hands it to every rank; each collective is
    enqueued on the current torch stream of the device, in place where the
    operation allows."""

    def __init__(self, dist, device):
        from . import _native as nat
        t = dev.require_cuda()
        self.nat, self.t = nat, t
        self.device = t.device(device)
        self.rank, self.world = dist.get_rank(), dist.get_world_size()
        nat.call("pf_nccl_load", _torch_nccl_path())
        uid = ctypes.create_string_buffer(128)
        if self.rank == 0:
            nat.call("pf_nccl_unique_id", uid)
        box = [bytes(uid.raw)]
        dist.broadcast_object_list(box, src=0)
        uid = ctypes.create_string_buffer(box[0], 128)
        h = ctypes.c_void_p(0)
        nat.call("pf_nccl_comm_init", self.world, uid, self.rank, self.device.index,
                 ctypes.byref(h))
        self.handle = h.value

    def _stream(self):
        return self.t.cuda.current_stream(self.device).cuda_stream

    def broadcast(self, x, src: int):
        self.nat.call("pf_nccl_broadcast", self.handle, x.data_ptr(), x.numel(),
                      _PF_T[str(x.dtype)], int(src), self._stream())

    def all_gather(self, x):
        """(world * x.numel(),) tensor: every rank's `x`, in rank order."""
        out = self.t.empty(self.world * x.numel(), dtype=x.dtype, device=x.device)
        self.nat.call("pf_nccl_all_gather", self.handle, x.data_ptr(), out.data_ptr(), x.numel(),
                      _PF_T[str(x.dtype)], self._stream())
        return out

    def all_reduce(self, x, op: str = "sum"):
        self.nat.call("pf_nccl_all_reduce", self.handle, x.data_ptr(), x.data_ptr(), x.numel(),
                      _PF_T[str(x.dtype)], _PF_OP[op], self._stream())

    def close(self):
        if self.handle:
            self.nat.call("pf_nccl_comm_destroy", self.handle)
            self.handle = None


class GroupComm:
    """The same collectives over a torch.distributed process group (CPU
    tensors: the host-logic tests on gloo)."""

    def __init__(self, dist):
        self.dist = dist
        self.rank, self.world = dist.get_rank(), dist.get_world_size()

    def broadcast(self, x, src: int):
        self.dist.broadcast(x, src=src)

    def all_gather(self, x):
        t = dev.torch()
        parts = [t.empty_like(x) for _ in range(self.world)]
        self.dist.all_gather(parts, x.contiguous())
        return t.cat([p.reshape(-1) for p in parts])

    def all_reduce(self, x, op: str = "sum"):
        ops = {"sum": self.dist.ReduceOp.SUM, "max": self.dist.ReduceOp.MAX,
               "min": self.dist.ReduceOp.MIN}
        self.dist.all_reduce(x, op=ops[op])

    def close(self):
        pass


def make_comm(dist, device):
    """NCCL (pf_nccl_*) for CUDA devices; the process group for CPU tensors."""
    t = dev.torch()
    if device is not None and t.device(device).type == "cuda":
        return NcclComm(dist, device)
    return GroupComm(dist)


def _torch_nccl_path() -> bytes | None:
    """Path of the NCCL library torch ships (used only if none is loaded yet)."""
    try:
        import nvidia.nccl  # type: ignore
        from pathlib import Path
        p = Path(list(nvidia.nccl.__path__)[0]) / "lib" / "libnccl.so.2"
        return str(p).encode() if p.exists() else None
    except Exception:
        return None


# ---------------------------------------------------------------------------
# Fields over row slabs
# ---------------------------------------------------------------------------

class SlabField:
    """This rank's slab of a divergence field (the sharded ``ScalarField``).

    ``values`` is the slab's device tensor (rows [row0, row0 + rows) of the
    global field); ``precision_flags`` are the WHOLE field's flags (the
    ``clamped`` word was max-reduced over the ranks before this object was
    made), read from the device on first access."""

    def __init__(self, values, flag_word, row0: int, kind: str, target: int, params: dict,
                 clamp: float):
        self.values, self._flag, self.row0 = values, flag_word, int(row0)
        self.kind, self.target, self.params, self._clamp = kind, int(target), params, clamp
        self.sign, self.residual = 1, None
        self._flags = None

    @property
    def rows(self) -> int:
        return int(self.values.numel())

    @property
    def precision_flags(self) -> tuple[str, ...]:
        if self._flags is None:
            fired = self._flag is not None and bool(int(self._flag.reshape(-1)[0].item()))
            self._flags = ("clamped",) if (fired and self._clamp > 0.0) else ()
        return self._flags


class ShardedField:
    """Per-rank driver of a row-sharded field evaluation.

    ``slab`` is this rank's :class:`~paper_1708_02845_b200._device.DeviceKernel`
    (rows ``bounds[rank]`` of the global P); ``dist`` the initialised
    ``torch.distributed`` module (the control plane); ``comm`` the data-plane
    collectives (default: NCCL through the C ABI on a CUDA device).
    """

    def __init__(self, slab, bounds, dist, device=None, comm=None):
        self.slab, self.bounds, self.dist = slab, bounds, dist
        self.rank = dist.get_rank()
        self.world = dist.get_world_size()
        self.device = device if device is not None else getattr(slab, "device", None)
        self.n = int(bounds[-1][1])
        a, b = bounds[self.rank]
        if (getattr(slab, "row0", a), getattr(slab, "rows", b - a)) != (a, b - a):
            raise ValueError("slab does not match this rank's partition")
        self.comm = comm if comm is not None else make_comm(dist, self.device)

    @classmethod
    def from_mesh(cls, mesh, dist, device=None, bounds=None, comm=None):
        """Build this rank's row slab of the Poisson kernel P straight into its
        shard: every rank factors -Lc_II and runs the forward
        solve (replicated, ~34 ms at C4), then runs the backward only for the
        fronts its rows, their 1-ring and their ancestors need
        (laplacian.DevicePoisson.slab_plan).  The slab is bitwise the rows of
        the single-GPU build; residual / row_sum_error are reduced with a max
        over ranks (exact).  Returns the ShardedField."""
        from . import laplacian as L
        t = dev.torch()
        world, rank = dist.get_world_size(), dist.get_rank()
        bounds = bounds or partition_rows(len(mesh.vertices), world)
        a, b = bounds[rank]
        dp = L.DevicePoisson(mesh, device=device)
        dk = dp.device_kernel(slab=(a, b - a))
        sf = cls(dk, bounds, dist, device=dk.device, comm=comm)
        diag = t.tensor([dk.residual, dk.row_sum_error], dtype=t.float64, device=dk.device)
        sf.comm.all_reduce(diag, "max")
        dk.residual, dk.row_sum_error = (float(x) for x in diag.cpu().numpy())
        sf.poisson = dp
        return sf

    def close(self):
        self.comm.close()

    # -- contract checks (divergence.py:157-165), identical on every rank ----
    def _check_target(self, p: int) -> int:
        p = int(p)
        if not 0 <= p < self.n:
            raise InvalidTargetError(f"target {p} out of range")
        return p

    def _clamp(self, clamp) -> float:
        """Kernel clamp; clamp <= 0 needs P > 0 on EVERY slab: the slab minima
        are min-reduced first so all ranks raise together (no rank is left
        waiting in a later collective)."""
        if clamp is not None and clamp > 0.0:
            return float(clamp)
        t = dev.torch()
        m = t.tensor([self.slab.min_value() if self.slab.rows else float("inf")],
                     dtype=t.float64, device=self.device)
        self.comm.all_reduce(m, "min")
        if float(m.item()) <= 0.0:
            raise DivergenceDomainError("zero kernel entries and clamping is disabled")
        return 0.0

    def target_row(self, p: int, k: int):
        """Broadcast P[p, :k] from its owner to every rank (the one data-path exchange)."""
        t = dev.torch()
        own = owner_of(p, self.bounds)
        if self.rank == own:
            row = self.slab.P[p - self.bounds[own][0], :k].contiguous()
        else:
            row = t.empty(k, dtype=t.float64, device=self.device)
        self.comm.broadcast(row, own)
        return row

    def field(self, fd, p: int, gather: bool = False, clamp=None, swap_order: bool = False):
        """The field to target p (divergence.py:154-187) over this rank's slab:
        a :class:`SlabField` whose ``precision_flags`` are the whole field's.
        With `gather`, the whole field as a host ``ScalarField`` on every rank."""
        p = self._check_target(p)
        c = self._clamp(fd.clamp if clamp is None else clamp)
        row = self.target_row(p, self.slab.k)
        vals, flag = _compute_slab(self.slab, fd, p, row, c, swap_order)
        self.comm.all_reduce(flag, "max")   # clamped fires if it fired on ANY slab
        params = dict(getattr(fd, "params", {}) or {})
        if swap_order:
            params["swap_order"] = True
        sf = SlabField(vals, flag, self.slab.row0, fd.name, p, params, c)
        return self.to_scalar_field(sf) if gather else sf

    def to_scalar_field(self, sf: SlabField):
        """All-gather a SlabField into the reference's host ``ScalarField``."""
        from .solvers import ScalarField
        full = self.gather(sf.values)
        host = full.cpu().numpy()
        return ScalarField(host, sf.kind, sf.target, sf.params, 1, None, sf.precision_flags)

    def sparse_field(self, fd, p: int, threshold: float | None = None, gather: bool = False):
        """This rank's slab of the sparse (CSR) field to target p (divergence.py:255-299).

        KL needs the target's dense log row: the dense row is broadcast as for
        :meth:`field`.  TV needs the target's sparsified row: its owner scatters it
        (K6 prep) and broadcasts the dense k-vector plus (S_p, dropped_p, nnz_p).
        CSR slabs should be partitioned with :func:`partition_by_weight` over nnz.
        Sparse pairs carry no flags (the reference's dv_pair_sparse has none).
        """
        import math
        t = dev.torch()
        p = self._check_target(p)
        n, k = self.n, self.slab.k
        thr = 1.0 / math.sqrt(n) if threshold is None else float(threshold)
        if thr < 0:
            raise ValueError("threshold must be nonnegative")
        if thr >= 1.0:
            raise ValueError(f"threshold {thr} >= 1 would empty rows")
        cut = thr / k
        from .divergence import _is_builtin
        if _is_builtin(fd, "kl"):
            payload = self.target_row(p, k)
        elif _is_builtin(fd, "tv"):
            own = owner_of(p, self.bounds)
            kp = k + (k & 1)
            payload = t.empty(kp + 4, dtype=t.float64, device=self.device)
            if self.rank == own:
                _sparse_tv_prep(self.slab, cut, thr == 0, p, payload)
            self.comm.broadcast(payload, own)
        else:
            raise NotImplementedError("sparse fields implement kl and tv")
        vals = _compute_sparse_slab(self.slab, fd, p, payload, cut, thr == 0)
        sf = SlabField(vals, None, self.slab.row0, fd.name, p,
                       dict(getattr(fd, "params", {}) or {}), 0.0)
        return self.to_scalar_field(sf) if gather else sf

    def target_rows(self, targets, k: int):
        """Rows P[targets, :k] on every rank: each rank fills the rows it owns and
        one all-reduce (sum) assembles them — exact, every other addend is 0."""
        t = dev.torch()
        targets = np.asarray(targets, dtype=np.int64).reshape(-1)
        rows = t.zeros((targets.size, k), dtype=t.float64, device=self.device)
        a, b = self.bounds[self.rank]
        mine = np.flatnonzero((targets >= a) & (targets < b))
        if mine.size:
            idx = t.from_numpy(targets[mine] - a).to(self.slab.P.device)
            rows[t.from_numpy(mine).to(rows.device)] = self.slab.P.index_select(0, idx)[:, :k].to(
                rows.device)
        self.comm.all_reduce(rows, "sum")
        return rows

    def field_batch(self, fd, targets, gather: bool = False, method: str = "auto",
                    clamp=None):
        """This rank's rows of the fields to T targets (rows x T, device) and the
        per-target ``clamped`` flags; all ranks' rows (n x T) if `gather`.

        KL runs K7 on the slab against the all-reduced target rows (SURVEY §8e
        item 3, row-sharded variant); the result is bitwise the single-GPU one.
        Other generators are T single-target :meth:`field` calls."""
        t = dev.torch()
        targets = np.asarray(targets, dtype=np.int64).reshape(-1)
        if targets.size and (targets.min() < 0 or targets.max() >= self.n):
            raise InvalidTargetError("target out of range")
        c = self._clamp(fd.clamp if clamp is None else clamp)
        from .divergence import _is_builtin
        if not _is_builtin(fd, "kl"):
            res = [self.field(fd, int(p), clamp=clamp) for p in targets]
            vals = (t.stack([r.values for r in res], dim=1) if res
                    else t.zeros((self.slab.rows, 0), dtype=t.float64, device=self.device))
            flags = np.array([bool(r.precision_flags) for r in res], dtype=bool)
        else:
            rows = self.target_rows(targets, self.slab.k)
            vals, flags = _compute_batch_slab(self.slab, fd, targets, rows, method, c)
            f = t.from_numpy(np.asarray(flags, dtype=np.int32)).to(self.device)
            self.comm.all_reduce(f, "max")
            flags = f.cpu().numpy().astype(bool)
        if not gather:
            return vals, flags
        return self.gather_rows(vals), flags

    def gather_rows(self, vals):
        """All-gather variable-size (rows x T) slabs into the (n x T) matrix."""
        t = dev.torch()
        T = vals.shape[1]
        sizes = [b - a for a, b in self.bounds]
        m = max(sizes)
        buf = t.zeros((m, T), dtype=vals.dtype, device=vals.device)
        buf[:vals.shape[0]] = vals
        parts = self.comm.all_gather(buf).reshape(self.world, m, T)
        return t.cat([parts[r, :sizes[r]] for r in range(self.world)])

    def gather(self, vals):
        """All-gather variable-size slabs into the full n-vector on every rank."""
        t = dev.torch()
        sizes = [b - a for a, b in self.bounds]
        m = max(sizes)
        if all(s == m for s in sizes):
            return self.comm.all_gather(vals.contiguous())
        buf = t.zeros(m, dtype=vals.dtype, device=vals.device)
        buf[:vals.numel()] = vals
        parts = self.comm.all_gather(buf).reshape(self.world, m)
        return t.cat([parts[r, :sizes[r]] for r in range(self.world)])

    def trace(self, mesh, fd, p: int, sources, settings=None, gather_paths: bool = False):
        """Trace `sources` down the field to target p (paths.py:292-307) with the
        sources partitioned over the ranks: the finished field slabs are
        all-gathered (the one place the north star allows it) and each rank
        traces its contiguous chunk of sources on its own copy of the field.
        Returns ``(source_indices, paths)`` for this rank, or with
        `gather_paths` the list of every path in source order on every rank."""
        from .config import DEFAULTS
        settings = settings or DEFAULTS
        p = self._check_target(p)
        sources = np.asarray(sources, dtype=np.int64).reshape(-1)
        _check_sources(sources, np.full(sources.size, p), self.n)
        sf = self.field(fd, p)
        full = self.gather(sf.values)
        a, b = partition_rows(sources.size, self.world)[self.rank]
        mine = np.arange(a, b)
        paths = _trace_local(mesh, full.reshape(1, -1), self.n, 1, np.array([p]), sources[mine],
                             None, settings)
        if not gather_paths:
            return mine, paths
        return _gather_paths(self.dist, sources.size, mine, paths)


def _check_sources(sources, targets_of, n):
    """paths.py:295-296 (source == target) and the source range, before any launch."""
    if sources.size and (sources.min() < 0 or sources.max() >= n):
        raise InvalidTargetError("source out of range")
    if np.any(sources == targets_of):
        raise InvalidTargetError("source equals target")


def _gather_paths(dist, total: int, mine, paths):
    """Every rank's (indices, paths) in global order (control-plane object gather)."""
    parts = [None] * dist.get_world_size()
    dist.all_gather_object(parts, (np.asarray(mine).tolist(), paths))
    out = [None] * total
    for idx, ps in parts:
        for i, pth in zip(idx, ps):
            out[i] = pth
    return out


def field_batch_by_targets(pk, fd, targets, dist, gather: bool = False, method: str = "auto",
                           clamp=None, comm=None):
    """Fields to T targets with the targets partitioned over the ranks and P
    replicated on every GPU (recommended: C5's 32.8 GB P
    fits each B200): rank r computes the n x T_r columns of its contiguous
    target chunk with K7 — no data-path collective.  Returns (this rank's
    columns (n x T_r, device), its flags, its target chunk), or with `gather`
    the full (n x T) matrix and flags on every rank."""
    t = dev.torch()
    targets = np.asarray(targets, dtype=np.int64).reshape(-1)
    world, rank = dist.get_world_size(), dist.get_rank()
    chunks = partition_rows(targets.size, world)
    a, b = chunks[rank]
    vals, flags = _local_batch(pk, fd, targets[a:b], clamp, method)
    if not gather:
        return vals, flags, targets[a:b]
    comm = comm if comm is not None else make_comm(dist, vals.device)
    n = vals.shape[0]
    m = max(e - s for s, e in chunks)
    buf = t.zeros((m, n), dtype=vals.dtype, device=vals.device)
    buf[:b - a] = vals.t()
    parts = comm.all_gather(buf).reshape(world, m, n)
    fl = t.zeros(m, dtype=t.int32, device=vals.device)
    fl[:b - a] = t.from_numpy(np.asarray(flags, dtype=np.int32)).to(vals.device)
    fparts = comm.all_gather(fl).reshape(world, m)
    full = t.cat([parts[r, :e - s] for r, (s, e) in enumerate(chunks)]).t()
    fall = t.cat([fparts[r, :e - s] for r, (s, e) in enumerate(chunks)]).cpu().numpy()
    return full, fall.astype(bool), targets


def trace_batch(mesh, pk, fd, targets, sources, field_of, dist, settings=None,
                method: str = "auto", clamp=None, gather_paths: bool = False,
                status_only: bool = False):
    """C5 on N GPUs (SURVEY §8e item 3, §8 a9 + a10): fields to T targets with
    the targets partitioned over the ranks (:func:`field_batch_by_targets`,
    P replicated) and each path p traced on the rank that owns its target
    ``targets[field_of[p]]``, straight from that rank's (n x T_r) batched
    output (``pf_trace_fields_f64``, no copy) — no field is exchanged.

    Every path equals ``triangle_descent(mesh, dv_field(pk, fd, targets[field_of[p]]),
    sources[p])``.  Returns ``(path_indices, paths)`` for this rank, or with
    `gather_paths` the list of every path in input order on every rank; with
    `status_only`, ``(path_indices, status codes, location counts)`` without
    building the host path objects (what a throughput measurement needs)."""
    from .config import DEFAULTS
    settings = settings or DEFAULTS
    targets = np.asarray(targets, dtype=np.int64).reshape(-1)
    sources = np.asarray(sources, dtype=np.int64).reshape(-1)
    field_of = np.asarray(field_of, dtype=np.int64).reshape(-1)
    n = len(mesh.vertices)
    if targets.size and (targets.min() < 0 or targets.max() >= n):
        raise InvalidTargetError("target out of range")
    if field_of.size != sources.size or (field_of.size and (
            field_of.min() < 0 or field_of.max() >= targets.size)):
        raise ValueError("field_of must map every source to one of the targets")
    _check_sources(sources, targets[field_of] if sources.size else sources, n)
    world, rank = dist.get_world_size(), dist.get_rank()
    a, b = partition_rows(targets.size, world)[rank]
    vals, _flags, mine_t = field_batch_by_targets(pk, fd, targets, dist, method=method,
                                                  clamp=clamp)
    mine = np.flatnonzero((field_of >= a) & (field_of < b))
    ldo = int(vals.stride(0)) if vals.dim() == 2 else 1
    if status_only:
        from .paths import trace_fields_status
        st, cnt = trace_fields_status(mesh, vals, 1, ldo, mine_t, sources[mine],
                                      field_of[mine] - a, settings)
        return mine, st, cnt
    paths = _trace_local(mesh, vals, 1, ldo, mine_t, sources[mine], field_of[mine] - a, settings)
    if not gather_paths:
        return mine, paths
    return _gather_paths(dist, sources.size, mine, paths)


def _trace_local(mesh, fields, field_ld, vertex_ld, targets, sources, field_of, settings):
    """K8 over this rank's paths (fields in any 2-D device layout)."""
    from .paths import trace_fields
    return trace_fields(mesh, fields, field_ld, vertex_ld, targets, sources, field_of, settings)


def _local_batch(pk, fd, targets, clamp, method):
    from .divergence import dv_field_batch_device
    return dv_field_batch_device(pk, fd, targets, clamp=clamp, method=method)


def _compute_batch_slab(slab, fd, targets, rows, method="auto", clamp=1e-300):
    """K7 on the slab for the global targets with their rows `rows` (T x k);
    `clamp` is the already-validated kernel clamp."""
    from .divergence import _kl_batch_slab
    t = dev.require_cuda()
    tg = t.from_numpy(np.asarray(targets, dtype=np.int64)).to(slab.device)
    return _kl_batch_slab(slab, tg, rows, float(clamp), method)


def _compute_slab(slab, fd, p: int, target_row, clamp: float, swap_order: bool = False):
    """The slab's field values to target p (CUDA kernels K0 + K2/K3/generic)
    and its flag words (device int32[4]; [0] = clamped on this slab)."""
    from .divergence import _field_device
    t = dev.require_cuda()
    out = t.empty(slab.rows + 2, dtype=t.float64, device=slab.device)
    s = t.cuda.current_stream(slab.device).cuda_stream
    st = _field_device(None, slab, fd, p, swap_order, clamp, out,
                       out.data_ptr() + slab.rows * 8, s, target_row=target_row)
    del st
    return out[:slab.rows], out[slab.rows:].view(t.int32)[:1]


def _sparse_tv_prep(slab, cut, strict, p, payload):
    """Owner side of the TV broadcast: K6 target prep into `payload` (vp, then tscal)."""
    from . import _native as nat
    t = dev.require_cuda()
    dc = slab.csr(cut, strict)
    kp = slab.k + (slab.k & 1)
    nat.call("pf_csr_target_prep_f64", dc.indptr.data_ptr(), dc.indices.data_ptr(),
             dc.data.data_ptr(), dc.dropped.data_ptr(), p - slab.row0, slab.k,
             payload.data_ptr(), payload.data_ptr() + kp * 8,
             t.cuda.current_stream(slab.device).cuda_stream)


def _compute_sparse_slab(slab, fd, p: int, payload, cut: float, strict: bool):
    """The slab's CSR field to target p (K5 with the broadcast dense row, or K6 with
    the broadcast sparsified target row)."""
    from . import _native as nat
    from .divergence import KL_GUARD_TAU, _CLAMP_LOG, _Staging
    t = dev.require_cuda()
    dc = slab.csr(cut, strict)
    s = t.cuda.current_stream(slab.device).cuda_stream
    out = t.empty(slab.rows + 2, dtype=t.float64, device=slab.device)
    flags = out.data_ptr() + slab.rows * 8
    out.view(t.int32)[2 * slab.rows:].zero_()
    if fd.name == "kl":
        st = _Staging(t, slab.k, slab.device)
        nat.call("pf_target_prep_f64", payload.data_ptr(), slab.k, _CLAMP_LOG, st.tgt, st.logt,
                 st.tmask, flags, s)
        entry, idx = dc.field_entry("kl")
        nat.call(entry, dc.indptr.data_ptr(), idx, dc.data.data_ptr(),
                 dc.log_data.data_ptr(), dc.hs.data_ptr(), slab.rows, slab.k, st.logt,
                 KL_GUARD_TAU, slab.row0, 0, slab.rows, out.data_ptr(), 0, flags,
                 1, s)
    else:
        kp = slab.k + (slab.k & 1)
        entry, idx = dc.field_entry("tv")
        nat.call(entry, dc.indptr.data_ptr(), idx, dc.data.data_ptr(),
                 dc.dropped.data_ptr(), slab.rows, slab.k, payload.data_ptr(),
                 payload.data_ptr() + kp * 8, slab.row0, 0, slab.rows, out.data_ptr(), 0, s)
    return out[:slab.rows]
