"""Row-sharded multi-GPU evaluation: one process per GPU over torch.distributed.

Every output row q of a divergence field depends only on row q of P and on
the target row, so the GPUs of one box own contiguous row slabs
(dense: balanced by row count; CSR: balanced by nnz) and evaluate them with
the single-GPU kernels unchanged — the N-GPU field is bitwise the 1-GPU
field.  The data path has exactly two exchanges, both NCCL over NVLink:

* the target row P[t, :] (k FP64) is broadcast from its owner rank
  (``ncclBroadcast``, 33 KB at k = 4,102);
* the finished field slabs are all-gathered (``ncclAllGather``, n FP64)
  only when a tracer on every rank needs the whole field.

Batched targets (K7) come in both layouts the survey
names: :meth:`ShardedField.field_batch` keeps P row-sharded and assembles
the T target rows with one all-reduce (each row is its owner's values plus
zeros: exact), then every rank contracts its slab; :func:`field_batch_by_targets`
replicates P (32.8 GB at C4 fits one B200) and partitions the targets, with
no data-path collective at all.

There are no reductions of computed values (the per-target ``clamped``
flags are OR-ed).  The host logic (partitioning, ownership,
broadcast/gather orchestration) is backend-agnostic and is exercised with the
gloo backend on CPU in tests/test_parallel.py; the slab computation itself is
always the CUDA kernels (``_compute_slab``).
"""

from __future__ import annotations

import numpy as np

from . import _device as dev


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
    for r, (a, b) in enumerate(bounds):
        if a <= row < b:
            return r
    raise IndexError(f"row {row} outside every slab")


class ShardedField:
    """Per-rank driver of a row-sharded field evaluation.

    ``slab`` is this rank's :class:`~paper_1708_02845_b200._device.DeviceKernel`
    (rows ``bounds[rank]`` of the global P); ``dist`` the initialised
    ``torch.distributed`` module (nccl on GPUs; gloo in the CPU tests).
    """

    def __init__(self, slab, bounds, dist, device=None):
        self.slab, self.bounds, self.dist = slab, bounds, dist
        self.rank = dist.get_rank()
        self.world = dist.get_world_size()
        self.device = device if device is not None else getattr(slab, "device", None)
        a, b = bounds[self.rank]
        if (getattr(slab, "row0", a), getattr(slab, "rows", b - a)) != (a, b - a):
            raise ValueError("slab does not match this rank's partition")

    @classmethod
    def from_mesh(cls, mesh, dist, device=None, bounds=None):
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
        diag = t.tensor([dk.residual, dk.row_sum_error], dtype=t.float64, device=dk.device)
        dist.all_reduce(diag, op=dist.ReduceOp.MAX)
        dk.residual, dk.row_sum_error = float(diag[0].item()), float(diag[1].item())
        return cls(dk, bounds, dist, device=dk.device)

    def target_row(self, p: int, k: int):
        """Broadcast P[p, :k] from its owner to every rank (the one data-path exchange)."""
        t = dev.torch()
        own = owner_of(p, self.bounds)
        if self.rank == own:
            row = self.slab.P[p - self.bounds[own][0], :k].contiguous()
        else:
            row = t.empty(k, dtype=t.float64, device=self.device)
        self.dist.broadcast(row, src=own)
        return row

    def field(self, fd, p: int, gather: bool = False, clamp=None):
        """This rank's slab of the field to target p (device); all ranks' if `gather`."""
        row = self.target_row(p, self.slab.k)
        vals = _compute_slab(self.slab, fd, p, row, clamp)
        if not gather:
            return vals
        return self.gather(vals)

    def sparse_field(self, fd, p: int, threshold: float | None = None, gather: bool = False):
        """This rank's slab of the sparse (CSR) field to target p (divergence.py:255-299).

        KL needs the target's dense log row: the dense row is broadcast as for
        :meth:`field`.  TV needs the target's sparsified row: its owner scatters it
        (K6 prep) and broadcasts the dense k-vector plus (S_p, dropped_p, nnz_p).
        CSR slabs should be partitioned with :func:`partition_by_weight` over nnz.
        """
        import math
        t = dev.torch()
        n, k = self.slab.n, self.slab.k
        thr = 1.0 / math.sqrt(n) if threshold is None else float(threshold)
        cut = thr / k
        if fd.name == "kl":
            payload = self.target_row(p, k)
        elif fd.name == "tv":
            own = owner_of(p, self.bounds)
            kp = k + (k & 1)
            payload = t.empty(kp + 4, dtype=t.float64, device=self.device)
            if self.rank == own:
                _sparse_tv_prep(self.slab, cut, thr == 0, p, payload)
            self.dist.broadcast(payload, src=own)
        else:
            raise NotImplementedError("sparse fields implement kl and tv")
        vals = _compute_sparse_slab(self.slab, fd, p, payload, cut, thr == 0)
        return self.gather(vals) if gather else vals

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
        self.dist.all_reduce(rows)
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
        n = self.bounds[-1][1]
        if targets.size and (targets.min() < 0 or targets.max() >= n):
            from .errors import InvalidTargetError
            raise InvalidTargetError("target out of range")
        if fd.name != "kl":
            cols = [self.field(fd, int(p), clamp=clamp) for p in targets]
            vals = t.stack(cols, dim=1) if cols else t.zeros((self.slab.rows, 0), dtype=t.float64)
            flags = np.zeros(targets.size, dtype=bool)
        else:
            rows = self.target_rows(targets, self.slab.k)
            vals, flags = _compute_batch_slab(self.slab, fd, targets, rows, method, clamp)
            f = t.from_numpy(np.asarray(flags, dtype=np.int32)).to(self.device)
            self.dist.all_reduce(f, op=self.dist.ReduceOp.MAX)
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
        parts = [t.empty((m, T), dtype=vals.dtype, device=vals.device) for _ in range(self.world)]
        self.dist.all_gather(parts, buf)
        return t.cat([parts[r][:sizes[r]] for r in range(self.world)])

    def gather(self, vals):
        """All-gather variable-size slabs into the full n-vector on every rank."""
        t = dev.torch()
        sizes = [b - a for a, b in self.bounds]
        m = max(sizes)
        buf = t.zeros(m, dtype=vals.dtype, device=vals.device)
        buf[:vals.numel()] = vals
        parts = [t.empty(m, dtype=vals.dtype, device=vals.device) for _ in range(self.world)]
        self.dist.all_gather(parts, buf)
        return t.cat([parts[r][:sizes[r]] for r in range(self.world)])


def field_batch_by_targets(pk, fd, targets, dist, gather: bool = False, method: str = "auto",
                           clamp=None):
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
    n = vals.shape[0]
    m = max(e - s for s, e in chunks)
    buf = t.zeros((m, n), dtype=vals.dtype, device=vals.device)
    buf[:b - a] = vals.t()
    parts = [t.empty((m, n), dtype=vals.dtype, device=vals.device) for _ in range(world)]
    dist.all_gather(parts, buf)
    fl = t.zeros(m, dtype=t.int32, device=vals.device)
    fl[:b - a] = t.from_numpy(np.asarray(flags, dtype=np.int32)).to(vals.device)
    fparts = [t.empty(m, dtype=t.int32, device=vals.device) for _ in range(world)]
    dist.all_gather(fparts, fl)
    full = t.cat([parts[r][:e - s] for r, (s, e) in enumerate(chunks)]).t()
    fall = t.cat([fparts[r][:e - s] for r, (s, e) in enumerate(chunks)]).cpu().numpy()
    return full, fall.astype(bool), targets


def _local_batch(pk, fd, targets, clamp, method):
    from .divergence import dv_field_batch_device
    return dv_field_batch_device(pk, fd, targets, clamp=clamp, method=method)


def _compute_batch_slab(slab, fd, targets, rows, method="auto", clamp=None):
    """K7 on the slab for the global targets with their rows `rows` (T x k)."""
    from .divergence import _effective_clamp, _kl_batch_slab
    t = dev.require_cuda()
    c = _effective_clamp(slab, fd.clamp if clamp is None else clamp)
    tg = t.from_numpy(np.asarray(targets, dtype=np.int64)).to(slab.device)
    return _kl_batch_slab(slab, tg, rows, c, method)


def _compute_slab(slab, fd, p: int, target_row, clamp=None):
    """The slab's field values to target p (CUDA kernels K0 + K2/K3/generic)."""
    from .divergence import _effective_clamp, _field_device
    t = dev.require_cuda()
    c = _effective_clamp(slab, fd.clamp if clamp is None else clamp)
    out = t.empty(slab.rows + 2, dtype=t.float64, device=slab.device)
    s = t.cuda.current_stream(slab.device).cuda_stream
    st = _field_device(None, slab, fd, p, False, c, out, out.data_ptr() + slab.rows * 8, s,
                       target_row=target_row)
    del st
    return out[:slab.rows]


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
                 slab.scratch(s, 8, "csrq").data_ptr(), s)
    else:
        kp = slab.k + (slab.k & 1)
        entry, idx = dc.field_entry("tv")
        nat.call(entry, dc.indptr.data_ptr(), idx, dc.data.data_ptr(),
                 dc.dropped.data_ptr(), slab.rows, slab.k, payload.data_ptr(),
                 payload.data_ptr() + kp * 8, slab.row0, 0, slab.rows, out.data_ptr(), 0, s)
    return out[:slab.rows]
