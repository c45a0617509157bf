"""Device-resident mirrors of the reference's immutable inputs.

A reference ``PoissonKernel`` is a frozen dataclass holding a read-only
numpy ``dense`` (``solvers.py:229-252``); ``sparsify`` returns a
``dataclasses.replace`` copy that shares the same ``dense`` array
(``divergence.py:237-240``).  The device copy is therefore keyed on the
identity of ``dense`` and lives as long as that array does, so the
reference's own caching (``DomainContext._pk``, ``domain.py:43-70``) decides
the device lifetime too.

HBM layout of P (one slab per GPU; the whole matrix on one GPU):
  rows x ld FP64, row-major, ld = round_up(k, 16) so every row starts on a
  128-byte boundary (full-sector 128-bit streaming loads); pad columns are
  zero (only the batched GEMM streams them, multiplied by zero logs).  Alongside: is_interior (uint8 per row) and the per-clamp
  negentropy H (FP64 per row, K1), built lazily.
"""

from __future__ import annotations

import threading
import weakref

import numpy as np

from . import _native as nat
from .errors import NativeError

_torch = None


def torch():
    """Import torch lazily (it is the buffer owner, not the compute path)."""
    global _torch
    if _torch is None:
        import torch as t
        _torch = t
    return _torch


_cuda_ok = False


def require_cuda():
    global _cuda_ok
    t = torch()
    if not _cuda_ok:
        if not t.cuda.is_available():
            raise NativeError(-101, "no CUDA device visible: the B200 path has no CPU fallback")
        nat.load()
        _cuda_ok = True
    return t


def i8_tiled_bytes(n: int, k: int) -> int:
    """Bytes of one K7 operand in the tiled layout (== pf_i8_tiled_bytes)."""
    return 0 if n <= 0 or k <= 0 else 7 * round_up(n, 128) * round_up(k, 32)


def round_up(x: int, m: int) -> int:
    return (x + m - 1) // m * m


def leading_dim(k: int) -> int:
    return round_up(k, 16)


class DeviceKernel:
    """Row slab [row0, row0+rows) of P resident in HBM, plus per-row state."""

    def __init__(self, dense: np.ndarray | None, boundary, *, device=None, row0: int = 0,
                 rows: int | None = None, n: int | None = None, k: int | None = None,
                 P_dev=None):
        t = require_cuda()
        self.device = (t.device(device) if device is not None
                       else t.device("cuda", t.cuda.current_device()))
        if dense is not None:
            n = dense.shape[0] if n is None else n
            k = dense.shape[1]
        if n is None or k is None:
            raise ValueError("need `dense`, or `n` and `k` with `P_dev`")
        self.n, self.k, self.row0 = int(n), int(k), int(row0)
        self.rows = int(rows if rows is not None else self.n - self.row0)
        if P_dev is not None:
            if (P_dev.dtype != t.float64 or P_dev.device != self.device or P_dev.dim() != 2
                    or P_dev.shape[0] != self.rows or P_dev.shape[1] < self.k
                    or P_dev.stride(1) != 1):
                raise ValueError("P_dev must be a row-major (rows, >=k) float64 tensor "
                                 "on the kernel device")
            self.ld = int(P_dev.stride(0))
            self.P = P_dev
        else:
            self.ld = leading_dim(self.k)
            self.P = t.empty((self.rows, self.ld), dtype=t.float64, device=self.device)
            if self.ld > self.k:
                self.P[:, self.k:] = 0.0  # pad columns are zero (K7 streams whole 16-col tiles)
            from ._hostpool import upload_rows
            upload_rows(t, self.P, dense, self.row0)
        self.boundary = (np.asarray(boundary, dtype=np.int64).reshape(-1)
                         if boundary is not None else np.zeros(0, dtype=np.int64))
        interior = np.ones(self.n, dtype=np.uint8)
        # The reference accepts any `boundary` array and only indexes with it in
        # dv_field's interior mask (divergence.py:173-174); keep out-of-range
        # entries here and let dv_field raise numpy's IndexError (dv_pair /
        # dv_at never read it).
        ok = (self.boundary >= -self.n) & (self.boundary < self.n)
        self.boundary_error = None
        if not ok.all():
            bad = int(self.boundary[~ok][0])
            self.boundary_error = (f"index {bad} is out of bounds for axis 0 with size "
                                   f"{self.n}")
        if self.boundary.size:
            interior[self.boundary[ok]] = 0
        self.is_interior = t.from_numpy(interior[self.row0:self.row0 + self.rows].copy()).to(self.device)
        self._H = {}
        self._csr = {}
        self._scratch = {}
        self._uniform = {}
        self._p32 = None
        self._min = None
        self._lock = threading.Lock()
        self._host = weakref.ref(dense) if dense is not None else None

    # -- per-row state ---------------------------------------------------
    def owns(self, row: int) -> bool:
        return self.row0 <= row < self.row0 + self.rows

    def negentropy(self, clamp: float):
        """H[r] = sum_b c(P) log c(P) for this slab (K1), cached per clamp."""
        key = float(clamp)
        with self._lock:
            h = self._H.get(key)
            if h is None:
                t = torch()
                h = t.empty(self.rows, dtype=t.float64, device=self.device)
                mn = t.full((1,), float("inf"), dtype=t.float64, device=self.device)
                stream = t.cuda.current_stream(self.device).cuda_stream
                nat.call("pf_row_negentropy_f64", self.P.data_ptr(), self.ld, self.rows,
                         self.k, key, h.data_ptr(), mn.data_ptr(), stream)
                self._H[key] = h
                if self._min is None:
                    self._min = mn
            return h

    def min_value(self) -> float:
        """min over the slab of P (divergence.py:162-165 domain check)."""
        if self._min is None:
            self.negentropy(1e-300)
        return float(self._min.item())

    def fp32(self):
        """(P32, ld32): FP32 copy of the slab for the FP32 storage mode (built once)."""
        with self._lock:
            if self._p32 is None:
                t = torch()
                ld32 = round_up(self.k, 32)
                P32 = t.empty((self.rows, ld32), dtype=t.float32, device=self.device)
                nat.call("pf_convert_f32", self.P.data_ptr(), self.ld, self.rows, self.k,
                         P32.data_ptr(), ld32, t.cuda.current_stream(self.device).cuda_stream)
                self._p32 = (P32, ld32)
            return self._p32

    def negentropy32(self, clamp: float):
        """H over the FP32 rows (FP64 accumulation), cached per clamp."""
        key = ("f32", float(clamp))
        P32, ld32 = self.fp32()
        with self._lock:
            h = self._H.get(key)
            if h is None:
                t = torch()
                h = t.empty(self.rows, dtype=t.float64, device=self.device)
                nat.call("pf_row_negentropy_f32", P32.data_ptr(), ld32, self.rows, self.k,
                         float(clamp), h.data_ptr(), t.cuda.current_stream(self.device).cuda_stream)
                self._H[key] = h
            return h

    def slices(self, clamp: float):
        """(A, ea, ldk): the 7 byte planes [7][rows][ldk] and per-row scale
        exponents of max(P, clamp) for K7 on the int8 tensor pipe
        (pf_slice_rows_u8), built once per clamp like H."""
        key = ("i8", float(clamp))
        with self._lock:
            hit = self._H.get(key)
            if hit is None:
                t = torch()
                ldk = round_up(self.k, 64)
                A = t.empty((7, self.rows, ldk), dtype=t.uint8, device=self.device)
                ea = t.empty(self.rows, dtype=t.int32, device=self.device)
                nat.call("pf_slice_rows_u8", self.P.data_ptr(), self.ld, self.rows, self.k,
                         float(clamp), ldk, A.data_ptr(), ea.data_ptr(),
                         t.cuda.current_stream(self.device).cuda_stream)
                hit = self._H[key] = (A, ea, ldk)
            return hit

    def slices_tiled(self, clamp: float):
        """(A, ea): the same byte planes in the tiled layout the CTA-pair
        kernel streams (pf_slice_rows_u8_tiled; pf_i8_tiled_bytes bytes)."""
        key = ("i8t", float(clamp))
        with self._lock:
            hit = self._H.get(key)
            if hit is None:
                t = torch()
                A = t.empty(i8_tiled_bytes(self.rows, self.k), dtype=t.uint8, device=self.device)
                ea = t.empty(self.rows, dtype=t.int32, device=self.device)
                nat.call("pf_slice_rows_u8_tiled", self.P.data_ptr(), self.ld, self.rows, self.k,
                         float(clamp), A.data_ptr(), ea.data_ptr(),
                         t.cuda.current_stream(self.device).cuda_stream)
                hit = self._H[key] = (A, ea)
            return hit

    def csr(self, cut: float, strict_positive: bool) -> "DeviceCSR":
        """The thresholded CSR view of this slab (K4), cached per (cut, mode)."""
        key = (float(cut), bool(strict_positive))
        with self._lock:
            c = self._csr.get(key)
            if c is None:
                c = DeviceCSR(self, float(cut), bool(strict_positive))
                self._csr[key] = c
            return c

    def mask_nonuniform(self, clamp: float) -> tuple[bool, object]:
        """(nonuniform, ref_row): do all interior rows share one below-clamp mask?

        Cached per clamp; ref_row is the first interior row (device view) or
        None when the slab has no interior rows.
        """
        key = float(clamp)
        with self._lock:
            hit = self._uniform.get(key)
        if hit is not None:
            return hit
        t = torch()
        interior = np.flatnonzero(self.is_interior.cpu().numpy())
        if interior.size == 0:
            res = (False, None)
        else:
            ref = self.P[int(interior[0]), :self.k]
            flag = t.zeros(1, dtype=t.int32, device=self.device)
            nat.call("pf_mask_uniform_f64", self.P.data_ptr(), self.ld, self.rows, self.k, key,
                     self.is_interior.data_ptr(), ref.data_ptr(), flag.data_ptr(),
                     t.cuda.current_stream(self.device).cuda_stream)
            res = (bool(flag.item()), ref)
        with self._lock:
            self._uniform[key] = res
        return res

    def scratch(self, stream_handle: int, nbytes: int, tag: str):
        """Per-(thread, stream, tag) device scratch reused across calls.

        Safe because every user of a scratch buffer enqueues on that same
        stream, so a later call's writes are ordered after the earlier call's
        kernels; threads never share one."""
        key = (threading.get_ident(), stream_handle, tag)
        with self._lock:
            buf = self._scratch.get(key)
        if buf is None or buf.numel() < nbytes:
            t = torch()
            buf = t.empty(nbytes, dtype=t.uint8, device=self.device)
            with self._lock:
                self._scratch[key] = buf
        return buf

    def row_ptr(self, p: int) -> int:
        """Device address of row p of this slab."""
        return self.P.data_ptr() + (p - self.row0) * self.ld * 8

    def target_row(self, p: int, host_dense: np.ndarray | None = None):
        """Device view of the raw target row P[p, :k].

        Owned rows are read in place; rows of another slab come from the host
        copy (single-process) — the multi-GPU path broadcasts instead
        (parallel.py).
        """
        t = torch()
        if self.owns(p):
            return self.P[p - self.row0, :self.k]
        if host_dense is None:
            host_dense = self._host() if self._host is not None else None
        if host_dense is None:
            raise NativeError(-102, f"target row {p} is not resident on this device")
        return t.from_numpy(np.array(host_dense[p], dtype=np.float64)).to(self.device)


class DeviceCSR:
    """CSR arrays of one slab built on the device from the dense rows (K4).

    Layout: indptr int64 (rows+1, slab-local) over ROW-ALIGNED rows — every
    row starts at an even offset (bit 0 of indptr[r+1] flags a pad) and a row
    with an odd entry count ends with one zero pad entry (data 0, log 0) that
    the kernels exclude, so a row's
    element order (and therefore its reduction) does not depend on where the
    row sits; indices int32 (ascending per row), data / log_data FP64,
    hs = sum v log v and dropped (FP64 per row), rownnz (int64, real counts).
    The algorithmic bytes are those of scipy's layout: nnz*(8+4) + rows*24.
    """

    def __init__(self, dk: DeviceKernel, cut: float, strict_positive: bool):
        t = torch()
        self.dk, self.cut, self.strict = dk, cut, strict_positive
        rows, dev_ = dk.rows, dk.device
        s = t.cuda.current_stream(dev_).cuda_stream
        # per-row arrays in one allocation: rownnz, indptr (rows + 1), hs, dropped
        rowbuf = t.empty(4 * rows + 1, dtype=t.int64, device=dev_)
        self.rownnz = rowbuf[:rows]
        nat.call("pf_csr_count_f64", dk.P.data_ptr(), dk.ld, rows, dk.k, cut,
                 int(strict_positive), self.rownnz.data_ptr(), s)
        self.indptr = rowbuf[rows:2 * rows + 1]
        self.indptr[:1].zero_()
        t.cumsum(self.rownnz + (self.rownnz & 1), 0, out=self.indptr[1:])
        # the padded and the real totals in ONE host round trip
        tot = t.stack([self.indptr[-1], self.rownnz.sum()]).cpu().tolist()
        self.nnz_pad, self.nnz = int(tot[0]), int(tot[1])
        self.indptr[1:] |= self.rownnz & 1  # pad flag in bit 0 of the row's end offset
        self.hs = rowbuf[2 * rows + 1:3 * rows + 1].view(t.float64)
        self.dropped = rowbuf[3 * rows + 1:].view(t.float64)
        # entry arrays in one allocation: data, log_data (FP64), indices (i32),
        # and the 16-bit column copy the K5/K6 field kernels stream (k <= 65,536:
        # 10 instead of 12 bytes per entry)
        cap = max(self.nnz_pad, 1)
        narrow = dk.k <= 65536
        cap8 = (cap + 7) // 8 * 8
        ent = t.empty(cap8 * (8 + 8 + 4 + (2 if narrow else 0)), dtype=t.uint8, device=dev_)
        self._entries = ent
        self.data = ent[:8 * cap8].view(t.float64)[:cap]
        self.log_data = ent[8 * cap8:16 * cap8].view(t.float64)[:cap]
        self.indices = ent[16 * cap8:20 * cap8].view(t.int32)[:cap]
        nat.call("pf_csr_fill_f64", dk.P.data_ptr(), dk.ld, rows, dk.k, cut,
                 int(strict_positive), self.indptr.data_ptr(), self.indices.data_ptr(),
                 self.data.data_ptr(), self.log_data.data_ptr(), self.hs.data_ptr(),
                 self.dropped.data_ptr(), s)
        self.indices16 = None
        if narrow:
            self.indices16 = ent[20 * cap8:22 * cap8].view(t.int16)[:cap]
            nat.call("pf_csr_narrow_u16", self.indices.data_ptr(), self.nnz_pad,
                     self.indices16.data_ptr(), s)

    def field_entry(self, name: str):
        """(C entry point, column-index pointer) of the K5 (kl) / K6 (tv) field
        kernel for this CSR: the 16-bit variant when the columns fit."""
        if self.indices16 is not None:
            return f"pf_csr_{name}_u16_f64", self.indices16.data_ptr()
        return f"pf_csr_{name}_f64", self.indices.data_ptr()

    def owns(self, row: int) -> bool:
        return self.dk.owns(row)

    def scipy_arrays(self, with_data: bool = True, with_log: bool = True):
        """(indptr, indices, data, log_data) in scipy's unpadded layout, on the
        device (pf_csr_unpad: one pass, no host round trip)."""
        t = torch()
        dev_ = self.dk.device
        ip = self.scipy_indptr()
        n = max(self.nnz, 1)
        idx = t.empty(n, dtype=t.int32, device=dev_)
        dat = t.empty(n, dtype=t.float64, device=dev_) if with_data else None
        lg = t.empty(n, dtype=t.float64, device=dev_) if with_log else None
        nat.call("pf_csr_unpad", self.indptr.data_ptr(), ip.data_ptr(), self.dk.rows,
                 self.indices.data_ptr(), self.data.data_ptr(), self.log_data.data_ptr(),
                 idx.data_ptr(), nat.ptr(dat), nat.ptr(lg),
                 t.cuda.current_stream(dev_).cuda_stream)
        m = self.nnz
        return ip, idx[:m], (dat[:m] if dat is not None else None), (
            lg[:m] if lg is not None else None)

    def real_mask(self):
        """Boolean mask over the padded arrays selecting the real entries."""
        t = torch()
        keep = t.ones(max(self.nnz_pad, 1), dtype=t.bool, device=self.dk.device)
        odd = (self.rownnz & 1).bool()
        pads = ((self.indptr[:-1] & ~1) + self.rownnz)[odd]
        keep[pads] = False
        return keep[:self.nnz_pad]

    def scipy_indptr(self):
        """indptr of the unpadded (scipy) layout, on the device."""
        t = torch()
        ip = t.zeros(self.dk.rows + 1, dtype=t.int64, device=self.dk.device)
        t.cumsum(self.rownnz, 0, out=ip[1:])
        return ip


_cache: dict[int, tuple[weakref.ref, DeviceKernel]] = {}
_cache_lock = threading.Lock()
_building: dict[int, threading.Lock] = {}   # per-array creation locks


def _lookup(dense):
    with _cache_lock:
        hit = _cache.get(id(dense))
        if hit is not None and hit[0]() is dense:
            return hit[1]
    return None


def device_kernel(pk) -> DeviceKernel:
    """The device mirror of ``pk.dense`` (uploaded on first use).

    Reentrant (FastAPI serves dv_field from a thread pool, SURVEY §8b
    "Threading"): concurrent first calls on the same kernel build ONE mirror —
    the others wait on that array's creation lock — while calls on other
    kernels proceed."""
    dense = pk.dense
    dk = _lookup(dense)
    if dk is not None:
        return dk
    with _cache_lock:
        lk = _building.setdefault(id(dense), threading.Lock())
    with lk:
        dk = _lookup(dense)
        if dk is None:
            dk = DeviceKernel(dense, getattr(pk, "boundary", None))
            register(dense, dk)
    with _cache_lock:
        if _building.get(id(dense)) is lk:
            del _building[id(dense)]
    return dk


# ---- device mirrors of returned fields ------------------------------------
# dv_field copies the field to the host (the reference returns numpy); a
# tracer call that follows on the same ScalarField (DomainContext.trace,
# domain.py:86-96) reads this device copy instead of uploading the values
# again.  Bounded: the most recent fields only.
_FIELD_KEEP = 8
_fields: dict[int, tuple] = {}
_fields_order: list[int] = []


def register_field(values, dev_values) -> None:
    key = id(values)

    def _drop(_ref, key=key):
        with _cache_lock:
            _fields.pop(key, None)

    with _cache_lock:
        _fields[key] = (weakref.ref(values, _drop), dev_values)
        _fields_order.append(key)
        while len(_fields_order) > _FIELD_KEEP:
            _fields.pop(_fields_order.pop(0), None)


def field_mirror(values):
    """The device copy of a field's host values, if it is still registered."""
    with _cache_lock:
        hit = _fields.get(id(values))
    if hit is not None and hit[0]() is values:
        return hit[1]
    return None


def register(dense: np.ndarray, dk: DeviceKernel) -> DeviceKernel:
    """Bind an existing device kernel (e.g. generated on the GPU) to a host array."""
    key = id(dense)

    def _drop(_ref, key=key):
        with _cache_lock:
            ent = _cache.get(key)
            if ent is not None and ent[0]() is None:
                del _cache[key]

    with _cache_lock:
        _cache[key] = (weakref.ref(dense, _drop), dk)
    return dk


def evict(pk) -> None:
    with _cache_lock:
        _cache.pop(id(pk.dense), None)
