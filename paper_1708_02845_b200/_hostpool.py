"""Pinned host buffers for returning device results as numpy arrays.

A field returned by the public API is an ``n``-vector the caller owns.
Copying it into a fresh pageable array costs page faults on every call, and a
fresh pinned allocation costs ~0.8 ms (measured, tools/micro_d2h.py).  This
pool hands out pinned buffers whose numpy view *is* the returned array: the
device-to-host copy is a straight DMA into already-mapped memory, and the
buffer goes back to the pool when the last numpy view of it is garbage
collected (``weakref.finalize`` on the array that owns the memory; numpy
collapses view chains onto that owner, so no live view can outlast it).
"""

from __future__ import annotations

import threading
import weakref

import numpy as np

_lock = threading.Lock()
_free: dict[tuple[int, str], list] = {}
_MAX_FREE_PER_SIZE = 8


def _give_back(key, tensor):
    with _lock:
        lst = _free.setdefault(key, [])
        if len(lst) < _MAX_FREE_PER_SIZE:
            lst.append(tensor)


def to_host(t, dbuf, stream) -> np.ndarray:
    """Copy device tensor `dbuf` into a pooled pinned buffer; returns the owning numpy array."""
    key = (int(dbuf.numel()), str(dbuf.dtype))
    with _lock:
        lst = _free.get(key)
        host = lst.pop() if lst else None
    if host is None:
        host = t.empty(dbuf.shape, dtype=dbuf.dtype, pin_memory=True)
    host = host.view(dbuf.shape)
    host.copy_(dbuf, non_blocking=True)
    stream.synchronize()
    arr = host.numpy()
    weakref.finalize(arr, _give_back, key, host)
    return arr


_tls = threading.local()


def pinned_view(t, arr: np.ndarray) -> int:
    """Copy a small host array into this thread's pinned scratch and return its
    address, which kernels read in place (pinned memory is mapped into the
    device's address space under UVA: no copy operation, no event).  Valid
    until this thread's next call; callers synchronize before returning."""
    need = max(int(arr.nbytes), 64)
    buf = getattr(_tls, "pinned", None)
    if buf is None or buf.numel() < need:
        buf = t.empty(max(need, 1 << 16), dtype=t.uint8, pin_memory=True)
        _tls.pinned = buf
    buf.numpy()[: arr.nbytes] = np.ascontiguousarray(arr).view(np.uint8).reshape(-1)
    return buf.data_ptr()


# -- host -> device row upload ------------------------------------------------
_UPLOAD_CHUNK_BYTES = 64 << 20
_UPLOAD_BUFFERS = 3
_upload_pool = None


def _threads():
    global _upload_pool
    if _upload_pool is None:
        import os
        from concurrent.futures import ThreadPoolExecutor
        _upload_pool = ThreadPoolExecutor(max_workers=min(16, os.cpu_count() or 1),
                                          thread_name_prefix="pf-upload")
    return _upload_pool


def upload_rows(t, dst, src: np.ndarray, row0: int = 0) -> None:
    """``dst[:, :k] = src[row0:row0+rows]`` for a (rows, >=k) device tensor.

    The reference's P is a pageable numpy array (``solvers.py:251-252``).  A plain
    ``copy_`` from pageable memory runs at the driver's bounce-buffer rate; here the
    rows go through ``_UPLOAD_BUFFERS`` pinned staging buffers instead: host threads
    fill buffer i+1 (``np.copyto`` releases the GIL) while the DMA of buffer i runs
    on a side stream, and a buffer is refilled only after its copy's event.
    """
    rows, k = int(dst.shape[0]), int(src.shape[1])
    if rows == 0:
        return
    chunk = max(1, _UPLOAD_CHUNK_BYTES // (8 * k))
    nbuf = min(_UPLOAD_BUFFERS, -(-rows // chunk))
    bufs = [t.empty((chunk, k), dtype=t.float64, pin_memory=True) for _ in range(nbuf)]
    views = [b.numpy() for b in bufs]
    done = [None] * nbuf
    stream = t.cuda.Stream(device=dst.device)
    pool = _threads()
    nthr = pool._max_workers
    with t.cuda.stream(stream):
        for i, a in enumerate(range(0, rows, chunk)):
            b = min(rows, a + chunk)
            j = i % nbuf
            if done[j] is not None:
                done[j].synchronize()
            hv = views[j]
            step = -(-(b - a) // nthr)
            futs = [pool.submit(np.copyto, hv[s:min(b - a, s + step)],
                                src[row0 + a + s:row0 + min(b, a + s + step)])
                    for s in range(0, b - a, step)]
            for f in futs:
                f.result()
            dst[a:b, :k].copy_(bufs[j][:b - a], non_blocking=True)
            ev = t.cuda.Event()
            ev.record(stream)
            done[j] = ev
    stream.synchronize()


# -- device -> host bulk download ----------------------------------------------
_DOWNLOAD_CHUNK_BYTES = 64 << 20
_dl_lock = threading.Lock()
_dl_bufs: list = []


def download(t, src) -> np.ndarray:
    """A fresh numpy copy of a large contiguous 1-D device tensor.

    Returned arrays the caller keeps (sparsify's CSR views: ~1 GB at C3) go
    through two persistent pinned 64 MB staging buffers: the DMA of chunk i+1
    runs while host threads scatter chunk i into the pageable result (first-
    touching its pages in parallel), instead of a pinned allocation the size
    of the result (~0.3 ms per MB) or a single-threaded pageable copy."""
    n = int(src.numel())
    esz = src.element_size()
    out = np.empty(n, dtype=np.dtype(str(src.dtype).replace("torch.", "")))
    if n == 0:
        return out
    flat = src.reshape(-1).view(t.uint8)
    dst = out.view(np.uint8)
    total = n * esz
    chunk = _DOWNLOAD_CHUNK_BYTES
    pool = _threads()
    nthr = pool._max_workers
    with _dl_lock:
        while len(_dl_bufs) < 2:
            _dl_bufs.append(t.empty(chunk, dtype=t.uint8, pin_memory=True))
        bufs = _dl_bufs
        evs = [t.cuda.Event(), t.cuda.Event()]
        stream = t.cuda.Stream(device=src.device)
        stream.wait_stream(t.cuda.current_stream(src.device))

        def scatter(j, a, b):
            hv = bufs[j].numpy()
            step = -(-(b - a) // nthr)
            futs = [pool.submit(np.copyto, dst[a + s:min(b, a + s + step)],
                                hv[s:min(b - a, s + step)]) for s in range(0, b - a, step)]
            for f in futs:
                f.result()

        pending = None
        for i, a in enumerate(range(0, total, chunk)):
            b = min(total, a + chunk)
            j = i & 1
            with t.cuda.stream(stream):
                bufs[j][:b - a].copy_(flat[a:b], non_blocking=True)
                evs[j].record(stream)
            if pending is not None:
                evs[pending[0]].synchronize()
                scatter(*pending)
            pending = (j, a, b)
        evs[pending[0]].synchronize()
        scatter(*pending)
    return out
