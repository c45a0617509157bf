"""numpy restatement of the reference divergence functions — TEST INFRASTRUCTURE.

Follows /root/reference/pkg/src/pathfield/divergence.py line by line (see
oracle/__init__.py for the rules on who may import this).  Generators are
named ("kl", "tv", "chi2", "hellinger", "alpha", "power-p") with the
reference's clamps (divergence.py:37-38, 79-103).

``dv_field_chunked`` is the bounded-memory, multi-threaded form used as the
CPU baseline: it evaluates exactly ``dv_at`` over row chunks, which the
survey found bitwise equal to ``dv_field``, with numpy releasing
the GIL inside its ufuncs so the chunks run on all host cores.
"""

from __future__ import annotations

import math
import os
from concurrent.futures import ThreadPoolExecutor

import numpy as np

CLAMP_LOG = 1e-300      # divergence.py:37
CLAMP_POWER = 1e-150    # divergence.py:38
NEG_NOISE = 1e-10       # divergence.py:39


def generator(name: str, alpha: float | None = None, power: int | None = None):
    """(f, clamp) of builtin_f (divergence.py:70-104)."""
    if name == "tv":
        return (lambda x: np.abs(1.0 - x)), CLAMP_POWER
    if name == "kl":
        return (lambda x: -np.log(x)), CLAMP_LOG
    if name == "chi2":
        return (lambda x: x * x - 1.0), CLAMP_POWER
    if name == "hellinger":
        return (lambda x: (np.sqrt(x) - 1.0) ** 2), CLAMP_POWER
    if name == "alpha":
        a = float(alpha)
        scale = 4.0 / (1.0 - a * a)
        expo = (1.0 + a) / 2.0
        return (lambda x: scale * (1.0 - x ** expo)), CLAMP_LOG
    if name == "power-p":
        p = int(power)
        return (lambda x: np.abs(1.0 - x) ** p), CLAMP_POWER
    raise ValueError(name)


def settle(v: float) -> float:
    """divergence.py:117-122."""
    return 0.0 if -NEG_NOISE < v < 0.0 else v


def dv_pair(dense, name, p, q, swap_order=False, clamp=None, **gp) -> float:
    """divergence.py:125-134 (+ _clamped_rows :107-114)."""
    f, c0 = generator(name, **gp)
    clamp = c0 if clamp is None else clamp
    P_row, Q_row = dense[p], dense[q]
    if swap_order:
        P_row, Q_row = Q_row, P_row
    if clamp is None or clamp <= 0.0:
        if np.any(Q_row <= 0.0) or np.any(P_row <= 0.0):
            raise ValueError("zero kernel entry and clamping is disabled")
        ps, qs = P_row, Q_row
    else:
        ps, qs = np.maximum(P_row, clamp), np.maximum(Q_row, clamp)
    return settle(float(qs @ f(ps / qs)))


def dv_at(dense, name, p, queries, swap_order=False, clamp=None, **gp) -> np.ndarray:
    """divergence.py:137-151."""
    f, c0 = generator(name, **gp)
    clamp = c0 if clamp is None else clamp
    queries = np.asarray(queries, dtype=np.int64)
    ps = np.maximum(dense[p], clamp)
    qs = np.maximum(dense[queries], clamp)
    if swap_order:
        vals = (ps[None, :] * f(qs / ps[None, :])).sum(axis=1)
    else:
        vals = (qs * f(ps[None, :] / qs)).sum(axis=1)
    vals[(vals > -NEG_NOISE) & (vals < 0.0)] = 0.0
    vals[queries == p] = 0.0
    return vals


def clamp_flag(dense, boundary, p, clamp) -> bool:
    """The ("clamped",) precision flag of dv_field (divergence.py:172-175), row-chunked."""
    interior = np.ones(dense.shape[0], dtype=bool)
    interior[np.asarray(boundary, dtype=np.int64)] = False
    tm = dense[p] < clamp
    step = max(1, (1 << 24) // max(1, dense.shape[1]))
    for a in range(0, dense.shape[0], step):
        b = min(dense.shape[0], a + step)
        rows = interior[a:b]
        if rows.any() and ((dense[a:b][rows] < clamp) != tm[None, :]).any():
            return True
    return False


def dv_field(dense, boundary, name, p, swap_order=False, clamp=None, **gp):
    """divergence.py:154-187; returns (values, precision_flags)."""
    f, c0 = generator(name, **gp)
    clamp = c0 if clamp is None else clamp
    if clamp is None or clamp <= 0.0:
        if np.any(dense <= 0.0):
            raise ValueError("zero kernel entries and clamping is disabled")
        ps_t, qs, fired = dense[p], dense, False
    else:
        ps_t = np.maximum(dense[p], clamp)
        qs = np.maximum(dense, clamp)
        onesided = (dense < clamp) != (dense[p][None, :] < clamp)
        interior = np.ones(dense.shape[0], dtype=bool)
        interior[np.asarray(boundary, dtype=np.int64)] = False
        fired = bool(onesided[interior].any())
    if swap_order:
        vals = (ps_t[None, :] * f(qs / ps_t[None, :])).sum(axis=1)
    else:
        vals = (qs * f(ps_t[None, :] / qs)).sum(axis=1)
    vals[(vals > -NEG_NOISE) & (vals < 0.0)] = 0.0
    vals[p] = 0.0
    return vals, (("clamped",) if fired else ())


def dv_field_chunked(dense, name, p, rows=None, chunk_rows=2048, threads=None, **gp):
    """dv_at over row chunks (bitwise == dv_field values), threaded.

    ``rows`` restricts the evaluation to a bounded sample (a slice or index
    array) for CPU timing.
    """
    n = dense.shape[0]
    idx = np.arange(n, dtype=np.int64) if rows is None else np.asarray(
        np.arange(n)[rows] if isinstance(rows, slice) else rows, dtype=np.int64)
    out = np.empty(idx.size)
    threads = threads or os.cpu_count() or 1
    chunks = [(a, min(idx.size, a + chunk_rows)) for a in range(0, idx.size, chunk_rows)]

    def work(ab):
        a, b = ab
        out[a:b] = dv_at(dense, name, p, idx[a:b], **gp)

    if threads == 1:
        for ab in chunks:
            work(ab)
    else:
        with ThreadPoolExecutor(threads) as ex:
            list(ex.map(work, chunks))
    return out


# ------------------------------------------------------------------ sparse --

def sparsify(dense, boundary, threshold=None):
    """divergence.py:194-240 without scipy: returns a dict of the views.

    The pattern is {P >= cut} (or {P > 0} at threshold 0) in row-major order
    with ascending columns, which is exactly what ``csr_matrix`` +
    ``eliminate_zeros`` produce.
    """
    n, k = dense.shape
    if threshold is None:
        threshold = 1.0 / math.sqrt(n)
    if threshold < 0:
        raise ValueError("threshold must be nonnegative")
    if threshold >= 1.0:
        raise ValueError(f"threshold {threshold} >= 1 would empty rows")
    cut = threshold / k
    keep = dense >= cut if threshold > 0 else dense > 0
    keep &= dense != 0.0  # eliminate_zeros (cut may be 0 only at threshold 0)
    rows, cols = np.nonzero(keep)
    data = dense[rows, cols]
    indptr = np.zeros(n + 1, dtype=np.int64)
    np.cumsum(np.bincount(rows, minlength=n), out=indptr[1:])
    log_sparse = np.log(data)
    log_dense = np.log(np.maximum(dense, CLAMP_LOG))
    # scipy's csr .sum(axis=1) is np.add.reduceat over the non-empty rows
    # (scipy/sparse/_compressed.py _minor_reduce): numpy pairwise summation.
    rowsum = np.zeros(n)
    nonempty = np.flatnonzero(np.diff(indptr))
    if nonempty.size:
        rowsum[nonempty] = np.add.reduceat(data, indptr[nonempty])
    dropped = np.clip(1.0 - rowsum, 0.0, None)
    interior = np.ones(n, dtype=bool)
    interior[np.asarray(boundary, dtype=np.int64)] = False
    m = int(interior.sum())
    sparsity = 100.0 * (1.0 - int(np.diff(indptr)[interior].sum()) / (m * k)) if m else 0.0
    return dict(threshold=float(threshold), indptr=indptr, indices=cols.astype(np.int64),
                data=data, log_sparse=log_sparse, log_dense=log_dense, dropped=dropped,
                row_cut=float(cut), sparsity_percent=float(sparsity))


def dv_pair_sparse_stats(sv, name, p, q, swap_order=False, **gp):
    """divergence.py:255-299 on the dict views of :func:`sparsify` (kl, tv)."""
    if swap_order:
        p, q = q, p
    ip, iq = sv["indptr"], sv["indices"]
    idx_p, val_p = iq[ip[p]:ip[p + 1]], sv["data"][ip[p]:ip[p + 1]]
    idx_q, val_q = iq[ip[q]:ip[q + 1]], sv["data"][ip[q]:ip[q + 1]]
    log_q = sv["log_sparse"][ip[q]:ip[q + 1]]
    if name == "kl":
        ops = int(idx_q.size)
        val = float(val_q @ (log_q - sv["log_dense"][p, idx_q]))
        return settle(val), ops
    if name == "tv":
        union = np.union1d(idx_p, idx_q)
        vp = np.zeros(union.size)
        vp[np.searchsorted(union, idx_p)] = val_p
        vq = np.zeros(union.size)
        vq[np.searchsorted(union, idx_q)] = val_q
        base = float(np.abs(vp - vq).sum())
        return base + float(sv["dropped"][p] + sv["dropped"][q]), int(union.size)
    raise NotImplementedError(name)


def dv_field_sparse(sv, name, p, rows=None):
    """[dv_pair_sparse(spk, f, p, q) for q in rows] — the reference's only sparse field."""
    n = sv["indptr"].size - 1
    rows = range(n) if rows is None else rows
    return np.array([dv_pair_sparse_stats(sv, name, p, int(q))[0] for q in rows])


def _kept_row(dense, cut, strict, r):
    row = dense[r]
    keep = (row > 0) if strict else (row >= cut)
    keep &= row != 0.0
    idx = np.flatnonzero(keep)
    vals = row[idx]
    s = np.add.reduceat(vals, [0])[0] if vals.size else 0.0  # scipy csr.sum(axis=1) order
    return idx, vals, max(0.0, 1.0 - s)


def dv_pair_sparse_direct(dense, p, q, name, threshold=None):
    """dv_pair_sparse_stats for one pair straight from the dense rows (no full CSR):
    the same formulas as :func:`dv_pair_sparse_stats` on the rows of sparsify
    (divergence.py:212-228, 255-295) — for inputs too large to sparsify on the host."""
    n, k = dense.shape
    if threshold is None:
        threshold = 1.0 / math.sqrt(n)
    cut = threshold / k
    strict = threshold == 0
    idx_p, val_p, drop_p = _kept_row(dense, cut, strict, p)
    idx_q, val_q, drop_q = _kept_row(dense, cut, strict, q)
    if name == "kl":
        log_q = np.log(val_q)
        lp = np.log(np.maximum(dense[p, idx_q], CLAMP_LOG))
        return settle(float(val_q @ (log_q - lp))), int(idx_q.size)
    union = np.union1d(idx_p, idx_q)
    vp = np.zeros(union.size)
    vp[np.searchsorted(union, idx_p)] = val_p
    vq = np.zeros(union.size)
    vq[np.searchsorted(union, idx_q)] = val_q
    return float(np.abs(vp - vq).sum()) + float(drop_p + drop_q), int(union.size)
