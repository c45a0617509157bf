"""f-divergence distances over Poisson-kernel rows — B200 device path.

Mirror of ``pathfield/divergence.py`` (same names, signatures, argument
meaning, return types and exceptions); every evaluation runs in the sm_100a
kernels of ``libpathfield_b200.so``:

========================  ==========================================  ==================
function                  reference                                   kernels
========================  ==========================================  ==================
builtin_f/FDivergence     divergence.py:42-104                        (host)
dv_pair                   divergence.py:125-134                       K0 + dense_at
dv_at                     divergence.py:137-151                       K0 + dense_at
dv_field                  divergence.py:154-187                       K0 + K2/K3/generic
sparsify                  divergence.py:194-240                       K4
dv_pair_sparse(_stats)    divergence.py:255-305                       K5/K6/csr_generic
dv_field_sparse           [dv_pair_sparse for q] (no reference API)   K5/K6/csr_generic
dv_field_batch            [dv_field for t] (no reference API)         K7
dv_field_f32              dv_field, FP32 storage (1e-5 tolerance)     dense32
========================  ==========================================  ==================

The divergence between target p and query q is
``DV(q, p) = sum_b max(Q,c) * f(max(P,c)/max(Q,c))`` with the generator's
clamp c (``divergence.py:12-21``).  KL uses the split form (see
``csrc/dense.cu``) with a cancellation guard that falls back, per row, to the
reference's per-element form; every other generator and ``swap_order`` run
the per-element form directly.
"""

from __future__ import annotations

from dataclasses import dataclass, field as dc_field
from typing import Callable

import numpy as np

from . import _device as dev
from . import _native as nat
from . import _userf
from .errors import DivergenceDomainError, InvalidTargetError
from .solvers import PoissonKernel, ScalarField

_CLAMP_LOG = 1e-300      # divergence.py:37
_CLAMP_POWER = 1e-150    # divergence.py:38
_NEG_NOISE = 1e-10       # divergence.py:39

#: Split-form KL guard: rows with |KL| < tau * (|H| + |cross|) are recomputed
#: in per-element form.  The split form's error is ~eps*(|H|+|cross|), so
#: unguarded rows carry at most ~eps/tau ~ 1e-13 relative error.
KL_GUARD_TAU = 1e-3

# PF_DIV_* codes of include/pathfield_b200.h
_KIND = {"kl": 0, "tv": 1, "chi2": 2, "hellinger": 3, "alpha": 4, "power-p": 5}


@dataclass(frozen=True)
class FDivergence:
    """A convex generator f on the positive reals with f(1) = 0 (divergence.py:42-56)."""

    name: str
    f: Callable[[np.ndarray], np.ndarray]
    strictly_convex: bool
    params: dict = dc_field(default_factory=dict)
    clamp: float = _CLAMP_LOG

    def __post_init__(self):
        val = float(self.f(np.array([1.0]))[0])
        if abs(val) > 1e-12:
            raise ValueError(f"f(1) must be 0, got {val} for {self.name}")
        _spot_check_convexity(self.f, self.name)


def _spot_check_convexity(f, name, trials=100):
    # divergence.py:59-67 (host-side validation of a user generator)
    rng = np.random.default_rng(12345)
    x = rng.uniform(1e-3, 10.0, size=(trials, 3))
    x.sort(axis=1)
    lo, mid, hi = x[:, 0], x[:, 1], x[:, 2]
    lam = (hi - mid) / (hi - lo)
    interp = lam * f(lo) + (1.0 - lam) * f(hi)
    if np.any(f(mid) > interp + 1e-9):
        raise ValueError(f"{name} failed the sampled convexity check")


def builtin_f(name: str, *, alpha: float | None = None,
              power: int | None = None) -> FDivergence:
    """Built-in generators, identical to divergence.py:70-104."""
    if name == "tv":
        return FDivergence("tv", lambda x: np.abs(1.0 - x), False, clamp=_CLAMP_POWER)
    if name == "kl":
        return FDivergence("kl", lambda x: -np.log(x), True, clamp=_CLAMP_LOG)
    if name == "chi2":
        return FDivergence("chi2", lambda x: x * x - 1.0, True, clamp=_CLAMP_POWER)
    if name == "hellinger":
        return FDivergence("hellinger", lambda x: (np.sqrt(x) - 1.0) ** 2, True,
                           clamp=_CLAMP_POWER)
    if name == "alpha":
        if alpha is None or alpha in (1.0, -1.0):
            raise ValueError("alpha divergence needs alpha != +-1")
        a = float(alpha)
        scale = 4.0 / (1.0 - a * a)
        expo = (1.0 + a) / 2.0
        return FDivergence("alpha", lambda x: scale * (1.0 - x ** expo), True,
                           {"alpha": a}, clamp=_CLAMP_LOG)
    if name == "power-p":
        if power is None or int(power) < 1 or power != int(power):
            raise ValueError("power-p needs an integer exponent p >= 1")
        p = int(power)
        return FDivergence("power-p", lambda x: np.abs(1.0 - x) ** p, p > 1,
                           {"power": p}, clamp=_CLAMP_POWER)
    raise ValueError(f"unknown divergence {name!r}")


def _kind_param(fd) -> tuple[int, float]:
    """The built-in device functor of a generator; NotImplementedError for a
    user generator on a path that only has built-in kernels (the dense field
    and dv_at paths compile user generators instead, _userf.py)."""
    r = _userf.resolve(fd)
    if r[0] != "builtin":
        raise NotImplementedError(
            f"generator {fd.name!r} is user-defined; this path evaluates the built-in "
            "generators only (divergence.py:70-104); dv_field / dv_at / dv_pair compile it")
    return r[1], r[2]


def _is_builtin(fd, name: str) -> bool:
    """fd is the built-in generator `name` (by expression, not by name alone)."""
    return getattr(fd, "name", None) == name and _userf.builtin_kind(fd) == _KIND[name]


def _effective_clamp(dk, clamp) -> float:
    """Kernel clamp; clamp <= 0 requires P > 0 everywhere (divergence.py:162-165)."""
    if clamp is None or clamp <= 0.0:
        if dk.min_value() <= 0.0:
            raise DivergenceDomainError("zero kernel entries and clamping is disabled")
        return 0.0
    return float(clamp)


class _Staging:
    """Device scratch for K0: clamped target row, its logs, mask.

    With `buf` given (a reused per-(thread, stream) scratch) nothing is allocated."""

    def __init__(self, t, k: int, device, buf=None):
        k_pad, m_pad = dev.round_up(k, 2), dev.round_up(k, 16)
        self.buf = buf if buf is not None else t.empty(16 * k_pad + m_pad, dtype=t.uint8,
                                                      device=device)
        base = self.buf.data_ptr()
        self.tgt = base
        self.logt = base + 8 * k_pad
        self.tmask = base + 16 * k_pad


def _field_device(pk, dk, fd, p: int, swap_order: bool, clamp: float, out_dev, flags_ptr,
                  stream, target_row=None):
    """Launch K0 + the field kernel for slab `dk` into `out_dev` (device)."""
    t = dev.torch()
    k_pad, m_pad = dev.round_up(dk.k, 2), dev.round_up(dk.k, 16)
    st = _Staging(t, dk.k, dk.device, dk.scratch(stream, 16 * k_pad + m_pad, "stage"))
    if target_row is not None:
        row_ptr = target_row.data_ptr()
    elif dk.owns(p):
        row_ptr = dk.row_ptr(p)
    else:
        st.row = dk.target_row(p)  # host copy of a row outside this slab; kept alive on st
        row_ptr = st.row.data_ptr()
    nat.call("pf_target_prep_f64", row_ptr, dk.k, clamp, st.tgt, st.logt, st.tmask,
             flags_ptr, stream)
    gen = _userf.resolve(fd)
    if gen[0] == "user":   # NVRTC-compiled generator (csrc/pf_jit.cu)
        nat.call("pf_dense_user_f64", gen[1].handle, dk.P.data_ptr(), dk.ld, dk.rows, dk.k,
                 st.tgt, st.tmask, clamp, int(bool(swap_order)), dk.row0, p,
                 dk.is_interior.data_ptr(), out_dev.data_ptr(), flags_ptr, stream)
        return st
    kind, param = gen[1], gen[2]
    if kind == 0 and not swap_order:
        H = dk.negentropy(clamp)
        nat.call("pf_dense_kl_f64", dk.P.data_ptr(), dk.ld, dk.rows, dk.k, H.data_ptr(),
                 st.tgt, st.logt, st.tmask, clamp, KL_GUARD_TAU, dk.row0, p,
                 dk.is_interior.data_ptr(), out_dev.data_ptr(), flags_ptr, stream)
    elif kind == 1 and not swap_order:
        nat.call("pf_dense_tv_f64", dk.P.data_ptr(), dk.ld, dk.rows, dk.k, st.tgt, st.tmask,
                 clamp, dk.row0, p, dk.is_interior.data_ptr(), out_dev.data_ptr(),
                 flags_ptr, stream)
    else:
        nat.call("pf_dense_generic_f64", dk.P.data_ptr(), dk.ld, dk.rows, dk.k, st.tgt,
                 st.tmask, clamp, kind, param, int(bool(swap_order)), dk.row0, p,
                 dk.is_interior.data_ptr(), out_dev.data_ptr(), flags_ptr, stream)
    return st  # keep scratch alive until the caller synchronises


def dv_field_device(pk: PoissonKernel, fd: FDivergence, p: int, swap_order: bool = False,
                    clamp: float | None = None):
    """Device-resident field: returns (values tensor (n,) on the GPU, flags tensor).

    Same arithmetic as :func:`dv_field`; nothing is copied back.  Used by the
    tracer and by ``bench.py``'s kernel-only timing.
    """
    if not 0 <= p < pk.n:
        raise InvalidTargetError(f"target {p} out of range")
    t = dev.require_cuda()
    dk = dev.device_kernel(pk)
    if clamp is None:
        clamp = fd.clamp
    c = _effective_clamp(dk, clamp)
    buf = t.empty(dk.rows + 2, dtype=t.float64, device=dk.device)
    flags_ptr = buf.data_ptr() + dk.rows * 8
    stream = t.cuda.current_stream(dk.device).cuda_stream
    st = _field_device(pk, dk, fd, p, swap_order, c, buf, flags_ptr, stream)
    del st
    return buf[:dk.rows], buf[dk.rows:].view(t.int32)


def _to_host(t, dbuf, stream_obj):
    """Device vector -> numpy array owned by the caller (pinned pool, _hostpool.py)."""
    from ._hostpool import to_host
    return to_host(t, dbuf, stream_obj)


def dv_field(pk: PoissonKernel, fd: FDivergence, p: int,
             swap_order: bool = False, clamp: float | None = None) -> ScalarField:
    """Divergence distance from target p to every vertex (divergence.py:154-187)."""
    if not 0 <= p < pk.n:
        raise InvalidTargetError(f"target {p} out of range")
    t = dev.require_cuda()
    dk = dev.device_kernel(pk)
    if clamp is None:
        clamp = fd.clamp
    c = _effective_clamp(dk, clamp)
    if c > 0.0 and dk.boundary_error:   # divergence.py:173-174 indexes with pk.boundary
        raise IndexError(dk.boundary_error)
    s = t.cuda.current_stream(dk.device)
    buf = t.empty(dk.rows + 2, dtype=t.float64, device=dk.device)
    flags_ptr = buf.data_ptr() + dk.rows * 8
    st = _field_device(pk, dk, fd, p, swap_order, c, buf, flags_ptr, s.cuda_stream)
    host = _to_host(t, buf, s)
    del st
    vals = host[:dk.rows]
    # a tracer call on this field (DomainContext.trace) reads the device copy
    dev.register_field(vals, buf[:dk.rows])
    flag_words = host[dk.rows:].view(np.uint32)
    fired = bool(flag_words[0]) and c > 0.0
    params = dict(getattr(fd, "params", {}) or {})
    if swap_order:
        params["swap_order"] = True
    return ScalarField(vals, fd.name, p, params, 1, None, ("clamped",) if fired else ())


from ._hostpool import pinned_view  # noqa: E402


def dv_at(pk: PoissonKernel, fd: FDivergence, p: int, queries,
          swap_order: bool = False, clamp: float | None = None) -> np.ndarray:
    """Distances from target p to a batch of query vertices (divergence.py:137-151)."""
    t = dev.require_cuda()
    dk = dev.device_kernel(pk)
    if clamp is None:
        clamp = fd.clamp
    q = np.asarray(queries, dtype=np.int64)
    if q.size and (q.min() < 0 or q.max() >= pk.n):
        raise IndexError("query index out of range")
    if not 0 <= p < pk.n:
        raise IndexError(f"target {p} out of range")
    # divergence.py:140-148 applies np.maximum(., clamp) directly (no domain check).
    c = float(clamp)
    gen = _userf.resolve(fd)
    s = t.cuda.current_stream(dk.device)
    k_pad, m_pad = dev.round_up(dk.k, 2), dev.round_up(dk.k, 16)
    st = _Staging(t, dk.k, dk.device, dk.scratch(s.cuda_stream, 16 * k_pad + m_pad, "stage"))
    row = dk.target_row(p)
    nat.call("pf_target_prep_f64", row.data_ptr(), dk.k, c, st.tgt, st.logt, st.tmask, 0,
             s.cuda_stream)
    # up to 64K queries are read by the kernel in place from this thread's pinned
    # scratch (mapped under UVA): no H2D copy operation on the critical path;
    # more go up in one copy
    if q.size <= 1 << 16:
        qptr = pinned_view(t, q)
    else:
        qd = t.from_numpy(q).to(dk.device)
        qptr = qd.data_ptr()
    out = t.empty(q.size, dtype=t.float64, device=dk.device)
    if gen[0] == "user":
        nat.call("pf_dense_user_at_f64", gen[1].handle, dk.P.data_ptr(), dk.ld, dk.rows, dk.k,
                 st.tgt, c, int(bool(swap_order)), dk.row0, p, qptr, q.size,
                 out.data_ptr(), s.cuda_stream)
    else:
        nat.call("pf_dense_at_f64", dk.P.data_ptr(), dk.ld, dk.rows, dk.k, st.tgt, c, gen[1],
                 gen[2], int(bool(swap_order)), dk.row0, p, qptr, q.size,
                 out.data_ptr(), s.cuda_stream)
    return _to_host(t, out, s)   # synchronizes the stream: the pinned queries are free


def _settle(value: float) -> float:
    if -_NEG_NOISE < value < 0.0:
        return 0.0
    return value


def dv_pair(pk: PoissonKernel, fd: FDivergence, p: int, q: int,
            swap_order: bool = False, clamp: float | None = None) -> float:
    """Divergence distance between target p and query q (divergence.py:125-134)."""
    if clamp is None:
        clamp = fd.clamp
    if clamp is None or clamp <= 0.0:
        # _clamped_rows (divergence.py:107-112): validate the two rows only.
        if np.any(pk.dense[q] <= 0.0) or np.any(pk.dense[p] <= 0.0):
            raise DivergenceDomainError("zero kernel entry and clamping is disabled")
    val = float(dv_at(pk, fd, p, [q], swap_order=swap_order, clamp=clamp)[0])
    return _settle(val)


# ---------------------------------------------------------------------------
# FP32 storage mode (north-star tolerance 1e-5 relative)
# ---------------------------------------------------------------------------

#: FP32 certification threshold (csrc/dense32.cu): rows below it are re-evaluated in FP64.
F32_GUARD_TAU = 1e-2


def dv_field_f32_device(pk: PoissonKernel, fd: FDivergence, p: int, clamp: float | None = None):
    """KL / TV field with the query rows streamed from an FP32 copy of P (half the
    HBM bytes); values within 1e-5 relative of the FP64 field (rows that the FP32
    rounding bound cannot certify are recomputed from the FP64 rows).
    Returns (values tensor, flags tensor) on the device."""
    if not (_is_builtin(fd, "kl") or _is_builtin(fd, "tv")):
        raise NotImplementedError("FP32 storage mode implements kl and tv")
    if not 0 <= p < pk.n:
        raise InvalidTargetError(f"target {p} out of range")
    t = dev.require_cuda()
    dk = dev.device_kernel(pk)
    c = _effective_clamp(dk, fd.clamp if clamp is None else clamp)
    P32, ld32 = dk.fp32()
    s = t.cuda.current_stream(dk.device)
    out = t.empty(dk.rows + 2, dtype=t.float64, device=dk.device)
    flags = out.data_ptr() + dk.rows * 8
    st = _Staging(t, dk.k, dk.device)
    row = dk.target_row(p)
    nat.call("pf_target_prep_f64", row.data_ptr(), dk.k, c, st.tgt, st.logt, st.tmask, flags,
             s.cuda_stream)
    if _is_builtin(fd, "kl"):
        H64 = dk.negentropy(c)   # H of the FP64 rows: the FP32 rounding only touches the cross term
        nat.call("pf_dense_kl_f32", P32.data_ptr(), ld32, dk.rows, dk.k, H64.data_ptr(), st.tgt,
                 st.logt, st.tmask, c, F32_GUARD_TAU, dk.row0, p, dk.is_interior.data_ptr(),
                 dk.P.data_ptr(), dk.ld, H64.data_ptr(), KL_GUARD_TAU, out.data_ptr(), flags,
                 s.cuda_stream)
    else:
        nat.call("pf_dense_tv_f32", P32.data_ptr(), ld32, dk.rows, dk.k, st.tgt, st.tmask, c,
                 F32_GUARD_TAU, dk.row0, p, dk.is_interior.data_ptr(), dk.P.data_ptr(), dk.ld,
                 out.data_ptr(), flags, s.cuda_stream)
    # clamped flag from the FP64 rows (see pf_mask_compare_f64 in the header)
    if c > 0.0:
        nonuni, ref = dk.mask_nonuniform(c)
        fw = out[dk.rows:].view(t.int32)
        if ref is not None:
            if nonuni:
                fw[0] = 1
            else:
                nat.call("pf_mask_compare_f64", row.data_ptr(), ref.data_ptr(), dk.k, c,
                         fw.data_ptr(), s.cuda_stream)
    del st
    return out[:dk.rows], out[dk.rows:].view(t.int32)


def dv_field_f32(pk: PoissonKernel, fd: FDivergence, p: int, clamp: float | None = None) -> ScalarField:
    """:func:`dv_field` in the FP32 storage mode (additive API; kl and tv)."""
    t = dev.require_cuda()
    vals, flags = dv_field_f32_device(pk, fd, p, clamp)
    s = t.cuda.current_stream(vals.device)
    host = _to_host(t, t.cat([vals, flags.view(t.float64)]), s)
    n = vals.numel()
    fired = bool(host[n:].view(np.uint32)[0])
    return ScalarField(host[:n], fd.name, p, dict(getattr(fd, "params", {}) or {}), 1, None,
                       ("clamped",) if fired else ())


# ---------------------------------------------------------------------------
# Batched targets (K7; no reference API: T x dv_field)
# ---------------------------------------------------------------------------

I8_MAX_K = 4717  # batched_i8.cu: 7 x k x 255^2 < 2^31
#: K7 on a CTA pair (tcgen05 cta_group::2): bitwise the single-CTA kernel's output
I8_CTA_PAIR = True


def guard_list_cap(rows: int, T: int) -> int:
    """Entries of the K7 guarded-pair list (a fuller list falls back to the scan)."""
    return int(min(rows * T, max(1 << 20, rows * T // 128)))


def dv_field_batch_device(pk: PoissonKernel, fd: FDivergence, targets, clamp=None,
                          method: str = "auto"):
    """Fields to T targets at once on the device: (values (n, T) tensor, flags (T,) bool array).

    KL (default order) runs as one contraction with a fused epilogue (K7):
    ``method="i8"`` is the exact-integer emulation of the FP64 GEMM on the
    int8 tensor pipe (tcgen05, batched_i8.cu; within 1e-10 of the reference
    like every FP64 path), ``"i8-f32"`` the same with 15 instead of 34 byte-
    pair GEMMs for the north-star FP32 tolerance (1e-5 relative), ``"f64"``
    the FP64 DMMA GEMM; ``"auto"`` picks i8 when k <= 4717 (falling back to
    f64 for a batch with a target entry above 1).  Any other generator or
    ``swap_order`` is T single-target launches.
    """
    if method not in ("auto", "i8", "i8-f32", "f64"):
        raise ValueError(f"method must be 'auto', 'i8', 'i8-f32' or 'f64', not {method!r}")
    t = dev.require_cuda()
    targets = np.asarray(targets, dtype=np.int64).reshape(-1)
    if targets.size and (targets.min() < 0 or targets.max() >= pk.n):
        raise InvalidTargetError("target out of range")
    dk = dev.device_kernel(pk)
    if clamp is None:
        clamp = fd.clamp
    c = _effective_clamp(dk, clamp)
    T = targets.size
    s = t.cuda.current_stream(dk.device)
    out = t.empty((dk.rows, max(T, 1)), dtype=t.float64, device=dk.device)
    if T == 0:
        return out[:, :0], np.zeros(0, dtype=bool)
    if not _is_builtin(fd, "kl"):
        flags = np.zeros(T, dtype=bool)
        for j, p in enumerate(targets):
            v, f = dv_field_device(pk, fd, int(p), clamp=clamp)
            out[:, j] = v
            flags[j] = bool(f[0].item()) and c > 0.0
        return out, flags
    if not all(dk.owns(int(p)) for p in targets):
        raise NotImplementedError("targets outside this slab: use "
                                  "parallel.ShardedField.field_batch")
    tg = t.from_numpy(targets).to(dk.device)
    Pt = dk.P.index_select(0, tg - dk.row0)
    return _kl_batch_slab(dk, tg, Pt, c, method, out)


def _kl_batch_slab(dk, tg, Pt, c: float, method: str, out=None):
    """K7 over the rows of slab `dk` for the global targets `tg` (device int64)
    whose raw rows are `Pt` (T x >=k, device): (values (rows, T), flags (T,)).

    The per-target ``clamped`` flag is exact for this slab's interior rows;
    over several slabs it is the OR of the slabs' flags."""
    t = dev.torch()
    s = t.cuda.current_stream(dk.device)
    T = int(tg.numel())
    if out is None:
        out = t.empty((dk.rows, max(T, 1)), dtype=t.float64, device=dk.device)
    H = dk.negentropy(c)
    ldl = dev.round_up(dk.k, 16)
    L = t.empty((T, ldl), dtype=t.float64, device=dk.device)
    Tc = t.empty((T, ldl), dtype=t.float64, device=dk.device)
    tflag = t.zeros(T + 1, dtype=t.int32, device=dk.device)
    nonuni, ref = dk.mask_nonuniform(c) if c > 0.0 else (False, None)
    nat.call("pf_batch_prep_f64", Pt.data_ptr(), Pt.stride(0), T, dk.k, ldl, c, nat.ptr(ref),
             L.data_ptr(), Tc.data_ptr(), tflag.data_ptr(), s.cuda_stream)
    use_i8 = method.startswith("i8") or (method == "auto" and dk.k <= I8_MAX_K)
    if use_i8:
        if dk.k > I8_MAX_K:
            raise ValueError(f"method={method!r} needs k <= {I8_MAX_K} (k = {dk.k})")
        tiled = bool(I8_CTA_PAIR)
        eb = t.empty(T, dtype=t.int32, device=dk.device)
        bad = t.zeros(1, dtype=t.int32, device=dk.device)
        if tiled:   # the CTA-pair kernel streams the tiled layout
            A, ea = dk.slices_tiled(c)
            B = t.empty(dev.i8_tiled_bytes(T, dk.k), dtype=t.uint8, device=dk.device)
            nat.call("pf_slice_targets_u8_tiled", L.data_ptr(), ldl, T, dk.k, B.data_ptr(),
                     eb.data_ptr(), bad.data_ptr(), s.cuda_stream)
        else:
            A, ea, ldk = dk.slices(c)
            B = t.empty((7, T, ldk), dtype=t.uint8, device=dk.device)
            nat.call("pf_slice_targets_u8", L.data_ptr(), ldl, T, dk.k, ldk, B.data_ptr(),
                     eb.data_ptr(), bad.data_ptr(), s.cuda_stream)
        if bool(bad.item()):
            if method != "auto":
                raise ValueError(f"method={method!r}: a target row has an entry above 1")
            use_i8 = False
    if use_i8:
        # the epilogue lists its guarded pairs; the fixup walks the list
        cap = guard_list_cap(dk.rows, T)
        glist = dk.scratch(s.cuda_stream, 8 * (cap + 1), "k7_guards").view(t.int64)
        glist[:1].zero_()
        grade = 32 if method == "i8-f32" else 64
        if tiled:
            nat.call("pf_batched_kl_i8_tiled", A.data_ptr(), ea.data_ptr(), dk.rows, B.data_ptr(),
                     eb.data_ptr(), T, dk.k, H.data_ptr(), tg.data_ptr(), KL_GUARD_TAU, dk.row0,
                     out.data_ptr(), out.stride(0), grade, glist.data_ptr(), cap, s.cuda_stream)
        else:
            nat.call("pf_batched_kl_i8_listed", A.data_ptr(), ea.data_ptr(), dk.rows,
                     B.data_ptr(), eb.data_ptr(), T, dk.k, ldk, H.data_ptr(), tg.data_ptr(),
                     KL_GUARD_TAU, dk.row0, out.data_ptr(), out.stride(0), grade, 0,
                     glist.data_ptr(), cap, s.cuda_stream)
        nat.call("pf_batched_kl_fixup_list_f64", dk.P.data_ptr(), dk.ld, dk.rows, dk.k,
                 Tc.data_ptr(), ldl, T, c, out.data_ptr(), out.stride(0),
                 tflag.data_ptr() + 4 * T, glist.data_ptr(), cap, s.cuda_stream)
    else:
        nat.call("pf_batched_kl_f64", dk.P.data_ptr(), dk.ld, dk.rows, dk.k, H.data_ptr(),
                 L.data_ptr(), Tc.data_ptr(), ldl, T, tg.data_ptr(), c, KL_GUARD_TAU, dk.row0,
                 out.data_ptr(), out.stride(0), tflag.data_ptr() + 4 * T, s.cuda_stream)
    tf = tflag.cpu().numpy()
    flags = (nonuni | (tf[:T] != 0)) if (c > 0.0 and ref is not None) else np.zeros(T, bool)
    return out, flags


def dv_field_batch(pk: PoissonKernel, fd: FDivergence, targets, clamp=None,
                   method: str = "auto"):
    """``np.column_stack([dv_field(pk, fd, t).values for t in targets])`` in one pass.

    Returns the (n, T) FP64 array; the per-target ``clamped`` flags are on
    :func:`dv_field_batch_device`.
    """
    t = dev.require_cuda()
    out, flags = dv_field_batch_device(pk, fd, targets, clamp, method)
    return _to_host(t, out, t.cuda.current_stream(out.device))


# ---------------------------------------------------------------------------
# Sparsification and sparse distances (divergence.py:194-305)
# ---------------------------------------------------------------------------

class LogDenseView:
    """``log_dense`` of a sparsified kernel (divergence.py:226), materialised lazily.

    The reference stores an n x k FP64 log matrix eagerly; the device path
    never needs it (the sparse KL reads only the target's log row, computed
    per call), so it is produced on the GPU (``pf_log_clamped_f64``) only
    when someone indexes it.
    """

    def __init__(self, dk):
        self._dk = dk
        self._arr = None
        self.shape = (dk.n, dk.k)
        self.dtype = np.dtype(np.float64)
        self.ndim = 2

    def _materialise(self) -> np.ndarray:
        if self._arr is None:
            t = dev.require_cuda()
            dk = self._dk
            outd = t.empty((dk.rows, dk.k), dtype=t.float64, device=dk.device)
            s = t.cuda.current_stream(dk.device)
            nat.call("pf_log_clamped_f64", dk.P.data_ptr(), dk.ld, dk.rows, dk.k, _CLAMP_LOG,
                     outd.data_ptr(), s.cuda_stream)
            self._arr = _to_host(t, outd, s)
            self._arr.setflags(write=False)
        return self._arr

    def __array__(self, dtype=None, copy=None):
        a = self._materialise()
        return a if dtype is None else a.astype(dtype)

    def __getitem__(self, idx):
        return self._materialise()[idx]

    def __len__(self):
        return self.shape[0]


def _csr_host(data, indices, indptr, shape):
    try:
        import scipy.sparse as sp
        return sp.csr_matrix((data, indices, indptr), shape=shape)
    except Exception:  # scipy absent: same attribute names
        from .solvers import CsrView
        return CsrView(data, indices, indptr, shape)


def sparsify(pk: PoissonKernel, threshold: float | None = None) -> PoissonKernel:
    """Add sparse + log views, dropping entries below threshold/k (divergence.py:194-240).

    The CSR pattern is built on the GPU (K4) and is bit-identical to
    ``csr_matrix`` + ``eliminate_zeros`` of the reference; ``dropped_mass``
    follows scipy's reduceat summation order bit for bit.
    """
    import dataclasses
    import math
    n, k = pk.n, pk.k
    if threshold is None:
        threshold = 1.0 / math.sqrt(n)
    if threshold < 0:
        raise ValueError("threshold must be nonnegative")
    if threshold >= 1.0:
        raise ValueError(f"threshold {threshold} >= 1 would empty rows")
    cut = threshold / k
    t = dev.require_cuda()
    dk = dev.device_kernel(pk)
    dc = dk.csr(cut, threshold == 0)
    s = t.cuda.current_stream(dk.device)
    nnz = dc.nnz
    idx_dtype = np.int32 if nnz < 2 ** 31 else np.int64
    # scipy's layout (row-alignment pads dropped) on the device, then bulk
    # downloads through pinned staging (_hostpool.download)
    from ._hostpool import download
    ip_d, idx_d, dat_d, log_d = dc.scipy_arrays()
    indptr = download(t, ip_d).astype(idx_dtype)
    indices = download(t, idx_d).astype(idx_dtype, copy=False)
    data = download(t, dat_d)
    logs = download(t, log_d)
    dropped = _to_host(t, dc.dropped, s).copy()
    interior = np.ones(n, dtype=bool)
    interior[np.asarray(pk.boundary, dtype=np.int64)] = False
    m = int(interior.sum())
    if m:
        nnz_interior = int(np.diff(indptr.astype(np.int64))[interior].sum())
        sparsity = 100.0 * (1.0 - nnz_interior / (m * k))
    else:
        sparsity = 0.0
    # the reference's log view shares the pattern arrays (divergence.py:224-225)
    return dataclasses.replace(
        pk, threshold=float(threshold), sparse=_csr_host(data, indices, indptr, (n, k)),
        log_sparse=_csr_host(logs, indices, indptr, (n, k)),
        log_dense=LogDenseView(dk), dropped_mass=dropped, row_cut=float(cut),
        sparsity_percent=float(sparsity))


def _device_csr(pk):
    if getattr(pk, "sparse", None) is None or getattr(pk, "log_dense", None) is None:
        raise DivergenceDomainError("kernel has no sparse views; run sparsify")
    dk = dev.device_kernel(pk)
    thr = getattr(pk, "threshold", None)
    return dk, dk.csr(float(pk.row_cut), thr == 0)


def _sparse_launch(pk, fd, p: int, queries=None, want_ops=False):
    """Launch K5/K6 (or the other-generator CSR kernels) for target p over all slab
    rows or `queries`; returns device tensors."""
    t = dev.require_cuda()
    # divergence.py:273-299 dispatches the sparse pair by NAME: kl / alpha over
    # supp(q) with the dense log row, tv over the union plus dropped mass, and
    # every other generator through fd.f over the union with the cut clamp
    name = fd.name
    if name == "alpha":
        kind, param = _KIND["alpha"], float(fd.params["alpha"])
    elif name in ("kl", "tv"):
        kind, param = _KIND[name], 0.0
    else:
        gen = _userf.resolve(fd)
        kind, param = (gen[1], gen[2]) if gen[0] == "builtin" else (-1, 0.0)
    dk, dc = _device_csr(pk)
    s = t.cuda.current_stream(dk.device)
    qd = None
    count = dk.rows
    if queries is not None:
        qd = t.from_numpy(np.asarray(queries, dtype=np.int64)).to(dk.device)
        count = qd.numel()
    out = t.empty(count + 2, dtype=t.float64, device=dk.device)
    flags = out.data_ptr() + count * 8
    out.view(t.int32)[2 * count:2 * count + 4].zero_()
    ops = t.empty(max(count, 1), dtype=t.int64, device=dk.device) if want_ops else None
    qptr = 0 if qd is None else qd.data_ptr()
    k_pad = dev.round_up(dk.k, 2)
    if not dk.owns(p):
        raise NotImplementedError("target row outside this slab: use parallel.ShardedField")
    if name in ("kl", "alpha"):
        st = _Staging(t, dk.k, dk.device)
        nat.call("pf_target_prep_f64", dk.row_ptr(p), dk.k, _CLAMP_LOG, st.tgt, st.logt,
                 st.tmask, flags, s.cuda_stream)
        if name == "kl":
            entry, idx = dc.field_entry("kl")
            nat.call(entry, dc.indptr.data_ptr(), idx,
                     dc.data.data_ptr(), dc.log_data.data_ptr(), dc.hs.data_ptr(), dk.rows,
                     dk.k, st.logt, KL_GUARD_TAU, dk.row0, qptr, count, out.data_ptr(),
                     nat.ptr(ops), flags, 1,
                     s.cuda_stream)
        else:
            nat.call("pf_csr_generic_f64", dc.indptr.data_ptr(), dc.indices.data_ptr(),
                     dc.data.data_ptr(), dc.log_data.data_ptr(), dk.rows, dk.k, kind, param,
                     0.0, 0, -1, st.logt, dk.row0, qptr, count, out.data_ptr(),
                     nat.ptr(ops), s.cuda_stream)
    elif name == "tv":
        st = t.empty(k_pad + 4, dtype=t.float64, device=dk.device)
        nat.call("pf_csr_target_prep_f64", dc.indptr.data_ptr(), dc.indices.data_ptr(),
                 dc.data.data_ptr(), dc.dropped.data_ptr(), p - dk.row0, dk.k, st.data_ptr(),
                 st.data_ptr() + k_pad * 8, s.cuda_stream)
        entry, idx = dc.field_entry("tv")
        nat.call(entry, dc.indptr.data_ptr(), idx, dc.data.data_ptr(),
                 dc.dropped.data_ptr(), dk.rows, dk.k, st.data_ptr(), st.data_ptr() + k_pad * 8,
                 dk.row0, qptr, count, out.data_ptr(), nat.ptr(ops), s.cuda_stream)
    else:
        # chi2 / hellinger / power-p: union form, weights clamped at the row cut
        # (divergence.py:296-299; the clamp when the cut is 0)
        row_cut = getattr(pk, "row_cut", None)
        cut = float(row_cut) if row_cut and row_cut > 0 else float(fd.clamp)
        st = None
        if kind < 0:   # a user generator: the NVRTC-compiled union kernel
            nat.call("pf_csr_user_f64", gen[1].handle, dc.indptr.data_ptr(),
                     dc.indices.data_ptr(), dc.data.data_ptr(), dk.rows, dk.row_ptr(p),
                     p - dk.row0, cut, dk.row0, qptr, count, out.data_ptr(), nat.ptr(ops),
                     s.cuda_stream)
        else:
            nat.call("pf_csr_generic_f64", dc.indptr.data_ptr(), dc.indices.data_ptr(),
                     dc.data.data_ptr(), dc.log_data.data_ptr(), dk.rows, dk.k, kind, param,
                     cut, dk.row_ptr(p), p - dk.row0, 0, dk.row0, qptr, count,
                     out.data_ptr(), nat.ptr(ops), s.cuda_stream)
    return out, ops, count, s, st


def dv_pair_sparse_stats(pk: PoissonKernel, fd: FDivergence, p: int, q: int,
                         swap_order: bool = False) -> tuple[float, int]:
    """Sparse-view divergence plus the summation-slot count (divergence.py:255-299)."""
    if getattr(pk, "sparse", None) is None or getattr(pk, "log_dense", None) is None:
        raise DivergenceDomainError("kernel has no sparse views; run sparsify")
    if swap_order:
        p, q = q, p
    t = dev.require_cuda()
    out, ops, count, s, st = _sparse_launch(pk, fd, int(p), [int(q)], want_ops=True)
    host = _to_host(t, out, s)
    nops = _to_host(t, ops, s)
    del st
    return float(host[0]), int(nops[0])


def dv_pair_sparse(pk: PoissonKernel, fd: FDivergence, p: int, q: int,
                   swap_order: bool = False) -> float:
    """Sparse-view divergence distance between target p and query q (divergence.py:302-305)."""
    return dv_pair_sparse_stats(pk, fd, p, q, swap_order)[0]


def dv_field_sparse(pk: PoissonKernel, fd: FDivergence, p: int) -> ScalarField:
    """Sparse field: ``[dv_pair_sparse(pk, fd, p, q) for q in range(n)]`` in one launch.

    Additive API (the reference has only the per-pair loop).
    """
    if not 0 <= p < pk.n:
        raise InvalidTargetError(f"target {p} out of range")
    t = dev.require_cuda()
    out, ops, count, s, st = _sparse_launch(pk, fd, int(p))
    host = _to_host(t, out, s)
    del st
    vals = host[:count]
    return ScalarField(vals, fd.name, int(p), dict(getattr(fd, "params", {}) or {}), 1, None, ())


def dv_field_sparse_device(pk: PoissonKernel, fd: FDivergence, p: int):
    """Device-resident sparse field (values tensor, flags tensor); used by bench.py."""
    t = dev.require_cuda()
    out, ops, count, s, st = _sparse_launch(pk, fd, int(p))
    return out[:count], out[count:].view(t.int32)


__all__ = [
    "FDivergence", "builtin_f", "dv_pair", "dv_at", "dv_field", "dv_field_device",
    "sparsify", "dv_pair_sparse", "dv_pair_sparse_stats", "dv_field_sparse",
    "dv_field_sparse_device", "dv_field_batch", "dv_field_batch_device", "dv_field_f32",
    "dv_field_f32_device", "LogDenseView", "KL_GUARD_TAU", "F32_GUARD_TAU",
]
