"""Field / path wire formats rendered on the GPU — mirror of ``pathfield/fileio.py``.

The reference formats every value in Python (``f"{v:.17g}"`` per CSV line,
``json.dumps`` → ``float.__repr__`` per JSON element): about a second per
million-vertex field.  Here the digits and the lines are produced by
``csrc/wire.cu`` (exact big-integer digit generation, CPython's layout rules)
and come back as one byte string, identical to the reference's text:

* :func:`field_to_csv`  (fileio.py:37-40, served by service/app.py:108-114)
* :func:`field_to_json` (fileio.py:43-53)
* :func:`path_to_csv`   (fileio.py:72-75)
* :func:`values_to_json_compact` — the service's JSON ``values`` list
  (``[v,v,...]``, starlette's separators, non-finite values rejected like
  ``json.dumps(allow_nan=False)``).

Inputs may be host arrays (the reference's ``ScalarField``/``TracedPath``) or
device tensors (e.g. :func:`~paper_1708_02845_b200.divergence.dv_field_device`),
in which case the values never leave the GPU as numbers.
"""

from __future__ import annotations

import json
import threading

import numpy as np

from . import _device as dev
from . import _native as nat

# line kinds of pf_format_lines (csrc/wire.cu)
_FIELD_CSV, _PATH_CSV, _JSON_INDENT, _JSON_COMPACT, _REPR, _G17 = range(6)
_SLOT = 64


def _device_values(t, values, width: int = 1):
    if hasattr(values, "is_cuda") and values.is_cuda:
        v = values.to(t.float64).contiguous()
    else:
        a = np.ascontiguousarray(values, dtype=np.float64)
        if not a.flags.writeable:  # e.g. ScalarField.values; torch wants a writable buffer
            a = a.copy()
        v = t.from_numpy(a).to(t.device("cuda", t.cuda.current_device()))
    return v.reshape(-1) if width == 1 else v.reshape(-1, width)


_pinned = threading.local()


def _pinned_buffer(t, nbytes: int):
    """Per-thread pinned host staging buffer, grown geometrically (a fresh
    pageable destination costs page faults on every copy)."""
    buf = getattr(_pinned, "buf", None)
    if buf is None or buf.numel() < nbytes:
        buf = t.empty(max(nbytes, 2 * (0 if buf is None else buf.numel()), 1 << 20),
                      dtype=t.uint8, pin_memory=True)
        _pinned.buf = buf
    return buf


def _render(values, kind: int, index0: int = 0, prefix: bytes = b"", suffix: bytes = b"") -> str:
    """prefix + one formatted line of `kind` per value (or (x, y) row) + suffix,
    assembled on the device and decoded once on the host."""
    t = dev.require_cuda()
    width = 2 if kind == _PATH_CSV else 1
    v = _device_values(t, values, width)
    n = v.shape[0]
    if n == 0:
        return (prefix + suffix).decode("ascii")
    s = t.cuda.current_stream(v.device)
    slots = t.empty(n * _SLOT, dtype=t.uint8, device=v.device)
    lens = t.empty(n, dtype=t.int32, device=v.device)
    flag = t.zeros(1, dtype=t.int32, device=v.device)
    nat.call("pf_format_lines", v.data_ptr(), n, kind, index0, slots.data_ptr(), lens.data_ptr(),
             flag.data_ptr(), s.cuda_stream)
    ends = t.cumsum(lens, 0, dtype=t.int64)
    offs = ends - lens + len(prefix)
    stats = t.stack([ends[-1], flag[0].to(t.int64)]).cpu()
    if kind == _JSON_COMPACT and int(stats[1]):
        raise ValueError("Out of range float values are not JSON compliant")
    body = int(stats[0])
    total = len(prefix) + body + len(suffix)
    out = t.empty(total, dtype=t.uint8, device=v.device)
    if prefix:
        out[:len(prefix)].copy_(t.frombuffer(bytearray(prefix), dtype=t.uint8))
    if suffix:
        out[total - len(suffix):].copy_(t.frombuffer(bytearray(suffix), dtype=t.uint8))
    nat.call("pf_pack_lines", slots.data_ptr(), lens.data_ptr(), offs.data_ptr(), n,
             out.data_ptr(), s.cuda_stream)
    host = _pinned_buffer(t, total)[:total]
    host.copy_(out, non_blocking=True)
    s.synchronize()
    return str(host.numpy().data, "ascii")


def format_lines(values, kind: int, index0: int = 0) -> bytes:
    """The packed lines of `kind` for every value, as bytes (testing aid).
    Raises ValueError for non-finite values in compact JSON."""
    return _render(values, kind, index0).encode("ascii")


def field_to_csv(field) -> str:
    """``vertex,value`` then ``f"{i},{v:.17g}"`` per vertex (fileio.py:37-40)."""
    return _render(field.values, _FIELD_CSV, prefix=b"vertex,value\n")


def field_to_json(field) -> str:
    """``json.dumps`` of the field payload with indent=2 (fileio.py:43-53)."""
    values = field.values
    n = int(values.shape[0]) if hasattr(values, "shape") else len(values)
    payload = {
        "kind": field.kind,
        "target": field.target,
        "params": field.params,
        "sign": field.sign,
        "residual": field.residual,
        "precision_flags": list(field.precision_flags),
        "values": ["\0values\0"] if n else [],
    }
    text = json.dumps(payload, indent=2) + "\n"
    if not n:
        return text
    head, tail = text.split(json.dumps("\0values\0"), 1)
    return _render(values, _JSON_INDENT, prefix=head.encode("ascii"),
                   suffix=tail.encode("ascii"))


def path_to_csv(path) -> str:
    """``x,y`` then ``f"{x:.17g},{y:.17g}"`` per point (fileio.py:72-75)."""
    pts = path.points if hasattr(path, "points") else path
    return _render(pts, _PATH_CSV, prefix=b"x,y\n")


def values_to_json_compact(values) -> str:
    """``json.dumps([float(v) for v in values], separators=(",", ":"),
    allow_nan=False)``: the service's JSON ``values`` array."""
    return _render(values, _JSON_COMPACT, prefix=b"[", suffix=b"]")


def format_g17(values) -> list[str]:
    """``[f"{v:.17g}" for v in values]`` (testing aid)."""
    return _split(values, _G17)


def format_repr(values) -> list[str]:
    """``[repr(float(v)) for v in values]`` (testing aid)."""
    return _split(values, _REPR)


def _split(values, kind):
    t = dev.require_cuda()
    v = _device_values(t, values)
    n = v.shape[0]
    if n == 0:
        return []
    s = t.cuda.current_stream(v.device).cuda_stream
    slots = t.empty(n * _SLOT, dtype=t.uint8, device=v.device)
    lens = t.empty(n, dtype=t.int32, device=v.device)
    nat.call("pf_format_lines", v.data_ptr(), n, kind, 0, slots.data_ptr(), lens.data_ptr(), 0, s)
    sl = slots.view(n, _SLOT).cpu().numpy()
    ln = lens.cpu().numpy()
    return [sl[i, :ln[i]].tobytes().decode("ascii") for i in range(n)]


__all__ = ["field_to_csv", "field_to_json", "path_to_csv", "values_to_json_compact",
           "format_lines", "format_g17", "format_repr"]
