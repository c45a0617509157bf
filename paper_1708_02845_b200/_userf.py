"""Divergence generators on the device: built-in kernels or NVRTC-compiled user f.

The reference's ``FDivergence(name, f, strictly_convex, params, clamp)``
(divergence.py:42-56) accepts ANY numpy callable f; dv_field / dv_at /
dv_pair evaluate it per element as ``q * f(p / q)`` (:137-187).  The device
path resolves a generator once:

* The name of a built-in (divergence.py:70-104) is NOT trusted by itself: a
  user may build ``FDivergence("kl", my_f, ...)``.  f is traced (below) and
  must give the built-in's expression for that name and params, or at least
  agree with the built-in generator on a fixed set of sample points, to run
  on the hand-written kernels.
* Any other f is traced symbolically: it is called once with a :class:`Sym`
  that records arithmetic, comparisons, ``np.where`` / ``np.clip`` and the
  numpy math ufuncs as a scalar CUDA expression of ``x``.  The expression's
  own numpy evaluator must reproduce f on sample points (within 1e-13
  relative), which rejects anything the trace could not see.  The expression
  is compiled with NVRTC for sm_100a (csrc/pf_jit.cu) and cached per
  expression.
* A generator that cannot be traced (data-dependent Python control flow,
  math-module calls, array-valued captures) raises NotImplementedError:
  there is no CPU fallback.
"""

from __future__ import annotations

import ctypes
import math
import threading

import numpy as np

from . import _native as nat

_KIND = {"kl": 0, "tv": 1, "chi2": 2, "hellinger": 3, "alpha": 4, "power-p": 5}


class TraceError(TypeError):
    """f does something the symbolic trace cannot express."""


def _lit(v) -> str:
    v = float(v)
    if math.isnan(v):
        return "__longlong_as_double(0x7ff8000000000000LL)"
    if math.isinf(v):
        return "__longlong_as_double(0x7ff0000000000000LL)" if v > 0 else \
            "__longlong_as_double((long long)0xfff0000000000000ULL)"
    r = repr(v)   # shortest round-trip decimal: the C++ literal is the same double
    if "e" not in r and "." not in r:
        r += ".0"
    return f"({r})"


class Sym:
    """A scalar expression of x: CUDA source `code` and a numpy evaluator `ev`."""

    __array_priority__ = 1000

    def __init__(self, code: str, ev, boolean: bool = False):
        self.code, self.ev, self.boolean = code, ev, boolean

    # -- refuse what a trace cannot see ---------------------------------------
    def __bool__(self):
        raise TraceError("data-dependent Python control flow in the generator")

    def __float__(self):
        raise TraceError("the generator converts its argument to a Python float")

    __int__ = __index__ = __float__

    def __len__(self):
        raise TraceError("the generator inspects the argument's shape")

    def __iter__(self):
        raise TraceError("the generator iterates over its argument")

    def __getattr__(self, name):
        if name.startswith("__"):   # protocol probes (numpy's __array_interface__ & co.)
            raise AttributeError(name)
        raise TraceError(f"the generator reads attribute {name!r} of its argument")

    # -- arithmetic -----------------------------------------------------------
    @staticmethod
    def wrap(v) -> "Sym":
        if isinstance(v, Sym):
            return v
        if isinstance(v, (bool, np.bool_)):
            return Sym("true" if v else "false", lambda x, v=bool(v): v, True)
        if isinstance(v, (int, float, np.integer, np.floating)) or (
                isinstance(v, np.ndarray) and v.ndim == 0):
            f = float(v)
            return Sym(_lit(f), lambda x, f=f: f)
        raise TraceError(f"the generator combines its argument with {type(v).__name__}")

    def _bin(self, other, op, npf, reverse=False):
        o = Sym.wrap(other)
        a, b = (o, self) if reverse else (self, o)
        return Sym(f"({a.code} {op} {b.code})", lambda x: npf(a.ev(x), b.ev(x)))

    def __add__(self, o):
        return self._bin(o, "+", np.add)

    def __radd__(self, o):
        return self._bin(o, "+", np.add, True)

    def __sub__(self, o):
        return self._bin(o, "-", np.subtract)

    def __rsub__(self, o):
        return self._bin(o, "-", np.subtract, True)

    def __mul__(self, o):
        return self._bin(o, "*", np.multiply)

    def __rmul__(self, o):
        return self._bin(o, "*", np.multiply, True)

    def __truediv__(self, o):
        return self._bin(o, "/", np.true_divide)

    def __rtruediv__(self, o):
        return self._bin(o, "/", np.true_divide, True)

    def __pow__(self, o):
        return _power(self, Sym.wrap(o))

    def __rpow__(self, o):
        return _power(Sym.wrap(o), self)

    def __neg__(self):
        a = self
        return Sym(f"(-{a.code})", lambda x: np.negative(a.ev(x)))

    def __pos__(self):
        return self

    def __abs__(self):
        return _call1("fabs", np.abs, self)

    def _cmp(self, o, op, npf):
        a, b = self, Sym.wrap(o)
        return Sym(f"({a.code} {op} {b.code})", lambda x: npf(a.ev(x), b.ev(x)), True)

    def __lt__(self, o):
        return self._cmp(o, "<", np.less)

    def __le__(self, o):
        return self._cmp(o, "<=", np.less_equal)

    def __gt__(self, o):
        return self._cmp(o, ">", np.greater)

    def __ge__(self, o):
        return self._cmp(o, ">=", np.greater_equal)

    def __eq__(self, o):  # noqa: D105
        return self._cmp(o, "==", np.equal)

    def __ne__(self, o):
        return self._cmp(o, "!=", np.not_equal)

    __hash__ = None

    # -- numpy protocol -------------------------------------------------------
    def __array_ufunc__(self, ufunc, method, *inputs, **kwargs):
        if method != "__call__" or kwargs:
            raise TraceError(f"numpy {ufunc.__name__}.{method} with {sorted(kwargs)}")
        args = [Sym.wrap(a) for a in inputs]
        name = ufunc.__name__
        if name in _UNARY and len(args) == 1:
            return _call1(_UNARY[name], ufunc, args[0])
        if name in _BINOP and len(args) == 2:
            return args[0]._bin(args[1], _BINOP[name], ufunc)
        if name in _CMP and len(args) == 2:
            return args[0]._cmp(args[1], _CMP[name], ufunc)
        if name == "power" and len(args) == 2:
            return _power(args[0], args[1])
        if name in _BINFN and len(args) == 2:
            fn = _BINFN[name]
            a, b = args
            return Sym(f"{fn}({a.code}, {b.code})", lambda x: ufunc(a.ev(x), b.ev(x)))
        if name == "square":
            a = args[0]
            return Sym(f"({a.code} * {a.code})", lambda x: np.square(a.ev(x)))
        if name in ("logical_and", "logical_or"):
            a, b = args
            op = "&&" if name == "logical_and" else "||"
            return Sym(f"({a.code} {op} {b.code})", lambda x: ufunc(a.ev(x), b.ev(x)), True)
        raise TraceError(f"numpy.{name} is not supported on the device")

    def __array_function__(self, func, types, args, kwargs):
        if func is np.where and len(args) == 3 and not kwargs:
            c, a, b = (Sym.wrap(v) for v in args)
            return Sym(f"({c.code} ? {a.code} : {b.code})",
                       lambda x: np.where(c.ev(x), a.ev(x), b.ev(x)))
        if func is np.clip and not kwargs and len(args) == 3:
            v, lo, hi = args
            out = Sym.wrap(v)
            if lo is not None:
                out = np.maximum(out, lo)
            if hi is not None:
                out = np.minimum(out, hi)
            return out
        raise TraceError(f"numpy.{getattr(func, '__name__', func)} is not supported on the device")


_UNARY = {"log": "log", "log2": "log2", "log10": "log10", "log1p": "log1p", "exp": "exp",
          "exp2": "exp2", "expm1": "expm1", "sqrt": "sqrt", "cbrt": "cbrt", "absolute": "fabs",
          "fabs": "fabs", "negative": "-", "sin": "sin", "cos": "cos", "tan": "tan",
          "arcsin": "asin", "arccos": "acos", "arctan": "atan", "sinh": "sinh", "cosh": "cosh",
          "tanh": "tanh", "arcsinh": "asinh", "arccosh": "acosh", "arctanh": "atanh",
          "floor": "floor", "ceil": "ceil", "rint": "rint", "trunc": "trunc",
          "reciprocal": "1.0 /", "positive": "+"}
_BINOP = {"add": "+", "subtract": "-", "multiply": "*", "true_divide": "/", "divide": "/"}
_CMP = {"less": "<", "less_equal": "<=", "greater": ">", "greater_equal": ">=", "equal": "==",
        "not_equal": "!="}
_BINFN = {"maximum": "fmax", "minimum": "fmin", "fmax": "fmax", "fmin": "fmin",
          "hypot": "hypot", "arctan2": "atan2", "copysign": "copysign", "logaddexp": None}
_BINFN.pop("logaddexp")
_NP_OF = {"fabs": np.abs, "-": np.negative, "1.0 /": np.reciprocal, "+": np.positive}


def _call1(fn: str, npf, a: Sym) -> Sym:
    code = f"({fn}({a.code}))" if fn not in ("-", "1.0 /", "+") else f"({fn} ({a.code}))"
    return Sym(code, lambda x: npf(a.ev(x)))


def _power(a: Sym, b: Sym) -> Sym:
    # numpy float power: x ** 2 is a square (fast path), anything else pow()
    if b.code == "(2.0)":
        return Sym(f"({a.code} * {a.code})", lambda x: np.power(a.ev(x), 2.0))
    return Sym(f"pow({a.code}, {b.code})", lambda x: np.power(a.ev(x), b.ev(x)))


_SAMPLES = np.concatenate([
    np.geomspace(1e-300, 1e-3, 61), np.linspace(1e-3, 10.0, 201), np.geomspace(10.0, 1e300, 61),
    [1.0, 0.5, 2.0, 1.0 - 2 ** -40, 1.0 + 2 ** -40]])


def trace(f) -> Sym:
    """Trace generator f into a scalar expression (TraceError if it cannot)."""
    x = Sym("x", lambda v: v)
    with np.errstate(all="ignore"):
        try:
            out = f(x)
        except TraceError:
            raise
        except Exception as exc:  # e.g. math.log(x), x.max(), array captures
            raise TraceError(f"{type(exc).__name__}: {exc}") from exc
    out = Sym.wrap(out) if not isinstance(out, Sym) else out
    if out.boolean:
        raise TraceError("the generator returns a boolean")
    with np.errstate(all="ignore"):
        want = np.asarray(f(_SAMPLES.copy()), dtype=np.float64)
        got = np.broadcast_to(np.asarray(out.ev(_SAMPLES.copy()), dtype=np.float64), want.shape)
    with np.errstate(all="ignore"):
        same = (want == got) | (np.isnan(want) & np.isnan(got)) | (
            np.abs(want - got) <= 1e-13 * np.abs(want))
    if want.shape != _SAMPLES.shape or not bool(same.all()):
        raise TraceError("the traced expression does not reproduce the generator")
    return out


# expressions of the built-in generators (divergence.py:70-104), traced once
def _builtin_code(name: str, params: dict) -> str | None:
    from .divergence import builtin_f
    try:
        if name == "alpha":
            fd = builtin_f(name, alpha=params.get("alpha"))
        elif name == "power-p":
            fd = builtin_f(name, power=params.get("power"))
        else:
            fd = builtin_f(name)
        return trace(fd.f).code
    except Exception:
        return None


_user_lock = threading.Lock()
_user_cache: dict[str, "UserGenerator"] = {}


class UserGenerator:
    """A user generator's kernels (pf_user_compile), compiled for sm_100a and
    loaded on first use (``handle``); ``load=False`` compiles only (no device)."""

    def __init__(self, code: str, load: bool = True):
        self.code, self._h, self._lock = code, None, threading.Lock()
        if not load:
            self._h = self._compile(False)

    def _compile(self, load: bool) -> int:
        h = ctypes.c_void_p(0)
        nat.call("pf_user_compile", self.code.encode(), _nvrtc_path(), int(load), ctypes.byref(h))
        return h.value

    @property
    def handle(self) -> int:
        if self._h is None:
            with self._lock:
                if self._h is None:
                    self._h = self._compile(True)
        return self._h

    def cubin_bytes(self) -> int:
        n = ctypes.c_int64(0)
        nat.call("pf_user_cubin_size", self._h or self.handle, ctypes.byref(n))
        return int(n.value)


def _nvrtc_path() -> bytes | None:
    try:
        import nvidia.cuda_nvrtc  # type: ignore
        from pathlib import Path
        for p in sorted((Path(list(nvidia.cuda_nvrtc.__path__)[0]) / "lib").glob("libnvrtc.so*")):
            return str(p).encode()
    except Exception:
        pass
    return None


_resolved: dict = {}


def resolve(fd):
    """``resolve_uncached`` memoised on the generator callable (weakly) plus
    the name and params it was resolved with."""
    import weakref
    f = fd.f
    name = getattr(fd, "name", None)
    key = (id(f), name, repr(sorted((getattr(fd, "params", {}) or {}).items())))
    hit = _resolved.get(key)
    if hit is not None and hit[0]() is f:
        return hit[1]
    res = resolve_uncached(fd)
    try:
        ref = weakref.ref(f, lambda _r, key=key: _resolved.pop(key, None))
    except TypeError:  # a callable without weakref support: not memoised
        return res
    _resolved[key] = (ref, res)
    return res


def builtin_kind(fd):
    """The PF_DIV_* kind if `fd` is (equivalent to) a built-in generator, else None."""
    r = resolve(fd)
    return r[1] if r[0] == "builtin" else None


def resolve_uncached(fd):
    """("builtin", kind, param) or ("user", UserGenerator) for generator `fd`."""
    name = getattr(fd, "name", None)
    params = dict(getattr(fd, "params", {}) or {})
    try:
        code = trace(fd.f).code
    except TraceError as exc:
        code, err = None, exc
    if name in _KIND:
        want = _builtin_code(name, params)
        if code is not None and code == want:
            return ("builtin",) + _kind_param(name, params)
        if code is None and _agrees_with_builtin(fd, name, params):
            return ("builtin",) + _kind_param(name, params)
    if code is None:
        raise NotImplementedError(
            f"generator {name!r} cannot run on the device: {err} (divergence.py:42-56 "
            "generators must be numpy expressions of x)")
    with _user_lock:
        ug = _user_cache.get(code)
        if ug is None:
            ug = _user_cache[code] = UserGenerator(code)
    return ("user", ug)


def _kind_param(name, params):
    kind = _KIND[name]
    if name == "alpha":
        return kind, float(params["alpha"])
    if name == "power-p":
        return kind, float(params["power"])
    return kind, 0.0


def _agrees_with_builtin(fd, name, params) -> bool:
    """An untraceable f named like a built-in runs the built-in kernel only if
    it equals the built-in generator on the sample points."""
    from .divergence import builtin_f
    try:
        ref = (builtin_f(name, alpha=params.get("alpha")) if name == "alpha" else
               builtin_f(name, power=params.get("power")) if name == "power-p" else
               builtin_f(name))
        with np.errstate(all="ignore"):
            a = np.asarray(fd.f(_SAMPLES.copy()), dtype=np.float64)
            b = np.asarray(ref.f(_SAMPLES.copy()), dtype=np.float64)
        return a.shape == b.shape and bool(((a == b) | (np.isnan(a) & np.isnan(b))).all())
    except Exception:
        return False
