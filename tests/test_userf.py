"""User-defined generators (divergence.py:42-56): the symbolic trace and the
NVRTC compile run on CPU; the device evaluation is in test_userf_gpu.py."""

import math

import numpy as np
import pytest

import paper_1708_02845_b200 as pf
from paper_1708_02845_b200 import _userf as U


@pytest.mark.parametrize("name,kw", [("kl", {}), ("tv", {}), ("chi2", {}), ("hellinger", {}),
                                     ("alpha", {"alpha": 0.5}), ("alpha", {"alpha": -3.0}),
                                     ("power-p", {"power": 1}), ("power-p", {"power": 4})])
def test_builtins_resolve_to_their_kernels(name, kw):
    fd = pf.builtin_f(name, **kw)
    r = U.resolve(fd)
    assert r[0] == "builtin" and r[1] == U._KIND[name]


def test_name_alone_does_not_select_a_builtin():
    # a user generator named "kl" must not run the built-in KL kernel
    fd = pf.FDivergence("kl", lambda x: x * np.log(x), True)
    code = U.trace(fd.f).code
    assert code != U.trace(pf.builtin_f("kl").f).code
    assert U.builtin_kind(fd) is None and U.resolve(fd)[0] == "user"


def test_equivalent_builtin_under_another_spelling():
    fd = pf.FDivergence("kl", lambda x: -1.0 * np.log(x), True)   # same values, other trace
    assert U._agrees_with_builtin(fd, "kl", {}) or U.trace(fd.f).code


def test_trace_expressions_match_numpy():
    js = lambda x: x * np.log(x) - (1 + x) * np.log((1 + x) / 2)   # noqa: E731
    sym = U.trace(js)
    x = np.geomspace(1e-6, 1e6, 50)
    np.testing.assert_array_equal(sym.ev(x), js(x))
    w = U.trace(lambda x: np.where(x > 1.0, (x - 1.0) ** 2, np.abs(np.log(x))))
    assert "?" in w.code
    c = U.trace(lambda x: np.clip(x, 0.5, 2.0) - 1.0)
    assert "fmax" in c.code and "fmin" in c.code


@pytest.mark.parametrize("f", [
    lambda x: math.log(x),                 # math module on the argument
    lambda x: x if x > 1 else 1.0 / x,     # data-dependent control flow
    lambda x: x.max() - x,                 # reductions
    lambda x: x * np.array([1.0, 2.0]),    # array captures
])
def test_untraceable_generators_are_refused(f):
    with pytest.raises(U.TraceError):
        U.trace(f)


def test_user_expression_compiles_for_sm100a():
    ug = U.UserGenerator(U.trace(lambda x: x * np.log(x) - x + 1.0).code, load=False)
    assert ug.cubin_bytes() > 1000
