"""CPU checks of the C ABI boundary: the library loads and exports every
entry point declared in include/pathfield_b200.h; host-side validation
raises the reference's exception types before anything is launched."""

import numpy as np
import pytest

import paper_1708_02845_b200 as pf
from paper_1708_02845_b200 import _native as nat


def test_header_symbols_exported():
    declared = nat.header_symbols()
    assert "pf_dense_kl_f64" in declared and "pf_dense_tv_f64" in declared
    lib = nat.load()
    missing = [s for s in declared if not hasattr(lib, s)]
    assert not missing, missing
    assert set(nat._SIGS) >= set(declared), set(declared) - set(nat._SIGS)


def test_version_and_error_string():
    lib = nat.load()
    assert lib.pf_version() >= 1
    assert isinstance(lib.pf_last_error(), bytes)


def test_argument_errors_without_launch():
    # validation failures return an error code, not a launch
    lib = nat.load()
    rc = lib.pf_dense_kl_f64(0, 4, 10, 4, 0, 0, 0, 0, 1e-300, 1e-3, 0, 0, 0, 0, 0, 0)
    assert rc != 0
    assert b"null" in lib.pf_last_error()
    rc = lib.pf_row_negentropy_f64(8, 3, 10, 3, 1e-300, 16, 0, 0)  # odd ld
    assert rc == -2  # PF_E_ALIGN


def _pk():
    dense = np.array([[0.5, 0.5, 0.0], [0.2, 0.3, 0.5], [0.0, 0.0, 1.0]])
    return pf.PoissonKernel(dense, np.array([2]), 0.0, 0.0)


def test_invalid_target_raises_reference_type():
    with pytest.raises(pf.InvalidTargetError):
        pf.dv_field(_pk(), pf.builtin_f("kl"), 5)
    with pytest.raises(pf.InvalidTargetError):
        pf.dv_field(_pk(), pf.builtin_f("kl"), -1)


def test_builtin_generators_mirror_reference():
    for name, kw in [("tv", {}), ("kl", {}), ("chi2", {}), ("hellinger", {}),
                     ("alpha", {"alpha": 0.5}), ("power-p", {"power": 3})]:
        fd = pf.builtin_f(name, **kw)
        assert abs(float(fd.f(np.array([1.0]))[0])) < 1e-12
    with pytest.raises(ValueError):
        pf.builtin_f("alpha", alpha=1.0)
    with pytest.raises(ValueError):
        pf.builtin_f("power-p", power=0)
    with pytest.raises(ValueError):
        pf.builtin_f("nope")
    with pytest.raises(ValueError):
        pf.FDivergence("bad-offset", lambda x: x, True)
    assert pf.builtin_f("kl").clamp == 1e-300 and pf.builtin_f("tv").clamp == 1e-150


def test_no_cpu_fallback():
    import torch
    if torch.cuda.is_available():
        pytest.skip("GPU present")
    with pytest.raises(pf.NativeError):
        pf.dv_field(_pk(), pf.builtin_f("kl"), 0)
