"""Wire formats on the device (csrc/wire.cu) against the reference's own
expressions (fileio.py:37-75: f"{i},{v:.17g}", json.dumps -> float.__repr__),
byte for byte, on the golden fields and on values spanning every binade,
subnormals, signed zeros and non-finite values."""

import json

import numpy as np
import pytest

import paper_1708_02845_b200 as pf
from paper_1708_02845_b200 import fileio as F
from tests.conftest import case

pytestmark = pytest.mark.gpu


def edge_values():
    v = [0.0, -0.0, 1.0, -1.0, 0.1, 0.5, 1e16, 1e17, 2e16 + 8, 1e-4, 1e-5, 9.999999999999999e22,
         5e-324, 2.2250738585072014e-308, 2.225073858507201e-308, 1.7976931348623157e308,
         2.0 ** 60, 123456789012345678.0, 0.3, 2.0 / 3, 1e23, 8.41e21, 5e-310, 1e22, 1e21,
         9007199254740993.0, 4.35e-7, 1234.5, 0.000123456789, 1e-300, 6.6e-75]
    v += [2.0 ** e for e in range(-1074, 1024)]
    v += [float(np.nextafter(2.0 ** e, 0)) for e in range(-1020, 1024, 3)]
    v += [10.0 ** e for e in range(-323, 309)]
    v += [float(np.nextafter(10.0 ** e, np.inf)) for e in range(-300, 300, 7)]
    return np.array(v + [-x for x in v[:400]])


def random_values(n, seed):
    rng = np.random.default_rng(seed)
    bits = rng.integers(0, 2 ** 63, n, dtype=np.int64).view(np.float64)
    bits = bits[np.isfinite(bits)]
    sign = np.where(rng.random(bits.size) < 0.5, -1.0, 1.0)
    mags = rng.random(n) * 10.0 ** rng.integers(-20, 20, n)
    return np.concatenate([bits * sign, mags])


@pytest.mark.parametrize("vals", ["edge", "random"])
def test_digits_match_cpython(vals):
    v = edge_values() if vals == "edge" else random_values(200_000, 5)
    g = F.format_g17(v)
    r = F.format_repr(v)
    bad_g = [(x, a) for x, a in zip(v, g) if a != f"{float(x):.17g}"]
    bad_r = [(x, a) for x, a in zip(v, r) if a != repr(float(x))]
    assert not bad_g[:5] and not bad_r[:5], (bad_g[:5], bad_r[:5])


def test_nonfinite_spellings():
    v = np.array([np.nan, np.inf, -np.inf, 1.5])
    assert F.format_g17(v) == ["nan", "inf", "-inf", "1.5"]
    assert F.format_repr(v) == ["nan", "inf", "-inf", "1.5"]
    body = F.format_lines(v, 2).decode()
    assert body == "NaN,\n    Infinity,\n    -Infinity,\n    1.5"
    with pytest.raises(ValueError):
        F.values_to_json_compact(v)


def _ref_csv(values):                       # fileio.py:37-40
    lines = ["vertex,value"]
    lines.extend(f"{i},{v:.17g}" for i, v in enumerate(values))
    return "\n".join(lines) + "\n"


def _ref_json(f):                           # fileio.py:43-53
    payload = {"kind": f.kind, "target": f.target, "params": f.params, "sign": f.sign,
               "residual": f.residual, "precision_flags": list(f.precision_flags),
               "values": [float(v) for v in f.values]}
    return json.dumps(payload, indent=2) + "\n"


@pytest.mark.parametrize("name", ["c1", "holes_fine"])
def test_field_files_byte_identical(name):
    c = case(name)
    pk = pf.PoissonKernel(c.dense, c.boundary, 0.0, 0.0)
    for g in ("kl", "tv"):
        fld = pf.dv_field(pk, pf.builtin_f(g), c.target)
        assert F.field_to_csv(fld) == _ref_csv(fld.values)
        assert F.field_to_json(fld) == _ref_json(fld)
        vals, _ = pf.dv_field_device(pk, pf.builtin_f(g), c.target)   # straight from HBM
        assert F.format_lines(vals, 0).decode() == _ref_csv(fld.values)[len("vertex,value\n"):]
        assert F.values_to_json_compact(fld.values) == json.dumps(
            [float(v) for v in fld.values], separators=(",", ":"), allow_nan=False)
    pts = c["path/kl/0/points"]
    ref = "x,y\n" + "".join(f"{x:.17g},{y:.17g}\n" for x, y in pts)  # fileio.py:72-75
    assert F.path_to_csv(np.array(pts)) == ref


def test_empty_field():
    f = pf.ScalarField(np.zeros(0), "kl", 0)
    assert F.field_to_csv(f) == "vertex,value\n"
    assert F.field_to_json(f) == _ref_json(f)
