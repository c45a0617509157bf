"""FP32 storage mode: fields within the north-star 1e-5 relative of the reference."""

import numpy as np
import pytest

import paper_1708_02845_b200 as pf
from paper_1708_02845_b200.divergence import dv_field_f32, dv_field_f32_device
from oracle import divergence as O
from oracle import inputs as I
from tests.conftest import CASES, case, rel_close

pytestmark = pytest.mark.gpu
RTOL32 = 1e-5


@pytest.mark.parametrize("name", CASES)
def test_f32_fields_match_reference(name):
    c = case(name)
    pk = pf.PoissonKernel(c.dense, c.boundary, 0.0, 0.0)
    for g in ("kl", "tv"):
        for ti, t in enumerate(c.targets):
            fld = dv_field_f32(pk, pf.builtin_f(g), t)
            ok, err = rel_close(fld.values, c[f"field/{g}/{ti}"], RTOL32)
            assert ok, (name, g, t, err)
            assert (fld.precision_flags == ("clamped",)) == bool(c[f"flags/{g}/{ti}"])
            assert fld.values[t] == 0.0


@pytest.mark.parametrize("spec", [{"gen": "holes", "spacing": 0.0125},
                                  {"gen": "rectangle", "length": 20.0, "width": 1.0, "spacing": 0.05}])
def test_f32_real_kernels(spec):
    mesh = I.build(spec)
    dense, boundary = I.poisson_kernel(mesh)
    pk = pf.PoissonKernel(dense, boundary, 0.0, 0.0)
    src, tgt = I.default_endpoints(mesh)
    for g in ("kl", "tv"):
        vals, flags = dv_field_f32_device(pk, pf.builtin_f(g), tgt)
        got = vals.cpu().numpy()
        ref, fl = O.dv_field(dense, boundary, g, tgt)
        ok, err = rel_close(got, ref, RTOL32)
        assert ok, (g, err)
        guarded = int(flags[1].item())
        print(spec["gen"], g, "guarded rows", guarded, "of", mesh.n, "max rel err", err)
        assert guarded < mesh.n // 2


def test_f32_ragged_k():
    for n, k in [(100, 5), (300, 37), (64, 4250), (513, 1)]:
        dense = I.synthetic_kernel(n, k, seed=k)
        pk = pf.PoissonKernel(dense, np.array([], np.int64), 0.0, 0.0)
        for g in ("kl", "tv"):
            got = dv_field_f32(pk, pf.builtin_f(g), n // 2).values
            ref, _ = O.dv_field(dense, [], g, n // 2)
            ok, err = rel_close(got, ref, RTOL32)
            assert ok, (n, k, g, err)
