"""K7 batched-target KL (one FP64 GEMM + fused epilogue) vs T x dv_field."""

import numpy as np
import pytest

import paper_1708_02845_b200 as pf
from oracle import divergence as O
from oracle import inputs as I
from tests.conftest import CASES, case, rel_close

pytestmark = pytest.mark.gpu
RTOL = 1e-10


@pytest.mark.parametrize("name", CASES)
def test_batch_matches_reference_fields(name):
    c = case(name)
    pk = pf.PoissonKernel(c.dense, c.boundary, 0.0, 0.0)
    targets = c.targets
    out, flags = pf.divergence.dv_field_batch_device(pk, pf.builtin_f("kl"), targets)
    got = out.cpu().numpy()
    for j, t in enumerate(targets):
        ok, err = rel_close(got[:, j], c[f"field/kl/{j}"], RTOL)
        assert ok, (name, j, err)
        assert bool(flags[j]) == bool(c[f"flags/kl/{j}"])
    host = pf.dv_field_batch(pk, pf.builtin_f("kl"), targets)
    np.testing.assert_array_equal(host, got)


def test_batch_equals_single_target_calls_large_T():
    # T spanning several 128-wide target tiles and a ragged row tile
    mesh = I.build({"gen": "holes", "spacing": 0.03, "seed": 1})
    dense, boundary = I.poisson_kernel(mesh)
    pk = pf.PoissonKernel(dense, boundary, 0.0, 0.0)
    rng = np.random.default_rng(3)
    targets = rng.choice(mesh.n, 300, replace=False)
    got = pf.dv_field_batch(pk, pf.builtin_f("kl"), targets)
    for j in range(0, 300, 23):
        ref, _ = O.dv_field(dense, boundary, "kl", int(targets[j]))
        ok, err = rel_close(got[:, j], ref, RTOL)
        assert ok, (j, err)


def test_batch_flags_nonuniform_masks_and_other_generators():
    dense = I.synthetic_kernel(700, 67, seed=4)
    dense[::7, 3] = 0.0          # interior rows with different zero patterns
    boundary = np.array([1, 5])
    pk = pf.PoissonKernel(dense, boundary, 0.0, 0.0)
    targets = [0, 7, 100, 699]
    out, flags = pf.divergence.dv_field_batch_device(pk, pf.builtin_f("kl"), targets)
    got = out.cpu().numpy()
    for j, t in enumerate(targets):
        ref, fl = O.dv_field(dense, boundary, "kl", t)
        ok, err = rel_close(got[:, j], ref, RTOL)
        assert ok, err
        assert bool(flags[j]) == bool(fl)
    tv = pf.dv_field_batch(pk, pf.builtin_f("tv"), targets)
    for j, t in enumerate(targets):
        ref, _ = O.dv_field(dense, boundary, "tv", t)
        ok, err = rel_close(tv[:, j], ref, RTOL)
        assert ok, err
