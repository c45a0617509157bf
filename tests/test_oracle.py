"""The CPU oracle is pinned to the reference's own outputs (tests/golden)."""

import numpy as np
import pytest

from oracle import divergence as O
from oracle import inputs as I
from tests.conftest import CASES, case, rel_close

GENS = {"kl": {}, "tv": {}, "chi2": {}, "hellinger": {}, "alpha": {"alpha": 0.5},
        "power-p": {"power": 3}}


@pytest.mark.parametrize("name", CASES)
def test_inputs_rebuild_bitwise(name):
    c = case(name)
    m = c.mesh
    assert I.sha(m.vertices) == c.meta["sha_vertices"]
    assert I.sha(m.triangles) == c.meta["sha_triangles"]
    assert I.sha(c.boundary) == c.meta["sha_boundary"]
    assert c.input_matches_reference()


@pytest.mark.parametrize("name", CASES)
def test_oracle_dense_fields_match_reference(name):
    c = case(name)
    with np.errstate(over="ignore", divide="ignore", invalid="ignore"):
        for key in c.keys():
            if not key.startswith("field/"):
                continue
            _, g, ti = key.split("/")
            t = c.targets[int(ti)]
            vals, flags = O.dv_field(c.dense, c.boundary, g, t, **GENS[g])
            np.testing.assert_array_equal(vals, c[key])  # same numpy arithmetic: bitwise
            assert bool(flags) == bool(c[f"flags/{g}/{ti}"])
            assert O.clamp_flag(c.dense, c.boundary, t, O.generator(g, **GENS[g])[1]) == bool(flags)


@pytest.mark.parametrize("name", CASES)
def test_oracle_at_and_pair(name):
    c = case(name)
    with np.errstate(over="ignore", divide="ignore", invalid="ignore"):
        for g in GENS:
            if f"at/{g}" not in c.keys():
                continue
            qs = c[f"at_q/{g}"]
            np.testing.assert_array_equal(O.dv_at(c.dense, g, c.target, qs, **GENS[g]), c[f"at/{g}"])
            pairs = [O.dv_pair(c.dense, g, c.target, int(q), **GENS[g]) for q in qs[:8]]
            ok, err = rel_close(pairs, c[f"pair/{g}"], 1e-12)
            assert ok, err


@pytest.mark.parametrize("name", ["c1", "corridor50"])
def test_oracle_chunked_equals_field(name):
    c = case(name)
    full = c["field/kl/0"]
    got = O.dv_field_chunked(c.dense, "kl", c.target, chunk_rows=100, threads=4)
    got[c.target] = 0.0
    np.testing.assert_array_equal(got, full)


@pytest.mark.parametrize("name", ["c1", "corridor50", "disk40"])
def test_oracle_sparsify_and_sparse_pairs(name):
    c = case(name)
    sv = O.sparsify(c.dense, c.boundary)
    np.testing.assert_array_equal(sv["indptr"], c["sp/indptr"])
    np.testing.assert_array_equal(sv["indices"], c["sp/indices"])
    assert I.sha(sv["data"]) == str(c["sp/sha_data"])
    thr, cut, spct = c["sp/meta"]
    assert sv["threshold"] == thr and sv["row_cut"] == cut
    assert abs(sv["sparsity_percent"] - spct) < 1e-12
    np.testing.assert_array_equal(sv["dropped"], c["sp/dropped"])
    rows = range(0, c.n, max(1, c.n // 200))
    for g in ("kl", "tv"):
        got = O.dv_field_sparse(sv, g, c.target, rows)
        ok, err = rel_close(got, c[f"spfield/{g}"][list(rows)], 1e-12)
        assert ok, (g, err)
