"""The CPU oracle is pinned to the reference's own outputs (tests/golden)."""

import json
from pathlib import Path

import numpy as np
import pytest

from oracle import divergence as O
from oracle import inputs as I
from oracle import tracer as OT
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


STATUS_CODE = {"reached": 0, "stuck": 1, "max-steps-exceeded": 2}


def encode_locs(locs):
    kind = np.array([0 if l[0] == "vertex" else 1 for l in locs], np.int8)
    i = np.array([l[1] for l in locs], np.int64)
    j = np.array([l[2] if l[0] == "edge" else -1 for l in locs], np.int64)
    t = np.array([l[3] if l[0] == "edge" else 0.0 for l in locs], np.float64)
    return kind, i, j, t


@pytest.mark.parametrize("name", CASES)
def test_oracle_tracer_matches_reference_paths(name):
    from oracle import tracer as TR
    c = case(name)
    m = c.mesh
    topo = TR.topology(m.triangles, m.n)
    srcs = c["path_sources"]
    for g in ("kl", "tv"):
        vals = c[f"field/{g}/0"]
        for pi, s in enumerate(srcs):
            gold = c.path(g, pi)
            res = TR.triangle_descent(m.vertices, m.triangles, m.areas, c.meta["bbox_diagonal"],
                                      vals, c.target, int(s), topo=topo)
            kind, i, j, t = encode_locs(res["locations"])
            np.testing.assert_array_equal(kind, gold["kind"])
            np.testing.assert_array_equal(i, gold["i"])
            np.testing.assert_array_equal(j, gold["j"])
            np.testing.assert_array_equal(t, gold["t"])
            np.testing.assert_array_equal(res["points"], gold["points"])
            assert STATUS_CODE[res["status"]] == int(gold["status"])
            assert (res["stuck_vertex"] if res["stuck_vertex"] is not None else -1) == int(gold["stuck"])


def test_topology_matches_reference_lists():
    from oracle import tracer as TR
    c = case("holes_fine")
    m = c.mesh
    vt_ptr, vt_idx, nb_ptr, nb_idx, tri_nbr = TR.topology(m.triangles, m.n)
    # rebuild the reference's lists the way mesh.py:146-157 does
    vt = [[] for _ in range(m.n)]
    for ti, (a, b, cc) in enumerate(m.triangles):
        vt[a].append(ti); vt[b].append(ti); vt[cc].append(ti)
    for v in range(0, m.n, 7):
        assert list(vt_idx[vt_ptr[v]:vt_ptr[v + 1]]) == sorted(vt[v])
    edges = {}
    for ti in range(len(m.triangles)):
        a, b, cc = m.triangles[ti]
        for i, j in ((a, b), (b, cc), (cc, a)):
            edges.setdefault((min(i, j), max(i, j)), []).append(ti)
    for ti in range(0, len(m.triangles), 5):
        for s in range(3):
            i, j = m.triangles[ti][(s + 1) % 3], m.triangles[ti][(s + 2) % 3]
            other = [x for x in edges[(min(i, j), max(i, j))] if x != ti]
            assert tri_nbr[ti, s] == (other[0] if other else -1)
    nbr = [set() for _ in range(m.n)]
    for (i, j) in edges:
        nbr[i].add(j); nbr[j].add(i)
    for v in range(0, m.n, 11):
        assert list(nb_idx[nb_ptr[v]:nb_ptr[v + 1]]) == sorted(nbr[v])


def test_sparse_pair_direct_matches_reference():
    c = case("corridor50")
    for g in ("kl", "tv"):
        for q in range(0, c.n, 37):
            v, ops = O.dv_pair_sparse_direct(c.dense, c.target, q, g)
            ok, err = rel_close([v], [c[f"spfield/{g}"][q]], 1e-14)
            assert ok, (g, q, err)
            assert ops == int(c[f"spops/{g}"][q])


def _hd():
    return np.load(Path(__file__).resolve().parent / "golden" / "hausdorff.npz")


def test_oracle_path_hausdorff_pinned():
    """oracle.tracer.path_hausdorff / resample_polyline == the reference's
    (paths.py:326-368, cKDTree) on the committed golden vectors, bitwise."""
    g = _hd()
    meta = json.loads(str(g["meta"]))
    for i in range(meta["synthetic"]):
        st = float(g[f"syn/{i}/step"])
        st = None if np.isnan(st) else st
        a, b = g[f"syn/{i}/a"], g[f"syn/{i}/b"]
        assert OT.path_hausdorff(a, b, st) == float(g[f"syn/{i}/h"]), i
        assert np.array_equal(OT.resample_polyline(a, 0.01), g[f"syn/{i}/ra"]), i
    for name in ("c1", "corridor50"):
        c = case(name)
        step = meta[name]["step"]
        for pi in range(meta[name]["npaths"]):
            pa, pb = c[f"path/kl/{pi}/points"], c[f"path/tv/{pi}/points"]
            assert OT.path_hausdorff(pa, pb, step) == float(g[f"{name}/step"][pi]), (name, pi)
        assert np.array_equal(OT.resample_polyline(c["path/kl/0/points"], step),
                              g[f"{name}/resampled0"])
