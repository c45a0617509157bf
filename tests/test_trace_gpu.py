"""K8 batched tracer on the B200 vs the reference's own paths (bit-exact)."""

import numpy as np
import pytest

import paper_1708_02845_b200 as pf
from oracle import tracer as TR
from tests.conftest import CASES, case

pytestmark = pytest.mark.gpu
STATUS = {"reached": 0, "stuck": 1, "max-steps-exceeded": 2}


def _mesh(c):
    m = c.mesh
    return pf.TriMesh(m.vertices, m.triangles)


def _assert_same(path, gold):
    kind = np.array([0 if l[0] == "vertex" else 1 for l in path.locations], np.int8)
    i = np.array([l[1] for l in path.locations], np.int64)
    j = np.array([l[2] if l[0] == "edge" else -1 for l in path.locations], np.int64)
    t = np.array([l[3] if l[0] == "edge" else 0.0 for l in path.locations], np.float64)
    np.testing.assert_array_equal(kind, gold["kind"])
    np.testing.assert_array_equal(i, gold["i"])
    np.testing.assert_array_equal(j, gold["j"])
    np.testing.assert_array_equal(t, gold["t"])
    np.testing.assert_array_equal(path.points, gold["points"])
    assert STATUS[path.status] == int(gold["status"])
    assert (path.stuck_vertex if path.stuck_vertex is not None else -1) == int(gold["stuck"])


@pytest.mark.parametrize("name", CASES)
def test_batch_paths_bitwise_on_reference_field(name):
    c = case(name)
    mesh = _mesh(c)
    srcs = c["path_sources"]
    for g in ("kl", "tv"):
        fld = pf.ScalarField(np.array(c[f"field/{g}/0"]), g, c.target)
        paths = pf.triangle_descent_batch(mesh, fld, srcs)
        for pi, p in enumerate(paths):
            _assert_same(p, c.path(g, pi))
        one = pf.triangle_descent(mesh, fld, int(srcs[0]))
        _assert_same(one, c.path(g, 0))


def test_multi_field_batch_and_overflow_rerun():
    c = case("disk40")
    mesh = _mesh(c)
    srcs = c["path_sources"]
    fk = pf.ScalarField(np.array(c["field/kl/0"]), "kl", c.target)
    ft = pf.ScalarField(np.array(c["field/tv/0"]), "tv", c.target)
    allsrc = np.concatenate([srcs, srcs])
    field_of = np.array([0] * len(srcs) + [1] * len(srcs))
    paths = pf.triangle_descent_batch(mesh, [fk, ft], allsrc, field_of=field_of)
    for pi in range(len(srcs)):
        _assert_same(paths[pi], c.path("kl", pi))
        _assert_same(paths[len(srcs) + pi], c.path("tv", pi))
    # force the overflow path: tiny output capacity, results must be unchanged
    from paper_1708_02845_b200 import paths as P
    buf, counts, over, extra = P.trace_arrays(mesh, [fk], [c.target], srcs, cap=3)
    assert over.size > 0
    out = P._host_paths(buf, counts, over, extra, srcs, np.array([c.target]), None)
    for pi, p in enumerate(out):
        _assert_same(p, c.path("kl", pi))


def test_end_to_end_gpu_field_paths_reach_and_match():
    """Trace on the GPU's own KL field; compare with the oracle traced on the same field
    values (bitwise), and with the reference's golden path (triangle sequence)."""
    c = case("holes_fine")
    mesh = _mesh(c)
    pk = pf.PoissonKernel(c.dense, c.boundary, 0.0, 0.0)
    srcs = c["path_sources"]
    m = c.mesh
    topo = TR.topology(m.triangles, m.n)
    mism = 0
    for g in ("kl", "tv"):
        fld = pf.dv_field(pk, pf.builtin_f(g), c.target)
        paths = pf.triangle_descent_batch(mesh, fld, srcs)
        for pi, (s, p) in enumerate(zip(srcs, paths)):
            assert p.status == "reached"
            o = TR.triangle_descent(m.vertices, m.triangles, m.areas, c.meta["bbox_diagonal"],
                                    fld.values, c.target, int(s), topo=topo)
            np.testing.assert_array_equal(p.points, o["points"])
            assert p.locations == o["locations"]
            gold = c.path(g, pi)
            mism += int(len(p.locations) != len(gold["kind"]) or
                        [l[1] for l in p.locations] != list(gold["i"]))
    assert mism == 0, f"{mism} paths changed their vertex/edge sequence vs the reference field"


def test_stuck_and_cap_and_errors():
    c = case("disk8")
    mesh = _mesh(c)
    vals = np.ones(mesh.n)
    vals[5] = 0.5
    p = pf.triangle_descent(mesh, pf.ScalarField(vals, "custom-f", 0), 5)
    assert p.status == "stuck" and p.stuck_vertex == 5 and len(p.points) == 1
    d = np.hypot(*(mesh.vertices - mesh.vertices[0]).T)
    fld = pf.ScalarField(d, "custom-f", 0)
    p = pf.triangle_descent(mesh, fld, 5, pf.Settings(step_cap_factor=0))
    assert p.status == "max-steps-exceeded" and len(p.points) == 1
    with pytest.raises(pf.InvalidTargetError):
        pf.triangle_descent(mesh, fld, 0)


def test_triangle_gradient_affine_exact():
    c = case("disk8")
    mesh = _mesh(c)
    v = mesh.vertices
    vals = 3.0 * v[:, 0] - 2.0 * v[:, 1] + 7.0
    for ti in range(0, len(mesh.triangles), 17):
        g = pf.triangle_gradient(mesh, vals, ti)
        np.testing.assert_allclose(g, [3.0, -2.0], rtol=0, atol=1e-12)


def test_device_hypot_matches_numpy_on_this_host():
    from paper_1708_02845_b200.paths import np_hypot_device
    rng = np.random.default_rng(0)
    x = rng.standard_normal(50000) * 10.0 ** rng.integers(-8, 8, 50000)
    y = rng.standard_normal(50000) * 10.0 ** rng.integers(-8, 8, 50000)
    got = np_hypot_device(x, y)
    ref = np.hypot(x, y)
    frac = float(np.mean(got == ref))
    print("device hypot == np.hypot on this host:", frac)
    assert frac == 1.0


@pytest.mark.parametrize("name", CASES)
def test_edge_descent_and_local_minima_match_reference(name):
    c = case(name)
    mesh = _mesh(c)
    srcs = c["path_sources"][:8]
    for g in ("kl", "tv", "noisy"):
        vals = c["noisy_field"] if g == "noisy" else c[f"field/{g}/0"]
        fld = pf.ScalarField(np.array(vals), "custom-f", c.target)
        assert pf.find_local_minima(mesh, fld) == [int(x) for x in c[f"minima/{g}"]]
        paths = pf.edge_descent_batch(mesh, fld, srcs)
        for pi, p in enumerate(paths):
            pre = f"epath/{g}/{pi}/"
            gold = {k[len(pre):]: c[k] for k in c.keys() if k.startswith(pre)}
            _assert_same(p, gold)
        one = pf.edge_descent(mesh, fld, int(srcs[0]))
        _assert_same(one, {k[len(f"epath/{g}/0/"):]: c[k] for k in c.keys()
                           if k.startswith(f"epath/{g}/0/")})
