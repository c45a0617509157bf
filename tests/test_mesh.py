"""The product's TriMesh mirror and topology builder vs the reference arrays (CPU)."""

import numpy as np
import pytest

import paper_1708_02845_b200 as pf
from paper_1708_02845_b200.mesh import topology
from oracle import inputs as I
from oracle import tracer as TR
from tests.conftest import CASES, case


@pytest.mark.parametrize("name", CASES)
def test_trimesh_mirror_matches_reference(name):
    c = case(name)
    m = c.mesh
    tm = pf.TriMesh(m.vertices, m.triangles)
    assert I.sha(tm.vertices) == c.meta["sha_vertices"]
    assert I.sha(tm.triangles) == c.meta["sha_triangles"]
    np.testing.assert_array_equal(tm.triangle_areas, m.areas)
    np.testing.assert_array_equal(tm.boundary_vertices, m.boundary_vertices)
    assert tm.bbox_diagonal == c.meta["bbox_diagonal"]


@pytest.mark.parametrize("name", CASES)
def test_topology_matches_oracle(name):
    c = case(name)
    m = c.mesh
    mine = topology(m.triangles, m.n)
    ref = TR.topology(m.triangles, m.n)
    for a, b in zip(mine, ref):
        np.testing.assert_array_equal(np.asarray(a, np.int64), np.asarray(b, np.int64))


def test_trimesh_orientation_normalised():
    c = case("disk8")
    m = c.mesh
    tm = pf.TriMesh(m.vertices, m.triangles[:, ::-1])  # all clockwise
    np.testing.assert_array_equal(tm.triangles, m.triangles)


def test_trimesh_validation():
    with pytest.raises(pf.errors.MeshFormatError):
        pf.TriMesh(np.zeros((3, 3)), [[0, 1, 2]])
    with pytest.raises(pf.errors.DegenerateGeometryError):
        pf.TriMesh([[0, 0], [1, 0], [2, 0]], [[0, 1, 2]])
    sq = pf.TriMesh([[0.0, 0.0], [1.0, 0.0], [1.0, 1.0], [0.0, 1.0]], [[0, 1, 2], [0, 2, 3]])
    assert sq.k == 4 and sq.m == 0
    assert sq.edge_adjacency[(0, 2)] == (0, 1)
    assert [list(x) for x in sq.vertex_triangles] == [[0, 1], [0], [0, 1], [1]]
