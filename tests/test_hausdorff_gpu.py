"""Path metric on the device (paths.py:326-368): resample_polyline and the
symmetric Hausdorff distance, bitwise against the reference's own outputs
(tests/golden/hausdorff.npz, made by running the reference with cKDTree),
including the default step whose resampled sets reach ~1e7 points."""

import json
from pathlib import Path

import numpy as np
import pytest

import paper_1708_02845_b200 as pf
from oracle import tracer as OT
from tests.conftest import case

pytestmark = pytest.mark.gpu


def _hd():
    return np.load(Path(__file__).resolve().parent / "golden" / "hausdorff.npz")


def test_synthetic_pairs_bitwise():
    g = _hd()
    meta = json.loads(str(g["meta"]))
    for i in range(meta["synthetic"]):
        st = float(g[f"syn/{i}/step"])
        st = None if np.isnan(st) else st
        a, b = g[f"syn/{i}/a"], g[f"syn/{i}/b"]
        assert pf.path_hausdorff(a, b, st) == float(g[f"syn/{i}/h"]), i
        assert np.array_equal(pf.resample_polyline(a, 0.01), g[f"syn/{i}/ra"]), i


@pytest.mark.parametrize("name", ["c1", "corridor50", "disk40", "holes_fine"])
def test_reference_paths_bitwise(name):
    g = _hd()
    meta = json.loads(str(g["meta"]))[name]
    c = case(name)
    pairs = [(c[f"path/kl/{pi}/points"], c[f"path/tv/{pi}/points"])
             for pi in range(meta["npaths"])]
    got = pf.path_hausdorff_batch(pairs, step=meta["step"])
    np.testing.assert_array_equal(got, g[f"{name}/step"])
    got_def = pf.path_hausdorff_batch(pairs)          # default step per pair
    np.testing.assert_array_equal(got_def, g[f"{name}/default"])
    assert np.array_equal(pf.resample_polyline(pairs[0][0], meta["step"]),
                          g[f"{name}/resampled0"])


def test_batch_equals_single_calls_and_oracle():
    rng = np.random.default_rng(3)
    polys = [np.cumsum(rng.standard_normal((int(rng.integers(1, 30)), 2)) * 0.1, axis=0)
             for _ in range(9)]
    polys[2][1] = polys[2][0]                          # zero-length segment
    polys.append(np.repeat([[0.1, 0.2]], 4, axis=0))   # zero-length path
    pairs = [(polys[i], polys[j]) for i in range(len(polys)) for j in range(len(polys))]
    got = pf.path_hausdorff_batch(pairs, step=0.005)
    for q, (a, b) in enumerate(pairs):
        assert got[q] == pf.path_hausdorff(a, b, 0.005) == OT.path_hausdorff(a, b, 0.005), q


def test_traced_path_objects_and_errors():
    c = case("c1")
    mesh_pts = c["path/kl/0/points"]
    tp = pf.TracedPath(np.array(mesh_pts), [("vertex", 0)] * len(mesh_pts), 0, 1, "reached", None)
    assert pf.path_hausdorff(tp, mesh_pts.copy()) == 0.0
    with pytest.raises(ValueError):
        pf.path_hausdorff(np.empty((0, 2)), np.array([[0.0, 0.0]]))
