"""Golden vectors for the path metric (paths.py:326-368), from the REFERENCE.

Run in the build container (the only place /root/reference exists), after
make_golden.py:

    python tests/golden/make_golden_hausdorff.py

Inputs are the reference's own traced paths stored in the case goldens (KL
path i vs TV path i of each case, at the mesh scale step the reference's
DomainContext.compare uses, domain.py:113, and at the default step) plus
synthetic polylines covering the edge cases of resample_polyline (single
points, zero-length segments and paths, offset straight lines as in
test_paths.py:185-200).  Writes tests/golden/hausdorff.npz.
"""

from __future__ import annotations

import json
import sys
from pathlib import Path

import numpy as np

REF = Path("/root/reference/pkg/src")
HERE = Path(__file__).resolve().parent
sys.path.insert(0, str(REF))
sys.path.insert(0, str(HERE.parent.parent))

from pathfield.paths import path_hausdorff, resample_polyline  # noqa: E402

from tests.golden.make_golden import CASES, ref_mesh  # noqa: E402


def synthetic():
    rng = np.random.default_rng(7)
    out = []
    a = np.column_stack([np.linspace(0, 1, 11), np.zeros(11)])
    out.append((a, a + [0.0, 0.3], 0.01))                 # test_paths.py:190
    out.append((a, a.copy(), None))                       # identical -> 0
    out.append((np.array([[0.2, 0.1]]), a, 0.05))         # single point vs line
    out.append((np.array([[0.2, 0.1]]), np.array([[0.5, -0.3]]), None))
    z = np.repeat([[0.3, 0.4]], 5, axis=0)
    out.append((z, a, 0.02))                              # zero-length path
    for trial in range(12):
        na, nb = rng.integers(2, 40, 2)
        p = np.cumsum(rng.standard_normal((na, 2)) * 0.1, axis=0)
        q = np.cumsum(rng.standard_normal((nb, 2)) * 0.1, axis=0) + rng.standard_normal(2) * 0.1
        if na > 4:
            p[3] = p[2]                                   # zero-length segment
        out.append((p, q, None if trial % 2 else 0.004))
    return out


def main():
    out = {}
    meta = {}
    for name in ("c1", "corridor50", "disk40", "holes_fine"):
        g = np.load(HERE / f"{name}.npz")
        npaths = len(g["path_sources"])
        mesh = ref_mesh(CASES[name])
        step = mesh.min_edge_length() / 4.0
        meta[name] = {"npaths": int(npaths), "step": step}
        vals_step, vals_def = [], []
        for pi in range(npaths):
            pa = g[f"path/kl/{pi}/points"]
            pb = g[f"path/tv/{pi}/points"]
            vals_step.append(path_hausdorff(pa, pb, step=step))
            vals_def.append(path_hausdorff(pa, pb))
        out[f"{name}/step"] = np.array(vals_step)
        out[f"{name}/default"] = np.array(vals_def)
        out[f"{name}/resampled0"] = resample_polyline(g["path/kl/0/points"], step)
    syn = synthetic()
    meta["synthetic"] = len(syn)
    for i, (p, q, st) in enumerate(syn):
        out[f"syn/{i}/a"] = p
        out[f"syn/{i}/b"] = q
        out[f"syn/{i}/step"] = np.array(np.nan if st is None else st)
        out[f"syn/{i}/h"] = np.array(path_hausdorff(p, q, step=st))
        out[f"syn/{i}/ra"] = resample_polyline(p, 0.01)
    out["meta"] = json.dumps(meta)
    np.savez_compressed(HERE / "hausdorff.npz", **out)
    print(json.dumps(meta))


if __name__ == "__main__":
    main()
