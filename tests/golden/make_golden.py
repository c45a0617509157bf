"""Generate golden vectors by running the REFERENCE package itself.

Run in the build container (the only place /root/reference exists):

    python tests/golden/make_golden.py

For every case it builds the mesh with the reference generators, the
Poisson kernel with the reference preprocessing, and records the
reference's own outputs of the hot-path functions (dv_field, dv_at,
dv_pair, sparsify, dv_pair_sparse_stats, triangle_descent).  Meshes and P
are NOT stored (except the tiny disk8 P): the GPU-side tests rebuild them
with oracle/inputs.py and compare against the sha256 digests recorded
here, which proves the rebuilt input is bitwise the reference's.
"""

from __future__ import annotations

import json
import sys
from pathlib import Path

import numpy as np

REF = Path("/root/reference/pkg/src")
HERE = Path(__file__).resolve().parent
ROOT = HERE.parent.parent
sys.path.insert(0, str(REF))
sys.path.insert(0, str(ROOT))

from pathfield import mesh as M  # noqa: E402
from pathfield.divergence import (builtin_f, dv_at, dv_field, dv_pair,  # noqa: E402
                                  dv_pair_sparse_stats, sparsify)
from pathfield.domain import default_endpoints  # noqa: E402
from pathfield.laplacian import assemble_cotan  # noqa: E402
from pathfield.paths import (edge_descent, find_local_minima,  # noqa: E402
                             triangle_descent)
from pathfield.solvers import ScalarField, poisson_kernel  # noqa: E402

from oracle import inputs as I  # noqa: E402

STATUS = {"reached": 0, "stuck": 1, "max-steps-exceeded": 2}

CASES = {
    "disk8": {"gen": "disk", "rings": 8},
    "c1": {"gen": "square_hole"},
    "corridor50": {"gen": "rectangle", "length": 10.0, "width": 0.2, "spacing": 0.05},
    "disk40": {"gen": "disk", "rings": 40},
    "holes_fine": {"gen": "holes", "spacing": 0.0225, "seed": 2, "jitter": 0.35},
}


def ref_mesh(spec):
    spec = dict(spec)
    gen = spec.pop("gen")
    if gen == "square_hole":
        m = I.square_hole_mesh(**spec)  # built from reference private helpers' restatement
        return M.TriMesh(m.vertices, m.triangles)
    fn = {"disk": M.generate_disk_mesh, "rectangle": M.generate_rectangle_mesh,
          "holes": M.generate_holes_mesh}[gen]
    return fn(**spec)


def encode_path(tp):
    kind, i, j, t = [], [], [], []
    for loc in tp.locations:
        if loc[0] == "vertex":
            kind.append(0), i.append(loc[1]), j.append(-1), t.append(0.0)
        else:
            kind.append(1), i.append(loc[1]), j.append(loc[2]), t.append(loc[3])
    return dict(kind=np.array(kind, np.int8), i=np.array(i, np.int64),
                j=np.array(j, np.int64), t=np.array(t, np.float64),
                points=np.array(tp.points, np.float64),
                status=STATUS[tp.status],
                stuck=-1 if tp.stuck_vertex is None else int(tp.stuck_vertex))


def main(only=None):
    for name, spec in CASES.items():
        if only and name not in only:
            continue
        mesh = ref_mesh(spec)
        pk = poisson_kernel(assemble_cotan(mesh))
        P = pk.dense
        n, k = P.shape
        src0, tgt0 = default_endpoints(mesh)
        rng = np.random.default_rng(0)
        interior = mesh.interior_vertices
        targets = [tgt0, int(interior[0]), int(mesh.boundary_vertices[0])]
        targets += [int(x) for x in rng.choice(interior, 2, replace=False)]
        out = {"meta": json.dumps({
            "case": name, "spec": spec, "n": n, "k": k, "targets": targets,
            "source": src0, "target": tgt0,
            "sha_vertices": I.sha(mesh.vertices), "sha_triangles": I.sha(mesh.triangles),
            "sha_P": I.sha(P), "sha_boundary": I.sha(pk.boundary),
            "bbox_diagonal": mesh.bbox_diagonal,
        })}
        if name == "disk8":
            out["P"] = P
            out["boundary"] = pk.boundary
        gens = [("kl", {}), ("tv", {})]
        if name in ("disk8", "c1"):
            gens += [("chi2", {}), ("hellinger", {}), ("alpha", {"alpha": 0.5}),
                     ("power-p", {"power": 3})]
        for gname, kw in gens:
            fd = builtin_f(gname, **kw)
            for ti, t in enumerate(targets):
                f = dv_field(pk, fd, t)
                out[f"field/{gname}/{ti}"] = f.values
                out[f"flags/{gname}/{ti}"] = np.array(len(f.precision_flags) > 0)
            if gname == "kl" and name in ("disk8", "c1"):
                out[f"field_swap/{gname}"] = dv_field(pk, fd, tgt0, swap_order=True).values
            qs = rng.choice(n, min(n, 64), replace=False)
            out[f"at_q/{gname}"] = qs
            out[f"at/{gname}"] = dv_at(pk, fd, tgt0, qs)
            out[f"pair/{gname}"] = np.array([dv_pair(pk, fd, tgt0, int(q)) for q in qs[:8]])
        if name in ("corridor50", "c1", "disk40"):
            spk = sparsify(pk)
            out["sp/indptr"] = spk.sparse.indptr.astype(np.int64)
            out["sp/indices"] = spk.sparse.indices.astype(np.int64)
            out["sp/sha_data"] = np.array(I.sha(spk.sparse.data))
            out["sp/dropped"] = spk.dropped_mass
            out["sp/meta"] = np.array([spk.threshold, spk.row_cut, spk.sparsity_percent])
            sgens = [("kl", {}), ("tv", {})]
            if name in ("corridor50", "c1"):
                sgens += [("chi2", {}), ("hellinger", {}), ("alpha", {"alpha": 0.5}),
                          ("power-p", {"power": 3})]
            for gname, kw in sgens:
                fd = builtin_f(gname, **kw)
                with np.errstate(all="ignore"):
                    vals, ops = zip(*[dv_pair_sparse_stats(spk, fd, tgt0, q) for q in range(n)])
                out[f"spfield/{gname}"] = np.array(vals)
                out[f"spops/{gname}"] = np.array(ops, np.int64)
        # traced paths on the reference's own fields
        npaths = {"disk8": 6, "c1": 12, "corridor50": 12, "disk40": 24, "holes_fine": 24}[name]
        srcs = [src0] + [int(x) for x in rng.choice(interior, npaths - 1, replace=False)]
        srcs = [s for s in srcs if s != tgt0]
        out["path_sources"] = np.array(srcs, np.int64)
        for gname in ("kl", "tv"):
            fld = dv_field(pk, builtin_f(gname), tgt0)
            for pi, s in enumerate(srcs):
                enc = encode_path(triangle_descent(mesh, fld, s))
                for key, val in enc.items():
                    out[f"path/{gname}/{pi}/{key}"] = np.asarray(val)
        # audits: edge walk paths and local minima, on the
        # reference fields and on a noisy field that has spurious minima
        noisy = dv_field(pk, builtin_f("kl"), tgt0).values.copy()
        noisy += np.random.default_rng(5).normal(0.0, 0.02 * noisy.std(), n)
        noisy[tgt0] = 0.0
        out["noisy_field"] = noisy
        for gname in ("kl", "tv", "noisy"):
            vals = noisy if gname == "noisy" else dv_field(pk, builtin_f(gname), tgt0).values
            fld = ScalarField(np.array(vals), "custom-f", tgt0)
            out[f"minima/{gname}"] = np.array(find_local_minima(mesh, fld), np.int64)
            for pi, s in enumerate(srcs[:8]):
                enc = encode_path(edge_descent(mesh, fld, s))
                for key, val in enc.items():
                    out[f"epath/{gname}/{pi}/{key}"] = np.asarray(val)
        np.savez_compressed(HERE / f"{name}.npz", **out)
        print(name, n, k, "targets", targets, "paths", len(srcs))


if __name__ == "__main__":
    main(sys.argv[1:] or None)
