"""Full-size parity on REAL Poisson kernels (run on the GPU box; minutes of CPU).

    python scripts/validate_real.py c2 > gpurun_out/validate_c2.json

Builds the config mesh with the reference's generators (oracle/inputs.py,
bitwise the reference's, see tests/test_oracle.py), the Poisson kernel with
the reference preprocessing (SuperLU), then compares on every row:

* dense KL / TV fields (GPU) vs the oracle (numpy restatement, chunked):
  max relative error, guarded rows, the clamp flag; and the KL guard
  threshold study (tau in 1e-3 .. 1e-5: worst unguarded error, guarded rows);
* sparsify: CSR pattern and dropped mass bit-exact; CSR KL / TV fields vs
  the reference's per-pair formulas;
* the tracer: paths from sampled sources on the GPU field vs the oracle
  tracer on the same field values (bitwise).

Prints one JSON object.
"""

from __future__ import annotations

import json
import sys
import time
from pathlib import Path

import numpy as np

ROOT = Path(__file__).resolve().parent.parent
sys.path.insert(0, str(ROOT))

SPECS = {
    "c2": {"gen": "rectangle", "length": 50.0, "width": 1.0, "spacing": 0.024},
    "c2p": {"gen": "rectangle", "length": 1.5, "width": 1.0, "spacing": 0.00405},
    "holes16k": {"gen": "holes", "spacing": 0.0125},
    "holes100k": {"gen": "holes", "spacing": 0.005},
}


def relerr(a, b):
    a, b = np.asarray(a), np.asarray(b)
    same = a == b
    with np.errstate(invalid="ignore", divide="ignore"):
        e = np.where(same, 0.0, np.abs(a - b) / np.maximum(np.abs(b), 1e-300))
    return float(e.max()) if e.size else 0.0, e


def main(name: str):
    import torch

    import paper_1708_02845_b200 as pf
    from paper_1708_02845_b200 import _device as dev
    from paper_1708_02845_b200 import _native as nat
    from oracle import divergence as O
    from oracle import inputs as I
    from oracle import tracer as TR

    res = {"case": name, "spec": SPECS[name]}
    t0 = time.perf_counter()
    mesh = I.build(SPECS[name])
    res["mesh_s"] = time.perf_counter() - t0
    t0 = time.perf_counter()
    dense, boundary = I.poisson_kernel(mesh)
    res["poisson_kernel_s"] = time.perf_counter() - t0
    n, k = dense.shape
    res.update(n=n, k=k)
    src, tgt = I.default_endpoints(mesh)
    rng = np.random.default_rng(0)
    targets = [tgt] + [int(x) for x in rng.choice(mesh.interior_vertices, 2, replace=False)]
    pk = pf.PoissonKernel(dense, boundary, 0.0, 0.0)

    dense_res = []
    for t in targets:
        for g in ("kl", "tv"):
            fld = pf.dv_field(pk, pf.builtin_f(g), t)
            ref = O.dv_field_chunked(dense, g, t, chunk_rows=1024)
            ref[t] = 0.0
            mx, _ = relerr(fld.values, ref)
            flag = O.clamp_flag(dense, boundary, t, O.generator(g)[1])
            dense_res.append({"target": t, "gen": g, "max_rel_err": mx,
                              "flag_ok": (fld.precision_flags == ("clamped",)) == flag})
    res["dense"] = dense_res

    # KL guard threshold study on the first target
    dk = dev.device_kernel(pk)
    t = targets[0]
    ref = O.dv_field_chunked(dense, "kl", t, chunk_rows=1024)
    ref[t] = 0.0
    study = []
    s = torch.cuda.current_stream().cuda_stream
    for tau in (1e-3, 1e-4, 1e-5, 1e-6):
        old = pf.divergence.KL_GUARD_TAU
        pf.divergence.KL_GUARD_TAU = tau
        vals, flags = pf.dv_field_device(pk, pf.builtin_f("kl"), t)
        torch.cuda.synchronize()
        pf.divergence.KL_GUARD_TAU = old
        mx, e = relerr(vals.cpu().numpy(), ref)
        study.append({"tau": tau, "guarded_rows": int(flags[1].item()), "max_rel_err": mx})
    res["kl_guard_study"] = study

    # sparse
    t0 = time.perf_counter()
    spk = pf.sparsify(pk)
    res["sparsify_gpu_s"] = time.perf_counter() - t0
    sv = O.sparsify(dense, boundary)
    res["csr_pattern_bitwise"] = bool(np.array_equal(spk.sparse.indptr, sv["indptr"])
                                      and np.array_equal(spk.sparse.indices, sv["indices"])
                                      and np.array_equal(spk.sparse.data, sv["data"]))
    res["dropped_bitwise"] = bool(np.array_equal(spk.dropped_mass, sv["dropped"]))
    res["nnz"] = int(spk.sparse.nnz)
    res["sparsity_percent"] = spk.sparsity_percent
    rows = rng.choice(n, min(n, 4000), replace=False)
    sp = []
    for g in ("kl", "tv"):
        fld = pf.dv_field_sparse(spk, pf.builtin_f(g), t)
        refs = O.dv_field_sparse(sv, g, t, rows)
        mx, _ = relerr(fld.values[rows], refs)
        sp.append({"gen": g, "rows_checked": int(rows.size), "max_rel_err": mx})
    res["sparse"] = sp

    # tracer on the GPU field vs the oracle tracer on the same values
    m = mesh
    tm = pf.TriMesh(m.vertices, m.triangles)
    topo = TR.topology(m.triangles, m.n)
    srcs = [src] + [int(x) for x in rng.choice(m.interior_vertices, 19, replace=False)]
    srcs = [x for x in srcs if x != tgt]
    tr = []
    for g in ("kl", "tv"):
        fld = pf.dv_field(pk, pf.builtin_f(g), tgt)
        t0 = time.perf_counter()
        paths = pf.triangle_descent_batch(tm, fld, srcs)
        gpu_s = time.perf_counter() - t0
        same = 0
        steps = 0
        t0 = time.perf_counter()
        for s_, p in zip(srcs, paths):
            o = TR.triangle_descent(m.vertices, m.triangles, m.areas, m.bbox_diagonal,
                                    fld.values, tgt, int(s_), topo=topo)
            same += int(np.array_equal(p.points, o["points"]) and p.locations == o["locations"]
                        and p.status == o["status"])
            steps += len(o["locations"])
        cpu_s = time.perf_counter() - t0
        tr.append({"gen": g, "paths": len(srcs), "bitwise_equal": same,
                   "reached": sum(p.status == "reached" for p in paths),
                   "locations": steps, "gpu_batch_s": gpu_s, "oracle_cpu_s": cpu_s})
    res["tracer"] = tr
    print(json.dumps(res))


if __name__ == "__main__":
    main(sys.argv[1] if len(sys.argv) > 1 else "holes16k")
