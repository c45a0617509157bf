"""Full-size parity on REAL Poisson kernels (run on the GPU box; minutes of CPU).

    python tools/validate_real.py c2 > gpurun_out/validate_c2.json

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
import os
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
    # C4: 20 small circular obstacles, n = 1,000,386, k = 4,102
    "c4": {"gen": "holes", "spacing": 0.0017, "size": [2.0, 1.25],
           "holes": [[0.2 + 0.4 * i, 0.16 + 0.31 * j, 0.0034] for i in range(5) for j in range(4)]},
}


def relerr(a, b):
    a, b = np.asarray(a), np.asarray(b)
    same = a == b
    with np.errstate(invalid="ignore", divide="ignore"):
        e = np.where(same, 0.0, np.abs(a - b) / np.maximum(np.abs(b), 1e-300))
    return float(e.max()) if e.size else 0.0, e


def _progress(res, msg, out_path=None):
    res.setdefault("log", []).append([round(time.perf_counter() - _T0, 1), msg])
    print(f"[{time.perf_counter() - _T0:8.1f}s] {msg}", file=sys.stderr, flush=True)
    if out_path:
        Path(out_path).write_text(json.dumps(res))


_T0 = time.perf_counter()


def main(name: str):
    import torch

    import paper_1708_02845_b200 as pf
    from paper_1708_02845_b200 import _device as dev
    from paper_1708_02845_b200 import _native as nat
    from oracle import divergence as O
    from oracle import inputs as I
    from oracle import tracer as TR

    res = {"case": name, "spec": SPECS[name]}
    part = os.environ.get("PF_PARTIAL")  # partial results written after every section
    t0 = time.perf_counter()
    mesh = I.build(SPECS[name])
    res["mesh_s"] = time.perf_counter() - t0
    _progress(res, f"mesh n={mesh.n}", part)
    t0 = time.perf_counter()
    if mesh.n > 200_000:
        dense, boundary = I.poisson_kernel_parallel(mesh, workers=int(os.environ.get("PF_WORKERS", "8")))
    else:
        dense, boundary = I.poisson_kernel(mesh)
    res["poisson_kernel_s"] = time.perf_counter() - t0
    n, k = dense.shape
    _progress(res, f"poisson kernel {n}x{k}", part)
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
    _progress(res, "dense fields", part)

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
    _progress(res, "guard study", part)

    # sparse
    import math
    thr = 1.0 / math.sqrt(n)
    cut = thr / k
    rows = rng.choice(n, min(n, 2000), replace=False)
    if n <= 500_000:
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
        ref_pair = lambda g, q: O.dv_pair_sparse_stats(sv, g, t, int(q))[0]  # noqa: E731
    else:
        # too large for host CSR copies (nnz ~ 2e9): check sampled rows of the device CSR
        import dataclasses
        torch.cuda.synchronize()
        t0 = time.perf_counter()
        dc = dk.csr(cut, False)
        torch.cuda.synchronize()
        res["sparsify_gpu_s"] = time.perf_counter() - t0
        indptr = dc.indptr.cpu().numpy()
        rownnz = dc.rownnz.cpu().numpy()
        dropped = dc.dropped.cpu().numpy()
        ok_pat = ok_drop = True
        for r in rows[:500]:
            a = int(indptr[r]) & ~1
            b = a + int(rownnz[r])  # row-aligned device layout: exclude the pad
            idx = dc.indices[a:b].cpu().numpy()
            dat = dc.data[a:b].cpu().numpy()
            ridx, rval, rdrop = O._kept_row(dense, cut, False, int(r))
            ok_pat &= bool(np.array_equal(idx, ridx) and np.array_equal(dat, rval))
            ok_drop &= bool(dropped[r] == rdrop)
        res["csr_pattern_bitwise_sampled_rows"] = 500
        res["csr_pattern_bitwise"] = ok_pat
        res["dropped_bitwise"] = ok_drop
        res["nnz"] = int(dc.nnz)
        res["sparsity_percent"] = 100.0 * (1.0 - dc.nnz / (n * k))
        spk = dataclasses.replace(pk, threshold=thr, sparse=object(),
                                  log_dense=pf.divergence.LogDenseView(dk), row_cut=cut)
        ref_pair = lambda g, q: O.dv_pair_sparse_direct(dense, t, int(q), g)[0]  # noqa: E731
    sp = []
    for g in ("kl", "tv"):
        fld = pf.dv_field_sparse(spk, pf.builtin_f(g), t)
        refs = np.array([ref_pair(g, q) for q in rows])
        mx, _ = relerr(fld.values[rows], refs)
        sp.append({"gen": g, "rows_checked": int(rows.size), "max_rel_err": mx})
    res["sparse"] = sp
    del spk
    _progress(res, "sparse", part)

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
    _progress(res, "tracer", part)

    # C5 pipeline on the real kernel: T targets as one batched KL contraction
    # (K7), spot-checked against single-target dv_field, then many paths traced
    # on the batched fields (source i -> target i % T) in one launch.
    import torch as _t
    T = int(os.environ.get("PF_BATCH_T", "1024" if n > 500_000 else "256"))
    npaths = int(os.environ.get("PF_PATHS", "10000" if n > 500_000 else "2000"))
    bt = rng.choice(m.interior_vertices, T, replace=False)
    _t.cuda.synchronize()
    t0 = time.perf_counter()
    out, bflags = pf.divergence.dv_field_batch_device(pk, pf.builtin_f("kl"), bt)
    _t.cuda.synchronize()
    batch_s = time.perf_counter() - t0
    worst = 0.0
    for j in range(0, T, max(1, T // 8)):
        single = pf.dv_field(pk, pf.builtin_f("kl"), int(bt[j])).values
        mx, _ = relerr(out[:, j].cpu().numpy(), single)
        worst = max(worst, mx)
    fields = out.t().contiguous()  # (T, n): one field per row for the tracer
    del out
    srcs = rng.choice(m.interior_vertices, npaths)
    fo = np.arange(npaths) % T
    srcs = np.where(srcs == bt[fo], (srcs + 1) % n, srcs)
    from paper_1708_02845_b200 import paths as PP
    PP.trace_arrays(tm, fields, bt, srcs[:256], fo[:256])  # warm-up
    _t.cuda.synchronize()
    t0 = time.perf_counter()
    buf, counts, over, extra = PP.trace_arrays(tm, fields, bt, srcs, fo)
    _t.cuda.synchronize()
    trace_s = time.perf_counter() - t0
    status = buf.status[:npaths].cpu().numpy()
    # bitwise spot check of a few batched paths against the oracle tracer
    spot = 0
    fh = None
    for i in range(0, npaths, max(1, npaths // 10)):
        if fh is None or fh[0] != fo[i]:
            fh = (fo[i], fields[fo[i]].cpu().numpy())
        o = TR.triangle_descent(m.vertices, m.triangles, m.areas, m.bbox_diagonal, fh[1],
                                int(bt[fo[i]]), int(srcs[i]), topo=topo)
        c = int(counts[i])
        a = i * buf.cap
        pts = np.column_stack([buf.x[a:a + c].cpu().numpy(), buf.y[a:a + c].cpu().numpy()])
        spot += int(c == len(o["locations"]) and np.array_equal(pts, o["points"]))
    res["c5_pipeline"] = {"T": T, "batch_kl_s": batch_s,
                          "batch_vs_single_max_rel_err": worst,
                          "clamped_flags": int(np.sum(bflags)),
                          "paths": npaths, "trace_s": trace_s,
                          "reached": int((status == 0).sum()),
                          "stuck": int((status == 1).sum()),
                          "mean_locations": float(counts.mean()),
                          "spot_bitwise": f"{spot}/{len(range(0, npaths, max(1, npaths // 10)))}"}
    _progress(res, "c5 pipeline", part)
    print(json.dumps(res))


if __name__ == "__main__":
    main(sys.argv[1] if len(sys.argv) > 1 else "holes16k")
