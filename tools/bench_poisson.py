"""Time (and optionally validate) the device Poisson kernel at full size.

    python tools/bench_poisson.py c2 [--validate] [--leaf 64] [--reps 3]

Phases: host plan (nd_plan.cpp), device Laplacian, multifrontal factor,
forward + backward solves and finalize (CUDA events on the launch stream).
--validate rebuilds the reference P with SuperLU (oracle/inputs.py,
poisson_kernel_parallel: the reference's factor + solve in column chunks on
all host cores) and compares componentwise, plus dense KL/TV fields.
"""

from __future__ import annotations

import argparse
import json
import os
import sys
import time
from pathlib import Path

import numpy as np

ROOT = Path(__file__).resolve().parent.parent
sys.path.insert(0, str(ROOT))

SPECS = {
    "c1": {"gen": "square_hole"},
    "c2": {"gen": "rectangle", "length": 50.0, "width": 1.0, "spacing": 0.024},
    "c2p": {"gen": "rectangle", "length": 1.5, "width": 1.0, "spacing": 0.00405},
    "holes100k": {"gen": "holes", "spacing": 0.005},
    "c4": {"gen": "holes", "spacing": 0.0017, "size": [2.0, 1.25],
           "holes": [[0.2 + 0.4 * i, 0.16 + 0.31 * j, 0.0034] for i in range(5) for j in range(4)]},
}


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("config", default="c2", nargs="?")
    ap.add_argument("--validate", action="store_true")
    ap.add_argument("--leaf", type=int, default=None)
    ap.add_argument("--reps", type=int, default=3)
    ap.add_argument("--workers", type=int, default=os.cpu_count() or 8)
    ap.add_argument("--slabs", type=int, default=0,
                    help="also time the row-slab builds of N ranks (one after another)")
    args = ap.parse_args()
    import torch
    from oracle import inputs as I
    import paper_1708_02845_b200.laplacian as L
    out = {"config": args.config, "spec": SPECS[args.config]}
    t0 = time.perf_counter()
    mesh = I.build(SPECS[args.config])
    out["mesh_s"] = time.perf_counter() - t0
    leaf = args.leaf or L.LEAF
    t0 = time.perf_counter()
    dp = L.DevicePoisson(mesh, leaf=leaf)
    out["setup_s"] = time.perf_counter() - t0  # topology + host plan + uploads
    t0 = time.perf_counter()
    L.NdPlan.from_mesh(mesh, leaf=leaf)
    out["plan_s"] = time.perf_counter() - t0
    out["stats"] = dp.plan.stats
    ev = lambda: torch.cuda.Event(enable_timing=True)  # noqa: E731
    P = None
    reps = []
    for rep in range(args.reps + 1):
        dp._lap, dp._F = None, None
        torch.cuda.synchronize()
        e0, e1, e2, e3 = ev(), ev(), ev(), ev()
        e0.record()
        dp.laplacian()
        e1.record()
        dp.factor()
        e2.record()
        P, residual, rse = dp.solve(P)
        e3.record()
        torch.cuda.synchronize()
        if rep:  # first pass warms up
            reps.append({"laplacian_ms": e0.elapsed_time(e1), "factor_ms": e1.elapsed_time(e2),
                         "solve_ms": e2.elapsed_time(e3), "total_ms": e0.elapsed_time(e3)})
    out["reps"] = reps
    out["median_total_ms"] = float(np.median([r["total_ms"] for r in reps]))
    out["residual"], out["row_sum_error"] = residual, rse
    n, k = dp.n, dp.k
    out["P_bytes"] = n * k * 8
    out["write_gbs"] = n * k * 8 / (np.median([r["solve_ms"] for r in reps]) * 1e-3) / 1e9
    print(json.dumps(out), flush=True)
    if args.slabs:
        from paper_1708_02845_b200.parallel import partition_rows
        sl = []
        for a, b in partition_rows(dp.n, args.slabs):
            dp.slab_plan(a, b - a)  # host plan outside the timing
            times = []
            for rep in range(3):
                ev0, ev1 = ev(), ev()
                torch.cuda.synchronize()
                ev0.record()
                Ps, r_, s_ = dp.solve(slab=(a, b - a))
                ev1.record()
                torch.cuda.synchronize()
                times.append(ev0.elapsed_time(ev1))
                del Ps
            spl = dp.slab_plan(a, b - a)
            sl.append({"rows": [a, b], "solve_ms": float(np.median(times)),
                       "fronts": spl["fronts"], "scratch_rows": spl["scratch_rows"]})
        fac = float(np.median([r["factor_ms"] + r["laplacian_ms"] for r in reps]))
        print(json.dumps({"slabs": args.slabs, "factor_ms_replicated": fac,
                          "max_slab_solve_ms": max(x["solve_ms"] for x in sl),
                          "per_rank_total_ms": fac + max(x["solve_ms"] for x in sl),
                          "per_slab": sl}), flush=True)
    if args.validate:
        t0 = time.perf_counter()
        ref, bnd = I.poisson_kernel_parallel(mesh, workers=args.workers)
        val = {"reference_superlu_s": time.perf_counter() - t0, "workers": args.workers}
        interior = np.flatnonzero(np.isin(np.arange(n), bnd, invert=True))
        step = 20000
        relmax, zero_mis, small_abs = 0.0, 0, 0.0
        for a in range(0, len(interior), step):
            rows = interior[a:a + step]
            x = P[torch.from_numpy(rows).to(P.device), :k].cpu().numpy()
            y = ref[rows]
            zero_mis += int(((x == 0) != (y == 0)).sum())
            big = y > 1e-290
            if big.any():
                relmax = max(relmax, float((np.abs(x[big] - y[big]) / y[big]).max()))
            if (~big).any():
                small_abs = max(small_abs, float(np.abs(x[~big] - y[~big]).max()))
        val.update(max_rel_P=relmax, zero_mismatches=zero_mis, max_abs_below_floor=small_abs)
        # downstream: dense KL / TV fields on both P at the default target; the
        # device P is bound to a zero-stride stand-in (no 33 GB host copy)
        import paper_1708_02845_b200 as pf
        from paper_1708_02845_b200 import _device as dev
        from paper_1708_02845_b200.solvers import PoissonKernel
        src, tgt = I.default_endpoints(mesh)
        pk_ref = PoissonKernel(ref, bnd, 0.0, 0.0)
        stand_in = np.broadcast_to(np.zeros(1), (n, k))
        pk_dev = PoissonKernel(stand_in, bnd, residual, rse)
        dev.register(pk_dev.dense, dev.DeviceKernel(None, bnd, n=n, k=k, P_dev=P))
        for g in ("kl", "tv"):
            a = pf.dv_field(pk_dev, pf.builtin_f(g), tgt).values
            b = pf.dv_field(pk_ref, pf.builtin_f(g), tgt).values
            nz = b != 0
            val[f"{g}_max_rel"] = float((np.abs(a[nz] - b[nz]) / np.abs(b[nz])).max())
            val[f"{g}_zero_equal"] = bool(np.array_equal(a == 0, b == 0))
        print(json.dumps({"validate": val}), flush=True)


if __name__ == "__main__":
    main()
