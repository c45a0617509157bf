"""C5 tracer: 10,000 paths over the K7 fields of the C4 mesh with the fields read
(a) in place from the (n, T) output (a field is a column: 8 KB between vertices) and
(b) from a field-major (T, n) copy (vertex neighbours share cache lines).  Timing
only: both traces are the same paths (asserted)."""
import json, sys, time
from pathlib import Path
sys.path.insert(0, str(Path(__file__).resolve().parent.parent))
import numpy as np
import torch as t
import bench as B
import paper_1708_02845_b200 as pf
from paper_1708_02845_b200 import laplacian as L, paths as PP
from workloads.meshes import c5_jobs

omesh, _ = B.build_mesh("c4")
dp, dk, _ = B.device_build(t, L, omesh, t.device("cuda", 0))
targets, src, fo = c5_jobs(omesh)
tm = B.omesh_tri(omesh, pf)
out, _ = pf.divergence._kl_batch_slab(dk, t.from_numpy(targets).cuda(),
                                       dk.P.index_select(0, t.from_numpy(targets).cuda()),
                                       1e-300, "i8")
T = targets.size
outT = out.t().contiguous()
res = {}
for name, arr, lay in (("column (n,T)", out, (1, T)), ("field-major (T,n)", outT, (dk.rows, 1))):
    for _ in range(2):
        PP.trace_arrays(tm, arr, targets, src, fo, layout=lay)
    t.cuda.synchronize()
    ms = []
    for _ in range(3):
        e0, e1 = t.cuda.Event(enable_timing=True), t.cuda.Event(enable_timing=True)
        e0.record()
        buf, counts, over, extra = PP.trace_arrays(tm, arr, targets, src, fo, layout=lay)
        e1.record()
        t.cuda.synchronize()
        ms.append(e0.elapsed_time(e1))
    res[name] = {"ms": sorted(ms), "mean_locations": float(counts.mean())}
print(json.dumps(res, indent=1))
