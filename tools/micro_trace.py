"""Where does a 10K-path tracer call spend its time?"""
import time
import numpy as np
import torch as t
from paper_1708_02845_b200 import mesh as M, paths as PP

mesh = M.grid_mesh(1000, 1000)
dm = M.device_mesh(mesh)
rng = np.random.default_rng(1)
T = 1024
targets = rng.choice(mesh.interior_vertices, T, replace=False)
tv = dm.V.index_select(0, t.from_numpy(targets).cuda())
fields = t.cdist(tv, dm.V)
src = rng.choice(mesh.n, 10_000)
fo = np.arange(10_000) % T
src = np.where(src == targets[fo], (src + 1) % mesh.n, src)
for rep in range(4):
    t.cuda.synchronize()
    t0 = time.perf_counter()
    buf, counts, over, extra = PP.trace_arrays(mesh, fields, targets, src, fo)
    t.cuda.synchronize()
    t1 = time.perf_counter()
    print(f"rep {rep}: trace_arrays {1e3*(t1-t0):.1f} ms, over={over.size}, cap={buf.cap}")
t.cuda.synchronize()
t0 = time.perf_counter()
b2 = PP.PathBuffers(t, 10_000, buf.cap, dm.device)
t.cuda.synchronize()
print(f"PathBuffers alloc {1e3*(time.perf_counter()-t0):.1f} ms")
