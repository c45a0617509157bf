"""D2H of a device P into a fresh host array: np.empty (4 KB pages, first-touch
faults) vs an anonymous mmap advised MADV_HUGEPAGE (2 MB pages)."""
import mmap, sys, time
import numpy as np
import torch as t
sys.path.insert(0, ".")
from paper_1708_02845_b200 import laplacian as L, _device as dev

print(open("/sys/kernel/mm/transparent_hugepage/enabled").read().strip(),
      open("/sys/kernel/mm/transparent_hugepage/defrag").read().strip())
rows, k = (int(sys.argv[1]), int(sys.argv[2])) if len(sys.argv) > 2 else (250_000, 4102)
ld = dev.leading_dim(k)
P = t.rand((rows, ld), dtype=t.float64, device="cuda")
gb = rows * k * 8 / 1e9

def huge_empty(shape):
    nbytes = int(np.prod(shape)) * 8
    mm = mmap.mmap(-1, nbytes, flags=mmap.MAP_PRIVATE | mmap.MAP_ANONYMOUS)
    mm.madvise(mmap.MADV_HUGEPAGE)
    return np.frombuffer(mm, dtype=np.float64).reshape(shape)

orig = np.empty
for name in ("np.empty", "hugepage mmap", "np.empty", "hugepage mmap"):
    alloc = orig if name == "np.empty" else huge_empty
    L.np.empty = lambda shape, *a, **kw: alloc(shape) if (isinstance(shape, tuple) and len(shape) == 2) else orig(shape, *a, **kw)
    t.cuda.synchronize()
    t0 = time.perf_counter()
    out = L.dense_to_host(P, rows, k)
    dt = time.perf_counter() - t0
    L.np.empty = orig
    assert np.array_equal(out[::9973], P[::9973, :k].cpu().numpy())
    print(f"{name:14s} {gb:.2f} GB  {1e3*dt:8.1f} ms  {gb/dt:6.1f} GB/s")
    del out
