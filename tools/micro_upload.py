"""Host P -> device upload rate: pageable copy_ (the old DeviceKernel path) vs the
pinned staged upload (_hostpool.upload_rows).  C2 shape by default."""
import sys, time
import numpy as np
import torch as t
sys.path.insert(0, ".")
from paper_1708_02845_b200 import _hostpool, _device as dev

rows, k = (int(sys.argv[1]), int(sys.argv[2])) if len(sys.argv) > 2 else (102104, 4250)
host = np.random.default_rng(0).random((rows, k))
ld = dev.leading_dim(k)
P = t.zeros((rows, ld), dtype=t.float64, device="cuda")
gb = rows * k * 8 / 1e9

def old():
    for a in range(0, rows, 65536):
        b = min(rows, a + 65536)
        src = np.array(host[a:b], dtype=np.float64, order="C")
        P[a:b, :k].copy_(t.from_numpy(src))
    t.cuda.synchronize()

def new():
    _hostpool.upload_rows(t, P, host, 0)
    t.cuda.synchronize()

for name, fn in (("pageable copy_", old), ("pinned staged", new)):
    fn()
    ts = []
    for _ in range(3):
        t0 = time.perf_counter(); fn(); ts.append(time.perf_counter() - t0)
    print(f"{name:16s} {gb:.2f} GB  median {1e3*np.median(ts):8.1f} ms  {gb/np.median(ts):6.1f} GB/s")
P2 = P[:, :k].cpu().numpy()
assert np.array_equal(P2, host), "mismatch"
print("bitwise ok")
