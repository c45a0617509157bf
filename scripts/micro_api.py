"""Per-call overhead of the public API (tiny P, so kernels are ~5 us)."""
import time
import numpy as np
import torch
import paper_1708_02845_b200 as pf

for n, k in [(4096, 64), (102104, 4250)]:
    rng = np.random.default_rng(0)
    dense = rng.random((n, k)); dense /= dense.sum(1, keepdims=True)
    pk = pf.PoissonKernel(dense, np.array([0]), 0.0, 0.0)
    kl = pf.builtin_f("kl")
    for _ in range(5):
        f = pf.dv_field(pk, kl, 7)
    torch.cuda.synchronize()
    t0 = time.perf_counter()
    keep = []
    for _ in range(50):
        keep.append(pf.dv_field(pk, kl, 7))
        if len(keep) > 3:
            keep.pop(0)
    el = (time.perf_counter() - t0) / 50
    vals, fl = pf.dv_field_device(pk, kl, 7)
    torch.cuda.synchronize()
    t0 = time.perf_counter()
    for _ in range(50):
        vals, fl = pf.dv_field_device(pk, kl, 7)
    torch.cuda.synchronize()
    el2 = (time.perf_counter() - t0) / 50
    print(f"n={n} k={k}: dv_field {el*1e6:.1f} us/call, dv_field_device {el2*1e6:.1f} us/call")
