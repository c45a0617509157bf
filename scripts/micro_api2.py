"""Breakdown of dv_field's per-call time (C2 shape)."""
import time
import numpy as np
import torch
import paper_1708_02845_b200 as pf
from paper_1708_02845_b200 import divergence as D, _device as dev, _hostpool as HP

n, k = 102104, 4250
rng = np.random.default_rng(0)
dense = rng.random((n, k)); dense /= dense.sum(1, keepdims=True)
pk = pf.PoissonKernel(dense, np.array([0]), 0.0, 0.0)
kl = pf.builtin_f("kl")
for _ in range(5):
    f = pf.dv_field(pk, kl, 7)
torch.cuda.synchronize()
dk = dev.device_kernel(pk)
s = torch.cuda.current_stream()

def timeit(fn, reps=30):
    torch.cuda.synchronize()
    t0 = time.perf_counter()
    keep = []
    for _ in range(reps):
        keep.append(fn())
        if len(keep) > 3:
            keep.pop(0)
    torch.cuda.synchronize()
    return (time.perf_counter() - t0) / reps * 1e6

buf = dk.scratch(s.cuda_stream, 8 * (n + 2), "out").view(torch.float64)[:n + 2]
print("pool sizes", {k_: len(v) for k_, v in HP._free.items()})
print("dv_field          %.1f us" % timeit(lambda: pf.dv_field(pk, kl, 7)))
print("dv_field_device   %.1f us" % timeit(lambda: pf.dv_field_device(pk, kl, 7)))
print("to_host(scratch)  %.1f us" % timeit(lambda: HP.to_host(torch, buf, s)))
fresh = torch.empty(n + 2, dtype=torch.float64, device="cuda")
print("to_host(fresh)    %.1f us" % timeit(lambda: HP.to_host(torch, fresh, s)))
print("cpu() copy        %.1f us" % timeit(lambda: fresh.cpu()))
print("pool sizes", {k_: len(v) for k_, v in HP._free.items()})
