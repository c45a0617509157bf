"""Micro-benchmark of field read-back strategies (n FP64 values, D2H)."""
import time
import numpy as np
import torch as t

n = 102_106
d = t.randn(n, dtype=t.float64, device="cuda")
s = t.cuda.current_stream()


def a_pinned_alloc():
    h = t.empty(n, dtype=t.float64, pin_memory=True)
    h.copy_(d, non_blocking=True); s.synchronize(); return h.numpy()


pool = t.empty(n, dtype=t.float64, pin_memory=True)


def b_pool_copy():
    pool.copy_(d, non_blocking=True); s.synchronize(); return pool.numpy().copy()


def c_pageable():
    out = np.empty(n)
    t.from_numpy(out).copy_(d); return out


def d_cpu():
    return d.cpu().numpy()


for fn in (a_pinned_alloc, b_pool_copy, c_pageable, d_cpu):
    for _ in range(5):
        r = fn()
    t.cuda.synchronize()
    t0 = time.perf_counter()
    keep = []
    for _ in range(50):
        keep.append(fn())
        if len(keep) > 2:
            keep.pop(0)
    el = (time.perf_counter() - t0) / 50
    print(f"{fn.__name__:16s} {el*1e6:8.1f} us")
