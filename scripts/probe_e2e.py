"""Diagnostic: where the public-API (e2e) time goes for C2-shaped dv_field
calls, and the device timeline (torch.profiler) of dv_field and of the CSR KL
launch pair.  Not a bench number.

python scripts/probe_e2e.py
"""
import math
import sys
import time
from pathlib import Path

ROOT = Path(__file__).resolve().parents[1]
sys.path.insert(0, str(ROOT))

import numpy as np
import torch as t

import bench
import paper_1708_02845_b200 as pf
from paper_1708_02845_b200 import _device as dev, _native as nat
from paper_1708_02845_b200 import divergence as D


def timeline(fn, label, reps=3):
    from torch.profiler import ProfilerActivity, profile
    fn()
    t.cuda.synchronize()
    with profile(activities=[ProfilerActivity.CPU, ProfilerActivity.CUDA]) as prof:
        for _ in range(reps):
            fn()
        t.cuda.synchronize()
    evs = [e for e in prof.events() if e.device_type.name == "CUDA"]
    evs.sort(key=lambda e: e.time_range.start)
    print(f"--- {label}: device timeline (us)")
    prev = None
    for e in evs:
        st, en = e.time_range.start, e.time_range.end
        gap = (st - prev) if prev is not None else 0
        print(f"  {e.name[:60]:60s} dur {en - st:8.1f}  gap {gap:8.1f}")
        prev = en


def main():
    d = t.device("cuda:0")
    rows, k = 102_104, 4_250
    ld = dev.leading_dim(k)
    P = bench.make_synthetic_slab(t, rows, k, ld, 0, d)
    host = np.empty((rows, k))
    for a in range(0, rows, 16384):
        b = min(rows, a + 16384)
        host[a:b] = P[a:b, :k].cpu().numpy()
    pk = pf.PoissonKernel(host, np.array([], np.int64), 0.0, 0.0)
    dk = dev.DeviceKernel(None, np.array([], np.int64), device=d, rows=rows, n=rows, k=k, P_dev=P)
    dev.register(host, dk)
    kl, tv = pf.builtin_f("kl"), pf.builtin_f("tv")
    target = rows // 3 + 1
    for _ in range(5):
        pf.dv_field(pk, kl, target)
    # phase breakdown
    acc = {"field_device": 0.0, "to_host": 0.0, "total": 0.0}
    orig_fd, orig_th = D._field_device, D._to_host

    def fd(*a, **kw):
        t0 = time.perf_counter()
        r = orig_fd(*a, **kw)
        acc["field_device"] += time.perf_counter() - t0
        return r

    def th(*a, **kw):
        t0 = time.perf_counter()
        r = orig_th(*a, **kw)
        acc["to_host"] += time.perf_counter() - t0
        return r

    D._field_device, D._to_host = fd, th
    n = 40
    for rep in range(3):
        for key in acc:
            acc[key] = 0.0
        t0 = time.perf_counter()
        for _ in range(n):
            a = pf.dv_field(pk, kl, target)
            b = pf.dv_field(pk, tv, target)
        acc["total"] = time.perf_counter() - t0
        print(f"rep {rep}: per step {1e3 * acc['total'] / n:.3f} ms; launches "
              f"{1e3 * acc['field_device'] / n:.3f} ms; to_host (copy + sync) "
              f"{1e3 * acc['to_host'] / n:.3f} ms")
    D._field_device, D._to_host = orig_fd, orig_th
    import cProfile
    import pstats
    pr = cProfile.Profile()
    pr.enable()
    for _ in range(100):
        a = pf.dv_field(pk, kl, target)
    pr.disable()
    pstats.Stats(pr).sort_stats("tottime").print_stats(18)
    timeline(lambda: (pf.dv_field(pk, kl, target), pf.dv_field(pk, tv, target)), "dv_field kl+tv", 1)
    del pk, host, dk, P
    t.cuda.empty_cache()
    # CSR KL pair
    P = bench.make_banded_slab(t, rows, k, ld, d)
    dk = dev.DeviceKernel(None, np.array([], np.int64), device=d, rows=rows, n=rows, k=k, P_dev=P)
    dc = dk.csr((1.0 / math.sqrt(rows)) / k, False)
    s = t.cuda.current_stream(d)
    k_pad = dev.round_up(k, 2)
    stage = t.empty(16 * k_pad + dev.round_up(k, 16), dtype=t.uint8, device=d)
    logt = stage.data_ptr() + 8 * k_pad
    out = t.empty(rows + 2, dtype=t.float64, device=d)
    flags = out.data_ptr() + rows * 8
    queue = t.empty(rows, dtype=t.int64, device=d)

    def csr():
        nat.call("pf_target_prep_f64", dk.P[target].data_ptr(), k, 1e-300, stage.data_ptr(), logt,
                 stage.data_ptr() + 16 * k_pad, flags, s.cuda_stream)
        nat.call("pf_csr_kl_f64", dc.indptr.data_ptr(), dc.indices.data_ptr(), dc.data.data_ptr(),
                 dc.log_data.data_ptr(), dc.hs.data_ptr(), rows, k, logt,
                 pf.divergence.KL_GUARD_TAU, 0, 0, rows, out.data_ptr(), 0, flags,
                 queue.data_ptr(), s.cuda_stream)

    timeline(csr, "csr kl", 2)


if __name__ == "__main__":
    main()
