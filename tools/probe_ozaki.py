"""GPU probe for K7 on the int8 tensor pipe (batched_i8.cu): accuracy against
the FP64 DMMA path and a torch FP64 GEMM, then timing at the C5 shape.

python tools/probe_ozaki.py [--big]
"""
import sys
import time
from pathlib import Path

ROOT = Path(__file__).resolve().parents[1]
sys.path.insert(0, str(ROOT))

import numpy as np
import torch as t

from paper_1708_02845_b200 import _device as dev, _native as nat

GUARD = 0x7ff8dead0000ba7c


def synth(rows, k, ld, seed, dev_):
    g = t.Generator(device=dev_)
    g.manual_seed(seed)
    P = t.zeros((rows, ld), dtype=t.float64, device=dev_)
    for a in range(0, rows, 32768):
        b = min(rows, a + 32768)
        x = t.randn((b - a, k), dtype=t.float64, device=dev_, generator=g) * 3.0
        x[:, 0] = -float("inf")
        P[a:b, :k] = t.softmax(x, dim=1)
    return P


def run(rows, k, T, seed=0, timing=False):
    d = t.device("cuda:0")
    s = t.cuda.current_stream(d).cuda_stream
    ld = dev.round_up(k, 16)
    ldl = ld
    ldk = dev.round_up(k, 64)
    clamp, tau = 1e-300, 1e-3
    P = synth(rows, k, ld, seed, d)
    H = t.empty(rows, dtype=t.float64, device=d)
    mn = t.empty(1, dtype=t.float64, device=d)
    nat.call("pf_row_negentropy_f64", P.data_ptr(), ld, rows, k, clamp, H.data_ptr(), mn.data_ptr(), s)
    rng = np.random.default_rng(seed)
    targets = np.sort(rng.choice(rows, T, replace=False)).astype(np.int64)
    tg = t.from_numpy(targets).to(d)
    Pt = P.index_select(0, tg).contiguous()
    L = t.empty((T, ldl), dtype=t.float64, device=d)
    Tc = t.empty((T, ldl), dtype=t.float64, device=d)
    nat.call("pf_batch_prep_f64", Pt.data_ptr(), ld, T, k, ldl, clamp, 0, L.data_ptr(),
             Tc.data_ptr(), 0, s)
    # FP64 DMMA path (product K7)
    o64 = t.empty((rows, T), dtype=t.float64, device=d)
    cnt = t.zeros(2, dtype=t.int32, device=d)
    nat.call("pf_batched_kl_f64", P.data_ptr(), ld, rows, k, H.data_ptr(), L.data_ptr(),
             Tc.data_ptr(), ldl, T, tg.data_ptr(), clamp, tau, 0, o64.data_ptr(), T,
             cnt.data_ptr(), s)
    # int8 path
    A = t.empty((7, rows, ldk), dtype=t.uint8, device=d)
    ea = t.empty(rows, dtype=t.int32, device=d)
    B = t.empty((7, T, ldk), dtype=t.uint8, device=d)
    eb = t.empty(T, dtype=t.int32, device=d)
    bad = t.zeros(1, dtype=t.int32, device=d)
    t.cuda.synchronize()
    t0 = time.perf_counter()
    nat.call("pf_slice_rows_u8", P.data_ptr(), ld, rows, k, clamp, ldk, A.data_ptr(), ea.data_ptr(), s)
    t.cuda.synchronize()
    slice_s = time.perf_counter() - t0
    nat.call("pf_slice_targets_u8", L.data_ptr(), ldl, T, k, ldk, B.data_ptr(), eb.data_ptr(),
             bad.data_ptr(), s)
    o8 = t.empty((rows, T), dtype=t.float64, device=d)
    nat.call("pf_batched_kl_i8", A.data_ptr(), ea.data_ptr(), rows, B.data_ptr(), eb.data_ptr(), T,
             k, ldk, H.data_ptr(), tg.data_ptr(), tau, 0, o8.data_ptr(), T, 64, s)
    raw = o8.clone()
    nat.call("pf_batched_kl_fixup_f64", P.data_ptr(), ld, rows, k, Tc.data_ptr(), ldl, T, clamp,
             o8.data_ptr(), T, cnt.data_ptr() + 4, s)
    t.cuda.synchronize()
    nguard = int((raw.view(t.int64) == GUARD).sum())
    # torch FP64 reference for S on a row sample
    idx = t.arange(0, rows, max(1, rows // 4096), device=d)
    Sref = (t.clamp(P[idx, :k], min=clamp) @ (-L[:, :k]).T)
    KLref = H[idx, None] + Sref
    rel8 = ((o8[idx] - KLref).abs() / KLref.abs().clamp(min=1e-300))
    rel64 = ((o64[idx] - KLref).abs() / KLref.abs().clamp(min=1e-300))
    rel_8_64 = ((o8 - o64).abs() / o64.abs().clamp(min=1e-300))
    tmask = t.zeros_like(rel_8_64, dtype=t.bool)
    tmask[tg, t.arange(T, device=d)] = True
    rel_8_64[tmask] = 0
    print(f"rows={rows} k={k} T={T}: bad={int(bad.item())} guarded i8={nguard} "
          f"(fixup count {cnt.tolist()}) slice_rows {slice_s*1e3:.1f} ms")
    print(f"  max rel err vs torch FP64 GEMM (sampled rows): i8 {rel8.max().item():.3e}  "
          f"dmma {rel64.max().item():.3e}; i8 vs dmma (all) {rel_8_64.max().item():.3e}; "
          f"zeros at targets: {bool((o8[tg, t.arange(T, device=d)] == 0).all())}")
    if timing:
        ev = [t.cuda.Event(enable_timing=True) for _ in range(4)]
        st = t.cuda.current_stream(d)
        for _ in range(2):
            nat.call("pf_batched_kl_i8", A.data_ptr(), ea.data_ptr(), rows, B.data_ptr(), eb.data_ptr(),
                     T, k, ldk, H.data_ptr(), tg.data_ptr(), tau, 0, o8.data_ptr(), T, 64, s)
        ev[0].record(st)
        reps = 3
        for _ in range(reps):
            nat.call("pf_batched_kl_i8", A.data_ptr(), ea.data_ptr(), rows, B.data_ptr(), eb.data_ptr(),
                     T, k, ldk, H.data_ptr(), tg.data_ptr(), tau, 0, o8.data_ptr(), T, 64, s)
        ev[1].record(st)
        for _ in range(reps):
            nat.call("pf_batched_kl_f64", P.data_ptr(), ld, rows, k, H.data_ptr(), L.data_ptr(),
                     Tc.data_ptr(), ldl, T, tg.data_ptr(), clamp, tau, 0, o64.data_ptr(), T,
                     cnt.data_ptr(), s)
        ev[2].record(st)
        t.cuda.synchronize()
        ms8 = ev[0].elapsed_time(ev[1]) / reps
        ms64 = ev[1].elapsed_time(ev[2]) / reps
        fl = 2.0 * rows * k * T
        print(f"  i8 GEMM+epilogue {ms8:.2f} ms = {fl/ms8/1e9:.1f} FP64-equivalent TFLOP/s "
              f"({34*fl/ms8/1e9:.0f} int8 TOPS); DMMA path {ms64:.2f} ms = {fl/ms64/1e9:.1f} TFLOP/s")


if __name__ == "__main__":
    run(1000, 300, 70, seed=1)
    run(4000, 4102, 256, seed=2)
    run(30000, 4250, 200, seed=3, timing=True)
    if "--big" in sys.argv:
        run(1_000_386, 4102, 1024, seed=4, timing=True)
