"""Sustained-load clocks/power probe: K7 i8 GEMM at C5 shape and the int8 UMMA
ceiling probe, each run back to back for ~2 s with NVML sampled every 5 ms.

python tools/probe_power.py
"""
import ctypes
import statistics
import sys
import threading
import time
from pathlib import Path

ROOT = Path(__file__).resolve().parents[1]
sys.path.insert(0, str(ROOT))

import numpy as np
import pynvml as N
import torch as t

from paper_1708_02845_b200 import _device as dev, _native as nat


class Sampler:
    def __init__(self):
        N.nvmlInit()
        self.h = N.nvmlDeviceGetHandleByIndex(0)
        self.s = []
        self.stop = threading.Event()

    def run(self):
        while not self.stop.is_set():
            self.s.append((N.nvmlDeviceGetClockInfo(self.h, N.NVML_CLOCK_SM),
                           N.nvmlDeviceGetPowerUsage(self.h) / 1000.0,
                           N.nvmlDeviceGetCurrentClocksEventReasons(self.h)))
            self.stop.wait(0.005)

    def __enter__(self):
        self.th = threading.Thread(target=self.run, daemon=True)
        self.th.start()
        return self

    def __exit__(self, *a):
        self.stop.set()
        self.th.join()

    def report(self, tag):
        mhz = [m for m, _, _ in self.s[len(self.s) // 4:]]
        pw = [p for _, p, _ in self.s[len(self.s) // 4:]]
        rs = 0
        for _, _, r in self.s:
            rs |= r
        print(f"{tag}: sm_mhz median {statistics.median(mhz):.0f} min {min(mhz)} "
              f"power median {statistics.median(pw):.0f} W max {max(pw):.0f} W reasons 0x{rs:x}")


def main():
    d = t.device("cuda:0")
    s = t.cuda.current_stream(d)
    rows, k, T = 1_000_386, 4102, 1024
    ldk = dev.round_up(k, 64)
    A = t.randint(0, 256, (7, rows, ldk), dtype=t.uint8, device=d)
    ea = t.zeros(rows, dtype=t.int32, device=d)
    B = t.randint(0, 256, (7, T, ldk), dtype=t.uint8, device=d)
    eb = t.zeros(T, dtype=t.int32, device=d)
    H = t.zeros(rows, dtype=t.float64, device=d)
    tg = t.arange(T, dtype=t.int64, device=d)
    out = t.empty((rows, T), dtype=t.float64, device=d)

    def gemm():
        nat.call("pf_batched_kl_i8", A.data_ptr(), ea.data_ptr(), rows, B.data_ptr(), eb.data_ptr(),
                 T, k, ldk, H.data_ptr(), tg.data_ptr(), 1e-3, 0, out.data_ptr(), T, 64, s.cuda_stream)

    gemm()
    t.cuda.synchronize()
    e0, e1 = t.cuda.Event(enable_timing=True), t.cuda.Event(enable_timing=True)
    with Sampler() as sm:
        e0.record(s)
        for _ in range(16):
            gemm()
        e1.record(s)
        t.cuda.synchronize()
    ms = e0.elapsed_time(e1) / 16
    print(f"i8 gemm C5: {ms:.2f} ms = {34 * 2.0 * rows * k * T / ms / 1e9:.0f} TOPS")
    sm.report("i8 gemm")
    fl = ctypes.c_int64(0)
    sink = t.empty(4, dtype=t.int32, device=d)
    nat.call("pf_probe_umma_i8", 1 << 12, ctypes.byref(fl), sink.data_ptr(), s.cuda_stream)
    t.cuda.synchronize()
    with Sampler() as sm:
        e0.record(s)
        for _ in range(40):
            nat.call("pf_probe_umma_i8", 1 << 16, ctypes.byref(fl), sink.data_ptr(), s.cuda_stream)
        e1.record(s)
        t.cuda.synchronize()
    ms = e0.elapsed_time(e1)
    print(f"umma probe sustained: {40 * fl.value / ms / 1e9:.0f} TOPS over {ms:.0f} ms")
    sm.report("umma probe")


if __name__ == "__main__":
    main()
