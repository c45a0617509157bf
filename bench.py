#!/usr/bin/env python
"""Benchmark: vertex-target divergence evaluations/s (KL + TV), B200.

Workload (BASELINE.json configs[1]): dense FP64 Poisson kernel
of the 50:1 corridor shape, 102,104 vertices x 4,250 boundary vertices PER GPU
(weak scaling: each rank owns one row slab of that size; the global mesh is
N x 102,104 rows), KL and TV distance fields to a single target.  One step =
[broadcast of the target row from its owner rank (NCCL, N>1 only)] + KL field
+ TV field over the rank's slab: 2 x rows evaluations per rank.

Synthetic data (softmax rows of N(0,1) with one exact-zero column, FP64): the
reference's real P for this shape takes ~2 min of SuperLU to build and is not
needed for a bandwidth measurement; parity is tested on real P in tests/.
P (3.47 GB/GPU) is far larger than L2 (126 MB), so no L2 flush is needed.

JSON keys beyond the driver contract:
  roofline      dominant kernel (dense KL) achieved GB/s from CUDA events on
                its launch stream, algorithmic bytes rows*(8k+16)+8k per launch
  cpu_baseline  the oracle numpy port (reference algorithm) on the host cores
  e2e           the same metric through the public API dv_field() with the
                field copied back to host memory every call

`--impl reference` times the reference's CPU algorithm (the oracle port,
oracle/divergence.py — the reference is pure Python and cannot travel to the
GPU box) on a bounded sample of the same workload, on all host threads.
"""

from __future__ import annotations

import argparse
import json
import os
import statistics
import subprocess
import sys
import threading
import time
from pathlib import Path

ROOT = Path(__file__).resolve().parent
sys.path.insert(0, str(ROOT))

WORKLOADS = {
    # name: (rows per GPU, k, description)
    "c2": (102_104, 4_250, "C2 corridor 50:1 dense KL+TV, single target"),
    "c2p": (106_030, 1_234, "C2' rectangle 1.5:1 dense KL+TV, single target"),
    "c4": (1_000_386, 4_102, "C4 holes x20 dense KL+TV, single target"),
}
METRIC = "vertex-target divergence evals/sec (KL, TV) at 1/2/4/8 B200; % HBM roofline"


def peaks():
    p = ROOT / "MEASURED_PEAKS.json"
    if p.exists():
        d = json.loads(p.read_text())
        return float(d["hbm_gbs"]), "measured"
    return 6650.0, "fallback"


class ClockSampler:
    """SM clocks and throttle reasons sampled DURING the timed region.

    NVML (nvidia-ml-py) every 5 ms; falls back to polling nvidia-smi when NVML
    is unavailable."""

    REASONS = {  # NVML clocks-event-reason bits
        "hw_slowdown": 0x8, "sw_thermal_slowdown": 0x20, "hw_thermal_slowdown": 0x40,
        "sw_power_cap": 0x4,
    }

    def __init__(self, index: int):
        self.index = index
        self.samples = []  # (sm_mhz, reasons_mask)
        self.max_mhz = None
        self._stop = threading.Event()
        self._t = None
        self._nvml = None

    def _run(self):
        try:
            import pynvml as N
            N.nvmlInit()
            h = N.nvmlDeviceGetHandleByIndex(self.index)
            self.max_mhz = float(N.nvmlDeviceGetMaxClockInfo(h, N.NVML_CLOCK_SM))
            get_reasons = getattr(N, "nvmlDeviceGetCurrentClocksEventReasons", None) or \
                N.nvmlDeviceGetCurrentClocksThrottleReasons
            while not self._stop.is_set():
                self.samples.append((float(N.nvmlDeviceGetClockInfo(h, N.NVML_CLOCK_SM)),
                                     int(get_reasons(h))))
                self._stop.wait(0.005)
            return
        except Exception:
            pass
        q = ("clocks.sm,clocks.max.sm,clocks_event_reasons.hw_slowdown,"
             "clocks_event_reasons.sw_thermal_slowdown,clocks_event_reasons.hw_thermal_slowdown,"
             "clocks_event_reasons.sw_power_cap")
        names = ["hw_slowdown", "sw_thermal_slowdown", "hw_thermal_slowdown", "sw_power_cap"]
        while not self._stop.is_set():
            try:
                out = subprocess.run(["nvidia-smi", f"--id={self.index}", f"--query-gpu={q}",
                                      "--format=csv,noheader,nounits"], capture_output=True,
                                     text=True, timeout=5).stdout.strip().split(",")
                mask = sum(self.REASONS[nm] for nm, v in zip(names, out[2:])
                           if v.strip().lower() == "active")
                self.max_mhz = float(out[1])
                self.samples.append((float(out[0]), mask))
            except Exception:
                pass
            self._stop.wait(0.05)

    def __enter__(self):
        self._t = threading.Thread(target=self._run, daemon=True)
        self._t.start()
        time.sleep(0.02)
        return self

    def __exit__(self, *a):
        self._stop.set()
        self._t.join(timeout=10)

    def summary(self):
        if not self.samples:
            return {"sm_mhz": None, "sm_max_mhz": self.max_mhz, "reasons": ["unsampled"]}
        mhz = [m for m, _ in self.samples]
        reasons = sorted({nm for _, mask in self.samples for nm, bit in self.REASONS.items()
                          if mask & bit})
        return {"sm_mhz": statistics.median(mhz), "sm_max_mhz": self.max_mhz,
                "sm_mhz_min": min(mhz), "reasons": reasons, "samples": len(self.samples),
                "source": "nvml" if len(self.samples) > 3 else "nvidia-smi"}


# --------------------------------------------------------------------------
def dist_env():
    ws = int(os.environ.get("WORLD_SIZE", "1"))
    rank = int(os.environ.get("RANK", "0"))
    local = int(os.environ.get("LOCAL_RANK", "0"))
    return ws, rank, local


def host_info() -> dict:
    """CPU model and the numeric library versions the CPU baseline ran on."""
    import platform
    info = {"cpu_model": platform.processor() or "unknown", "logical_cpus": os.cpu_count()}
    try:
        for line in Path("/proc/cpuinfo").read_text().splitlines():
            if line.startswith("model name"):
                info["cpu_model"] = line.split(":", 1)[1].strip()
                break
    except OSError:
        pass
    import numpy as np
    info["numpy"] = np.__version__
    try:
        import scipy
        info["scipy"] = scipy.__version__
    except ImportError:
        pass
    try:
        cfg = np.show_config(mode="dicts")
        info["blas"] = "{} {}".format(cfg["Build Dependencies"]["blas"].get("name", "?"),
                                      cfg["Build Dependencies"]["blas"].get("version", ""))
    except Exception:
        pass
    return info


def cpu_sample_rows(k: int, rows: int, seed: int):
    import numpy as np
    from oracle.inputs import synthetic_kernel
    P = synthetic_kernel(rows, k, seed)
    P[:, 0] = 0.0
    return P


class CpuReference:
    """Oracle port (reference algorithm: dv_at over row chunks == dv_field,
    SURVEY A.1) on a bounded sample of rows of the workload shape, on all host
    threads.  The sample is sized once so one KL+TV pass takes ~budget_s."""

    def __init__(self, k: int, budget_s: float, threads: int):
        from oracle import divergence as O
        self.O, self.k, self.threads = O, k, threads
        calib = cpu_sample_rows(k, 1024, seed=7)
        t0 = time.perf_counter()
        self._pass(calib)
        dt = max(time.perf_counter() - t0, 1e-3)
        self.rows = int(min(200_000, max(1024, 1024 * budget_s / dt)))
        self.P = cpu_sample_rows(k, self.rows, seed=11)
        self.sample = (f"KL+TV fields over {self.rows} sampled rows x k={k} "
                       f"(target row 0), {threads} threads")

    def _pass(self, P):
        self.O.dv_field_chunked(P, "kl", 0, chunk_rows=256, threads=self.threads)
        self.O.dv_field_chunked(P, "tv", 0, chunk_rows=256, threads=self.threads)

    def step(self):
        t0 = time.perf_counter()
        self._pass(self.P)
        el = time.perf_counter() - t0
        return 2 * self.rows / el, el


# ---- bounded CPU baselines of the side workloads (SURVEY §8d "CPU timing
# beside it"): the oracle restatement of the reference algorithm on all host
# cores (fork workers: the reference's per-pair / per-path loops are Python).
_CPU_STATE: dict = {}


def _cpu_pool_run(fn, items, procs):
    """Run fn over items in `procs` forked workers; returns (results, seconds)."""
    import multiprocessing as mp
    t0 = time.perf_counter()
    if procs <= 1:
        res = [fn(x) for x in items]
    else:
        with mp.get_context("fork").Pool(procs) as pool:
            res = pool.map(fn, items, chunksize=max(1, len(items) // (4 * procs)))
    return res, time.perf_counter() - t0


def _csr_pairs(chunk):
    from oracle import divergence as O
    sv, name, p = _CPU_STATE["csr"]
    return [O.dv_pair_sparse_stats(sv, name, p, int(q))[0] for q in chunk]


def cpu_baseline_csr(rows_full: int, k: int, n_sample: int = 4096, pairs: int = 8192):
    """dv_pair_sparse_stats loop (divergence.py:255-305, restated in
    oracle/divergence.py) over `pairs` sampled query rows of a C3-shaped
    banded P (same generator, `n_sample` rows), all host cores."""
    import math
    import numpy as np
    from oracle import divergence as O
    b = np.arange(k, dtype=np.float64)[None, :]
    q = np.linspace(0, rows_full - 1, n_sample)[:, None]
    c1 = np.floor(q / rows_full * (k / 2))
    x = np.exp(-np.abs(b - c1) / 12.5) + np.exp(-np.abs(b - ((k - 1) - c1)) / 12.5)
    P = x / x.sum(axis=1, keepdims=True)
    sv = O.sparsify(P, np.array([], np.int64), threshold=1.0 / math.sqrt(rows_full))
    procs = os.cpu_count() or 1
    rng = np.random.default_rng(5)
    qs = rng.integers(0, n_sample, pairs)
    out = {}
    for name in ("kl", "tv"):
        _CPU_STATE["csr"] = (sv, name, n_sample // 3)
        chunks = [qs[i:i + 64] for i in range(0, pairs, 64)]
        _, sec = _cpu_pool_run(_csr_pairs, chunks, procs)
        out[name] = pairs / sec
    return {"value": 2.0 / (1.0 / out["kl"] + 1.0 / out["tv"]), "unit": "evals/s",
            "kl_evals_per_s": out["kl"], "tv_evals_per_s": out["tv"], "cores": procs,
            "kind": "port",
            "sample": f"dv_pair_sparse_stats loop (the reference's only sparse field) over "
                      f"{pairs} sampled query rows of a {n_sample} x {k} C3-banded P "
                      f"sparsified at 1/sqrt({rows_full}), {procs} processes"}


def cpu_baseline_batched(k: int, targets: int = 4, rows: int = 8192):
    """T x dv_field (the reference has no batched API): dv_at over row chunks
    for `targets` targets over a `rows`-row synthetic sample, all threads;
    evals/s extrapolates linearly to T = 1024."""
    import numpy as np
    from oracle import divergence as O
    P = cpu_sample_rows(k, rows, seed=13)
    threads = os.cpu_count() or 1
    t0 = time.perf_counter()
    for t in range(targets):
        O.dv_field_chunked(P, "kl", 1 + t, chunk_rows=256, threads=threads)
    sec = time.perf_counter() - t0
    return {"value": rows * targets / sec, "unit": "evals/s", "cores": threads, "kind": "port",
            "sample": f"KL fields (dv_at row chunks == dv_field) for {targets} targets over "
                      f"{rows} sampled rows x k={k}, {threads} threads; the reference "
                      "evaluates T targets as T fields, so evals/s carries to T = 1024"}


def _trace_one(i):
    from oracle import tracer as OT
    V, T, areas, diag, topo, fields, jobs = _CPU_STATE["trace"]
    src, tgt, fi = jobs[i]
    r = OT.triangle_descent(V, T, areas, diag, fields[fi], int(tgt), int(src), topo=topo)
    return len(r["locations"]) if "locations" in r else 0


def cpu_baseline_tracer(mesh, V_dev_fields, targets, src, fo, paths: int = 200):
    """triangle_descent (paths.py:292-307, oracle/tracer.py) for `paths`
    sampled (source, target) pairs of the C5 tracer workload, all cores."""
    import numpy as np
    from oracle import tracer as OT
    pick = np.flatnonzero(fo < 32)[:paths]
    used = np.unique(fo[pick])
    fields = {int(f): V_dev_fields[int(f)].cpu().numpy() for f in used}
    V = np.asarray(mesh.vertices)
    T = np.asarray(mesh.triangles)
    topo = OT.topology(T, len(V))
    _CPU_STATE["trace"] = (V, T, np.asarray(mesh.triangle_areas), float(mesh.bbox_diagonal),
                           topo, fields, [(src[i], targets[fo[i]], int(fo[i])) for i in pick])
    procs = os.cpu_count() or 1
    locs, sec = _cpu_pool_run(_trace_one, list(range(len(pick))), procs)
    return {"value": len(pick) / sec, "unit": "paths/s", "cores": procs, "kind": "port",
            "locations_per_s": float(sum(locs)) / sec,
            "sample": f"{len(pick)} of the 10,000 paths (targets 0-31), oracle/tracer.py "
                      f"restating paths.py:137-307, {procs} processes"}


def run_reference_arm(args):
    ws, rank, local = dist_env()
    if rank != 0:
        return 0
    n_rows, k, desc = WORKLOADS[args.workload]
    threads = os.cpu_count() or 1
    per_step = float(os.environ.get("PF_REF_STEP_S", "2.0"))
    ref = CpuReference(k, per_step, threads)
    for _ in range(args.warmup):
        ref.step()
    vals, els = [], []
    for _ in range(args.steps):
        v, el = ref.step()
        vals.append(v)
        els.append(el)
    sample = ref.sample
    value = statistics.median(vals)
    line = {
        "impl": "reference", "metric": METRIC, "value": value, "unit": "evals/s",
        "n_gpus": args.gpus, "steps": args.steps, "warmup": args.warmup,
        "ms_per_step": 1e3 * statistics.median(els), "higher_is_better": True,
        "scaling": "weak", "vs_baseline": None, "dtype": "f64", "data": "synthetic",
        "config": {"workload": desc, "rows_per_gpu": n_rows, "k": k},
        "cpu_baseline": {"value": value, "unit": "evals/s", "cores": threads, "kind": "port",
                         "host": host_info(),
                         "sample": sample + "; oracle/divergence.py restating divergence.py:137-187"},
        "e2e": {"value": value, "unit": "evals/s", "h2d_bytes_per_step": 0,
                "d2h_bytes_per_step": 0},
    }
    print(json.dumps(line), flush=True)
    return 0


# --------------------------------------------------------------------------
def make_synthetic_slab(t, rows, k, ld, seed, device, chunk=8192):
    """Softmax rows of N(0,1) with column 0 exactly zero, on the GPU (FP64)."""
    P = t.empty((rows, ld), dtype=t.float64, device=device)
    g = t.Generator(device=device)
    g.manual_seed(1234 + seed)
    for a in range(0, rows, chunk):
        b = min(rows, a + chunk)
        x = t.randn((b - a, k), dtype=t.float64, device=device, generator=g)
        x[:, 0] = -float("inf")
        P[a:b, :k] = t.softmax(x, dim=1)
    P[:, k:] = 0.0
    return P


def make_banded_slab(t, rows, k, ld, device, width=12.5, chunk=8192):
    """Corridor-like synthetic P: each row's mass on two exponential bands
    (bottom wall at column c, top wall at k-1-c, c moving along the corridor),
    ~487 entries per row above the 1/sqrt(n) cut — the C3 nnz/row."""
    P = t.empty((rows, ld), dtype=t.float64, device=device)
    b = t.arange(k, dtype=t.float64, device=device)[None, :]
    for a in range(0, rows, chunk):
        e = min(rows, a + chunk)
        q = t.arange(a, e, dtype=t.float64, device=device)[:, None]
        c1 = t.floor(q / rows * (k / 2))
        c2 = (k - 1) - c1
        x = t.exp(-t.abs(b - c1) / width) + t.exp(-t.abs(b - c2) / width)
        P[a:e, :k] = x / x.sum(dim=1, keepdim=True)
    P[:, k:] = 0.0
    return P


class DenseStep:
    """One KL + TV field step over a slab through the C ABI, buffers preallocated.
    With `sharded` (parallel.ShardedField) the target row is NCCL-broadcast."""

    def __init__(self, t, nat, dev, dk, target, tau, sharded=None):
        self.t, self.nat, self.dk = t, nat, dk
        self.target, self.tau, self.sh = target, tau, sharded
        k, rows = dk.k, dk.rows
        self.k_pad, m_pad = dev.round_up(k, 2), dev.round_up(k, 16)
        self.stage = t.empty(16 * self.k_pad + m_pad, dtype=t.uint8, device=dk.device)
        base = self.stage.data_ptr()
        self.tgt, self.logt, self.tmask = base, base + 8 * self.k_pad, base + 16 * self.k_pad
        self.out_kl = t.empty(rows + 2, dtype=t.float64, device=dk.device)
        self.out_tv = t.empty(rows + 2, dtype=t.float64, device=dk.device)
        self.fk = self.out_kl.data_ptr() + rows * 8
        self.ft = self.out_tv.data_ptr() + rows * 8
        self.H = dk.negentropy(1e-300)
        self.stream = t.cuda.current_stream(dk.device)
        self.ev = [(t.cuda.Event(enable_timing=True), t.cuda.Event(enable_timing=True))
                   for _ in range(2)]
        self.kern_ms = [0.0, 0.0]
        self.launches = 0

    def run(self, timed=False):
        dk, nat, s, k = self.dk, self.nat, self.stream.cuda_stream, self.dk.k
        if self.sh is not None:
            rowp = self.sh.target_row(self.target, k).data_ptr()
            self._keep = rowp
        else:
            rowp = dk.P[self.target - dk.row0].data_ptr()
        nat.call("pf_target_prep_f64", rowp, k, 1e-300, self.tgt, self.logt, self.tmask, self.fk, s)
        if timed:
            self.ev[0][0].record(self.stream)
        nat.call("pf_dense_kl_f64", dk.P.data_ptr(), dk.ld, dk.rows, k, self.H.data_ptr(),
                 self.tgt, self.logt, self.tmask, 1e-300, self.tau, dk.row0, self.target,
                 dk.is_interior.data_ptr(), self.out_kl.data_ptr(), self.fk, s)
        if timed:
            self.ev[0][1].record(self.stream)
        nat.call("pf_target_prep_f64", rowp, k, 1e-150, self.tgt, 0, self.tmask, self.ft, s)
        if timed:
            self.ev[1][0].record(self.stream)
        nat.call("pf_dense_tv_f64", dk.P.data_ptr(), dk.ld, dk.rows, k, self.tgt, self.tmask,
                 1e-150, dk.row0, self.target, dk.is_interior.data_ptr(),
                 self.out_tv.data_ptr(), self.ft, s)
        if timed:
            self.ev[1][1].record(self.stream)
            self.stream.synchronize()
            self.kern_ms[0] += self.ev[0][0].elapsed_time(self.ev[0][1])
            self.kern_ms[1] += self.ev[1][0].elapsed_time(self.ev[1][1])
        self.launches += 4   # 2 x target prep, K2, K3


NORTH_STAR_HBM_GBS = 8000.0  # BASELINE.json north_star: "~8 TB/s per GPU"


def _roof(bytes_, ms, peak):
    ach = bytes_ / (ms / 1e3) / 1e9
    return {"bound": "hbm", "achieved": ach, "peak": peak, "unit": "GB/s", "frac": ach / peak,
            "frac_of_8tbs": ach / NORTH_STAR_HBM_GBS,
            "algorithmic_bytes_per_launch": bytes_, "avg_launch_ms": ms}


def extra_f32(t, nat, dev, pf, dk, target, steps, peak):
    """C2 in the FP32 storage mode (query rows from an FP32 copy; 1e-5 tolerance)."""
    rows, k = dk.rows, dk.k
    P32, ld32 = dk.fp32()
    H32 = dk.negentropy32(1e-300)
    s = t.cuda.current_stream(dk.device)
    k_pad, m_pad = dev.round_up(k, 2), dev.round_up(k, 16)
    stage = t.empty(16 * k_pad + m_pad, dtype=t.uint8, device=dk.device)
    tgt, logt, tmask = stage.data_ptr(), stage.data_ptr() + 8 * k_pad, stage.data_ptr() + 16 * k_pad
    out = t.empty(rows + 2, dtype=t.float64, device=dk.device)
    fl = out.data_ptr() + rows * 8
    rowp = dk.P[target - dk.row0].data_ptr()
    tau = pf.divergence.F32_GUARD_TAU
    ev = [t.cuda.Event(enable_timing=True) for _ in range(4)]
    ms = [0.0, 0.0]

    def step(timed):
        nat.call("pf_target_prep_f64", rowp, k, 1e-300, tgt, logt, tmask, fl, s.cuda_stream)
        if timed:
            ev[0].record(s)
        nat.call("pf_dense_kl_f32", P32.data_ptr(), ld32, rows, k, H32.data_ptr(), tgt, logt, tmask,
                 1e-300, tau, dk.row0, target, dk.is_interior.data_ptr(), dk.P.data_ptr(), dk.ld,
                 out.data_ptr(), fl, s.cuda_stream)
        if timed:
            ev[1].record(s)
        nat.call("pf_target_prep_f64", rowp, k, 1e-150, tgt, 0, tmask, fl, s.cuda_stream)
        if timed:
            ev[2].record(s)
        nat.call("pf_dense_tv_f32", P32.data_ptr(), ld32, rows, k, tgt, tmask, 1e-150, tau, dk.row0,
                 target, dk.is_interior.data_ptr(), dk.P.data_ptr(), dk.ld, out.data_ptr(), fl,
                 s.cuda_stream)
        if timed:
            ev[3].record(s)
            s.synchronize()
            ms[0] += ev[0].elapsed_time(ev[1])
            ms[1] += ev[2].elapsed_time(ev[3])

    for _ in range(3):
        step(False)
    n = max(3, steps)
    for _ in range(n):
        step(True)
    kl_ms, tv_ms = ms[0] / n, ms[1] / n
    guarded = int(out[rows:].view(t.int32)[1].item())
    return {"workload": "C2 shape in the FP32 storage mode (P streamed as FP32, FP64 logs / "
                        "accumulation, 1e-5 relative tolerance)",
            "evals_per_s": 2 * rows / ((kl_ms + tv_ms) / 1e3), "tv_guarded_rows_last": guarded,
            "kl": _roof(rows * (4 * k + 16) + 8 * k, kl_ms, peak),
            "tv": _roof(rows * (4 * k + 8) + 8 * k, tv_ms, peak)}


def extra_c4_and_c5(t, nat, dev, pf, device, steps, peak):
    """C4 dense KL+TV (1,000,386 x 4,102 on one GPU) and C5 batched KL (T = 1024)."""
    import numpy as np
    rows, k, _ = WORKLOADS["c4"]
    ld = dev.leading_dim(k)
    P = make_synthetic_slab(t, rows, k, ld, 7, device, chunk=32768)
    dk = dev.DeviceKernel(None, np.array([], np.int64), device=device, rows=rows, n=rows, k=k,
                          P_dev=P)
    target = rows // 3 + 1
    st = DenseStep(t, nat, dev, dk, target, pf.divergence.KL_GUARD_TAU)
    for _ in range(2):
        st.run()
    n = max(2, min(steps, 5))
    for _ in range(n):
        st.run(timed=True)
    kl_ms, tv_ms = st.kern_ms[0] / n, st.kern_ms[1] / n
    c4 = {"workload": "C4 shape 1,000,386 x 4,102 dense FP64 (32.8 GB), synthetic, 1 GPU",
          "evals_per_s": 2 * rows / ((kl_ms + tv_ms) / 1e3),
          "kl": _roof(rows * (8 * k + 16) + 8 * k, kl_ms, peak),
          "tv": _roof(rows * (8 * k + 8) + 8 * k, tv_ms, peak)}
    del st
    # ---- C5: 1024 targets, KL as one contraction + fused epilogue (K7).  Product
    # path: exact-integer emulation of the FP64 GEMM on the int8 tensor pipe
    # (tcgen05, batched_i8.cu); the FP64 DMMA GEMM is timed beside it.
    import ctypes
    T = 1024
    rng = np.random.default_rng(0)
    targets = rng.choice(rows, T, replace=False)
    tg = t.from_numpy(targets.astype(np.int64)).to(device)
    H = dk.negentropy(1e-300)
    ldl = dev.round_up(k, 16)
    Pt = dk.P.index_select(0, tg)
    L = t.empty((T, ldl), dtype=t.float64, device=device)
    Tc = t.empty((T, ldl), dtype=t.float64, device=device)
    out = t.empty((rows, T), dtype=t.float64, device=device)
    cnt = t.zeros(1, dtype=t.int32, device=device)
    s = t.cuda.current_stream(device)
    e0, e1, e2 = (t.cuda.Event(enable_timing=True) for _ in range(3))
    tau = pf.divergence.KL_GUARD_TAU
    e0.record(s)
    A, ea, ldk = dk.slices(1e-300)          # once per P (like H)
    e1.record(s)
    t.cuda.synchronize()
    slice_ms = e0.elapsed_time(e1)
    B = t.empty((7, T, ldk), dtype=t.uint8, device=device)
    eb = t.empty(T, dtype=t.int32, device=device)
    bad = t.zeros(1, dtype=t.int32, device=device)
    gemm_ms = [0.0]

    def batch_i8(timed=False, grade=64):
        nat.call("pf_batch_prep_f64", Pt.data_ptr(), Pt.stride(0), T, k, ldl, 1e-300, 0,
                 L.data_ptr(), Tc.data_ptr(), 0, s.cuda_stream)
        nat.call("pf_slice_targets_u8", L.data_ptr(), ldl, T, k, ldk, B.data_ptr(), eb.data_ptr(),
                 bad.data_ptr(), s.cuda_stream)
        if timed:
            e1.record(s)
        nat.call("pf_batched_kl_i8", A.data_ptr(), ea.data_ptr(), rows, B.data_ptr(),
                 eb.data_ptr(), T, k, ldk, H.data_ptr(), tg.data_ptr(), tau, 0, out.data_ptr(),
                 out.stride(0), grade, s.cuda_stream)
        if timed:
            e2.record(s)
        nat.call("pf_batched_kl_fixup_f64", dk.P.data_ptr(), dk.ld, rows, k, Tc.data_ptr(), ldl,
                 T, 1e-300, out.data_ptr(), out.stride(0), cnt.data_ptr(), s.cuda_stream)

    def batch_f64():
        nat.call("pf_batch_prep_f64", Pt.data_ptr(), Pt.stride(0), T, k, ldl, 1e-300, 0,
                 L.data_ptr(), Tc.data_ptr(), 0, s.cuda_stream)
        nat.call("pf_batched_kl_f64", dk.P.data_ptr(), dk.ld, rows, k, H.data_ptr(), L.data_ptr(),
                 Tc.data_ptr(), ldl, T, tg.data_ptr(), 1e-300, tau, 0,
                 out.data_ptr(), out.stride(0), cnt.data_ptr(), s.cuda_stream)

    def timed(fn, reps):
        fn()
        t.cuda.synchronize()
        st, en = t.cuda.Event(enable_timing=True), t.cuda.Event(enable_timing=True)
        st.record(s)
        for _ in range(reps):
            fn()
        en.record(s)
        t.cuda.synchronize()
        return st.elapsed_time(en) / reps

    reps = 3
    ms = timed(batch_i8, reps)
    batch_i8(True)
    t.cuda.synchronize()
    gemm_only = e1.elapsed_time(e2)
    guarded = int(cnt.item())
    ms_f32grade = timed(lambda: batch_i8(grade=32), reps)
    ms64 = timed(batch_f64, 1)
    flops = 2.0 * rows * k * T
    # measured ceilings of this GPU: sustained DFMA, and the int8 tensor pipe
    fl = ctypes.c_int64(0)
    probe = t.empty(2, dtype=t.float64, device=device)

    def probe_rate(name, iters):
        nat.call(name, iters // 4, ctypes.byref(fl), probe.data_ptr(), s.cuda_stream)
        t.cuda.synchronize()
        e0.record(s)
        nat.call(name, iters, ctypes.byref(fl), probe.data_ptr(), s.cuda_stream)
        e1.record(s)
        t.cuda.synchronize()
        return fl.value / (e0.elapsed_time(e1) / 1e3) / 1e12

    dfma_tf = probe_rate("pf_probe_dfma_f64", 1 << 16)
    i8_tops = probe_rate("pf_probe_umma_i8", 1 << 14)
    int_ops = 34 * flops
    ach = int_ops / (gemm_only / 1e3) / 1e12
    c5 = {"workload": "C5 shape: 1,000,386 x 4,102 P, T = 1024 targets, KL as one contraction "
                      "+ fused epilogue (K7 on the int8 tensor pipe: 34 exact byte-pair GEMMs "
                      "emulating the FP64 GEMM), synthetic, 1 GPU",
          "evals_per_s": rows * T / (ms / 1e3), "ms_per_batch": ms,
          "gemm_ms": gemm_only, "guarded_pairs": guarded,
          "fp64_equivalent_tflops": flops / (ms / 1e3) / 1e12,
          "slice_rows_ms_once_per_P": slice_ms,
          "roofline": {"bound": "tensor", "achieved": ach, "peak": i8_tops, "unit": "TOPS (int8)",
                       "frac": ach / i8_tops,
                       "algorithmic_ops_per_launch": int_ops,
                       "peak_kind": "measured: pf_probe_umma_i8 (M128 N256 K32 u8 tcgen05.mma "
                                    "back to back from shared memory, all SMs)"},
          "fp32_grade": {"note": "same kernel, 15 byte-pair GEMMs (levels 2..6 of the top 5 "
                                 "planes): the north-star FP32 tolerance 1e-5",
                         "ms_per_batch": ms_f32grade,
                         "evals_per_s": rows * T / (ms_f32grade / 1e3)},
          "fp64_dmma_path": {"ms_per_batch": ms64, "evals_per_s": rows * T / (ms64 / 1e3),
                             "achieved_tflops": flops / (ms64 / 1e3) / 1e12,
                             "dfma_peak_tflops": dfma_tf,
                             "frac": flops / (ms64 / 1e3) / 1e12 / dfma_tf}}
    if not NO_CPU:
        try:
            c5["cpu_baseline"] = cpu_baseline_batched(k)
        except Exception as exc:
            c5["cpu_baseline"] = {"error": f"{type(exc).__name__}: {exc}"}
    del A, B
    del out, L, Tc, Pt, dk, P
    t.cuda.empty_cache()
    return c4, c5


def extra_c3(t, nat, dev, pf, device, steps, peak):
    """C3: CSR KL + TV over the corridor-shaped sparse kernel (102,104 x 4,250)."""
    import math
    import numpy as np
    rows, k, _ = WORKLOADS["c2"]
    ld = dev.leading_dim(k)
    P = make_banded_slab(t, rows, k, ld, device)
    dk = dev.DeviceKernel(None, np.array([], np.int64), device=device, rows=rows, n=rows, k=k,
                          P_dev=P)
    cut = (1.0 / math.sqrt(rows)) / k
    t0 = t.cuda.Event(enable_timing=True)
    t1 = t.cuda.Event(enable_timing=True)
    s = t.cuda.current_stream(device)
    t0.record(s)
    dc = dk.csr(cut, False)
    t1.record(s)
    t.cuda.synchronize()
    build_ms = t0.elapsed_time(t1)
    target = rows // 3 + 1
    k_pad = dev.round_up(k, 2)
    stage = t.empty(16 * k_pad + dev.round_up(k, 16), dtype=t.uint8, device=device)
    logt = stage.data_ptr() + 8 * k_pad
    vp = t.empty(k_pad + 4, dtype=t.float64, device=device)
    out = t.empty(rows + 2, dtype=t.float64, device=device)
    flags = out.data_ptr() + rows * 8
    queue = t.empty(rows, dtype=t.int64, device=device)
    kl_entry, kl_idx = dc.field_entry("kl")   # 16-bit columns (k < 65,536)
    tv_entry, tv_idx = dc.field_entry("tv")
    ev = [t.cuda.Event(enable_timing=True) for _ in range(4)]
    ms = [0.0, 0.0]

    def step(timed):
        nat.call("pf_target_prep_f64", dk.P[target].data_ptr(), k, 1e-300, stage.data_ptr(), logt,
                 stage.data_ptr() + 16 * k_pad, flags, s.cuda_stream)
        if timed:
            ev[0].record(s)
        nat.call(kl_entry, dc.indptr.data_ptr(), kl_idx, dc.data.data_ptr(),
                 dc.log_data.data_ptr(), dc.hs.data_ptr(), rows, k, logt,
                 pf.divergence.KL_GUARD_TAU, 0, 0, rows, out.data_ptr(), 0, flags,
                 queue.data_ptr(), s.cuda_stream)
        if timed:
            ev[1].record(s)
        nat.call("pf_csr_target_prep_f64", dc.indptr.data_ptr(), dc.indices.data_ptr(),
                 dc.data.data_ptr(), dc.dropped.data_ptr(), target, k, vp.data_ptr(),
                 vp.data_ptr() + k_pad * 8, s.cuda_stream)
        if timed:
            ev[2].record(s)
        nat.call(tv_entry, dc.indptr.data_ptr(), tv_idx, dc.data.data_ptr(),
                 dc.dropped.data_ptr(), rows, k, vp.data_ptr(), vp.data_ptr() + k_pad * 8, 0, 0,
                 rows, out.data_ptr(), 0, s.cuda_stream)
        if timed:
            ev[3].record(s)
            s.synchronize()
            ms[0] += ev[0].elapsed_time(ev[1])
            ms[1] += ev[2].elapsed_time(ev[3])

    for _ in range(3):
        step(False)
    n = max(3, steps)
    for _ in range(n):
        step(True)
    kl_ms, tv_ms = ms[0] / n, ms[1] / n
    nnz = dc.nnz
    res = {"workload": "C3 shape: 102,104 x 4,250 corridor-banded synthetic P, threshold 1/sqrt(n)",
           "columns": "uint16 device copy (10 B/entry streamed; algorithmic bytes are scipy's "
                      "int32 layout, 12 B/entry)" if dc.indices16 is not None else "int32",
           "nnz": nnz, "nnz_per_row": nnz / rows,
           "sparsity_percent": 100.0 * (1 - nnz / (rows * k)),
           "sparsify_build_ms": build_ms,
           "evals_per_s": 2 * rows / ((kl_ms + tv_ms) / 1e3),
           "kl": _roof(nnz * 12 + rows * 24 + 8 * k, kl_ms, peak),
           "tv": _roof(nnz * 12 + rows * 24 + 16 * k, tv_ms, peak)}
    del dc, dk, P
    t.cuda.empty_cache()
    if not NO_CPU:
        try:
            res["cpu_baseline"] = cpu_baseline_csr(rows, k)
        except Exception as exc:
            res["cpu_baseline"] = {"error": f"{type(exc).__name__}: {exc}"}
    return res


def extra_wire(t, dev, pf, device):
    """Field CSV / JSON wire formats of a C4-sized field (1,000,386 values) on
    the GPU (csrc/wire.cu) vs the reference's Python expressions
    (fileio.py:37-53) timed on a 100,000-value sample of the same values."""
    import numpy as np
    from paper_1708_02845_b200 import fileio as F
    n = 1_000_386
    rng = np.random.default_rng(3)
    vals = rng.random(n) * 10.0 ** rng.uniform(-3, 1, n)   # KL-field-like magnitudes
    dvals = t.from_numpy(vals).to(device)
    fld = pf.ScalarField(vals.copy(), "kl", 0)
    F.field_to_csv(fld)
    F._render(dvals, 0)
    w0 = time.perf_counter()
    F._render(dvals, 0)
    dev_ms = 1e3 * (time.perf_counter() - w0)
    w0 = time.perf_counter()
    csv = F.field_to_csv(fld)
    csv_ms = 1e3 * (time.perf_counter() - w0)
    w0 = time.perf_counter()
    js = F.field_to_json(fld)
    json_ms = 1e3 * (time.perf_counter() - w0)
    m = 100_000
    w0 = time.perf_counter()
    ref = "\n".join(["vertex,value"] + [f"{i},{v:.17g}" for i, v in enumerate(fld.values[:m])])
    ref_csv_ms = 1e3 * (time.perf_counter() - w0) * n / m
    w0 = time.perf_counter()
    json.dumps({"values": [float(v) for v in fld.values[:m]]}, indent=2)
    ref_json_ms = 1e3 * (time.perf_counter() - w0) * n / m
    assert csv.startswith(ref[:1000])
    return {"workload": "field_to_csv / field_to_json of a 1,000,386-value field (C4 rows)",
            "bytes_csv": len(csv), "bytes_json": len(js),
            "hbm_values_to_csv_str_ms": dev_ms, "field_to_csv_ms": csv_ms,
            "field_to_json_ms": json_ms,
            "reference_python_csv_ms_extrapolated": ref_csv_ms,
            "reference_python_json_ms_extrapolated": ref_json_ms,
            "note": "hbm_values_to_csv_str_ms: device-resident values to the CSV body as a "
                    "Python str (kernels, D2H, decode); field_to_*_ms: wall clock from a host "
                    "ScalarField to the "
                    "returned str (H2D, kernels, D2H, decode); reference: the fileio.py "
                    "expressions on 100,000 values x 10.01"}


def extra_poisson(t, nat, dev, device, dfma_peak=None):
    """the Poisson kernel P itself on the device (cotan Laplacian,
    nested-dissection multifrontal Cholesky, multi-RHS solves) at C2 and C4,
    beside the reference algorithm (SuperLU factor + column solves,
    oracle/inputs.poisson_kernel_parallel on all host cores) at C2."""
    import numpy as np
    from oracle import inputs as I
    import paper_1708_02845_b200.laplacian as L
    specs = {"c2": {"gen": "rectangle", "length": 50.0, "width": 1.0, "spacing": 0.024},
             "c4": {"gen": "holes", "spacing": 0.0017, "size": [2.0, 1.25],
                    "holes": [[0.2 + 0.4 * i, 0.16 + 0.31 * j, 0.0034]
                              for i in range(5) for j in range(4)]}}
    if dfma_peak is None:  # measured sustained DFMA rate of this GPU (pf_probe_dfma_f64)
        import ctypes
        fl = ctypes.c_int64(0)
        probe = t.empty(2, dtype=t.float64, device=device)
        s = t.cuda.current_stream(device)
        nat.call("pf_probe_dfma_f64", 1 << 14, ctypes.byref(fl), probe.data_ptr(), s.cuda_stream)
        t.cuda.synchronize()
        p0, p1 = t.cuda.Event(enable_timing=True), t.cuda.Event(enable_timing=True)
        p0.record(s)
        nat.call("pf_probe_dfma_f64", 1 << 16, ctypes.byref(fl), probe.data_ptr(), s.cuda_stream)
        p1.record(s)
        t.cuda.synchronize()
        dfma_peak = fl.value / (p0.elapsed_time(p1) / 1e3) / 1e12
    out = {"dfma_peak_tflops": dfma_peak}
    for name, spec in specs.items():
        t0 = time.perf_counter()
        omesh = I.build(spec)
        # the reference TriMesh holds its boundary as a field computed at construction
        # (mesh.py:79-82); the oracle mesh recomputes it per access, so freeze it here
        from types import SimpleNamespace
        mesh = SimpleNamespace(vertices=omesh.vertices, triangles=omesh.triangles,
                               boundary_vertices=omesh.boundary_vertices)
        mesh_s = time.perf_counter() - t0
        t0 = time.perf_counter()
        dp = L.DevicePoisson(mesh)
        setup_s = time.perf_counter() - t0
        ev = lambda: t.cuda.Event(enable_timing=True)  # noqa: E731
        P, reps = None, []
        for rep in range(3):
            dp._lap, dp._F = None, None
            t.cuda.synchronize()
            e0, e1 = ev(), ev()
            phases = {}
            e0.record()
            dp.laplacian()
            dp.factor()
            P, residual, rse = dp.solve(P, events=phases)
            e1.record()
            t.cuda.synchronize()
            if rep:
                reps.append((e0.elapsed_time(e1), phases["fwd0"].elapsed_time(phases["bwd0"]),
                             phases["bwd0"].elapsed_time(phases["bwd1"]),
                             e0.elapsed_time(phases["fwd0"])))
        tot, fwd, bwd, fac = (float(np.median([r[i] for r in reps])) for i in range(4))
        fl = dp.solve_flops()
        st = dp.plan.stats
        res = {"workload": f"{name}: {dp.n:,} vertices x {dp.k:,} boundary columns "
                           f"({dp.n * dp.k * 8 / 1e9:.2f} GB FP64 P, device-resident)",
               "total_ms": tot, "laplacian_factor_inverse_ms": fac, "forward_ms": fwd,
               "backward_ms": bwd, "residual": residual, "row_sum_error": rse,
               "fronts": st["nodes"], "levels": st["levels"], "max_front": st["max_f"],
               "host_plan_and_upload_s": setup_s, "mesh_build_s": mesh_s,
               "backward_roofline": {
                   "bound": "fp64", "unit": "TFLOP/s",
                   "achieved": fl["backward"] / (bwd * 1e-3) / 1e12,
                   "issued": fl["backward_issued"] / (bwd * 1e-3) / 1e12,
                   "peak": dfma_peak, "frac": (fl["backward"] / (bwd * 1e-3) / 1e12 / dfma_peak
                                               if dfma_peak else None),
                   "algorithmic_flops": fl["backward"],
                   "kernel": "pf::mf_bwd_gemm_kernel (DMMA m8n8k4, gathered rows)"}}
        kk = dp.k
        del P, dp
        t.cuda.empty_cache()
        # end to end through the public API: topology + plan + uploads + device
        # build + the pinned, chunked host copy of P (the reference returns P on
        # the host); the device P stays registered as the mirror of pk.dense
        t.cuda.synchronize()
        w0 = time.perf_counter()
        pk = L.poisson_kernel(mesh)
        res["e2e_poisson_kernel_s"] = time.perf_counter() - w0
        res["e2e_d2h_bytes"] = int(pk.dense.nbytes)
        P = dev.device_kernel(pk).P
        if name == "c2":
            t0 = time.perf_counter()
            ref, _ = I.poisson_kernel_parallel(omesh, workers=os.cpu_count() or 8)
            cpu_s = time.perf_counter() - t0
            idx = np.random.default_rng(0).choice(np.asarray(omesh.interior_vertices), 2000,
                                                  replace=False)
            x = P[t.from_numpy(idx).to(P.device), :kk].cpu().numpy()
            y = ref[idx]
            big = y > 1e-290
            res["cpu_baseline"] = {"value_s": cpu_s, "cores": os.cpu_count(), "kind": "port",
                                   "sample": "SuperLU factor of -Lc_II + solves of all k "
                                             "columns in 64-column chunks, one process per "
                                             "core (oracle/inputs.poisson_kernel_parallel)"}
            res["speedup_vs_cpu"] = cpu_s / (tot * 1e-3)
            res["e2e_speedup_vs_cpu"] = cpu_s / res["e2e_poisson_kernel_s"]
            res["max_rel_vs_superlu_2000_rows"] = float(
                (np.abs(x[big] - y[big]) / y[big]).max())
            del ref
        out[name] = res
        del P, pk
        t.cuda.empty_cache()
    return out


def extra_tracer(t, nat, dev, pf, device):
    """C5 tracer shape: 10,000 paths on a 1,002,001-vertex mesh, 1,024 target fields."""
    import numpy as np
    from paper_1708_02845_b200 import mesh as M
    from paper_1708_02845_b200 import paths as PP
    t0 = time.perf_counter()
    mesh = M.grid_mesh(1000, 1000)
    build_s = time.perf_counter() - t0
    dm = M.device_mesh(mesh)
    rng = np.random.default_rng(1)
    T = 1024
    targets = rng.choice(mesh.interior_vertices, T, replace=False)
    V = dm.V
    tv = V.index_select(0, t.from_numpy(targets).to(device))
    # Euclidean distance fields (the reference tests' smooth descent field), (T, n)
    fields = t.cdist(tv, V)
    npaths = 10_000
    src = rng.choice(mesh.n, npaths)
    fo = np.arange(npaths) % T
    src = np.where(src == targets[fo], (src + 1) % mesh.n, src)
    for _ in range(2):  # warm-up at full size (workspace + topology caches)
        PP.trace_arrays(mesh, fields, targets, src, fo)
    t.cuda.synchronize()
    e0, e1 = t.cuda.Event(enable_timing=True), t.cuda.Event(enable_timing=True)
    s = t.cuda.current_stream(device)
    w0 = time.perf_counter()
    e0.record(s)
    buf, counts, over, extra = PP.trace_arrays(mesh, fields, targets, src, fo)
    e1.record(s)
    t.cuda.synchronize()
    wall = time.perf_counter() - w0
    ms = e0.elapsed_time(e1)
    status = buf.status.cpu().numpy()
    cpu = None
    if not NO_CPU:
        try:
            cpu = cpu_baseline_tracer(mesh, fields, targets, src, fo)
        except Exception as exc:
            cpu = {"error": f"{type(exc).__name__}: {exc}"}
    return {"cpu_baseline": cpu,
            "workload": "10,000 paths (source i -> target i % 1024), 1000x1000 grid mesh "
                        "(1,002,001 vertices, 2,000,000 triangles), Euclidean fields",
            "paths_per_s": npaths / (ms / 1e3), "ms": ms, "wall_ms_incl_launch": 1e3 * wall,
            "locations_per_s": float(counts.sum()) / (ms / 1e3),
            "mean_locations": float(counts.mean()), "max_locations": int(counts.max()),
            "reached": int((status == 0).sum()), "overflow_reruns": int(over.size),
            "mesh_build_s": build_s}


def run_native(args):
    import numpy as np
    import torch as t

    import paper_1708_02845_b200 as pf
    from paper_1708_02845_b200 import _device as dev
    from paper_1708_02845_b200 import _native as nat
    from paper_1708_02845_b200 import parallel as par

    ws, rank, local = dist_env()
    if args.gpus != ws and ws > 1:
        raise SystemExit(f"--gpus {args.gpus} but WORLD_SIZE={ws}")
    t.cuda.set_device(local)
    device = t.device("cuda", local)
    dist = None
    if ws > 1:
        import torch.distributed as dist
        dist.init_process_group("nccl", device_id=device)

    rows, k, desc = WORKLOADS[args.workload]
    n_total = rows * ws
    bounds = [(r * rows, (r + 1) * rows) for r in range(ws)]  # weak scaling: equal slabs
    row0 = rank * rows
    ld = dev.leading_dim(k)
    P_dev = make_synthetic_slab(t, rows, k, ld, rank, device)
    dk = dev.DeviceKernel(None, np.array([], np.int64), device=device, row0=row0, rows=rows,
                          n=n_total, k=k, P_dev=P_dev)
    target = n_total // 3 + 1
    sharded = par.ShardedField(dk, bounds, dist, device=device) if ws > 1 else None
    step = DenseStep(t, nat, dev, dk, target, pf.divergence.KL_GUARD_TAU, sharded)
    stream = step.stream

    def barrier():
        t.cuda.synchronize()
        if dist is not None:
            dist.barrier()
        t.cuda.synchronize()

    def max_over_ranks(x):
        if dist is None:
            return x
        v = t.tensor([x], dtype=t.float64, device=device)
        dist.all_reduce(v, op=dist.ReduceOp.MAX)
        return float(v.item())

    for _ in range(args.warmup):
        step.run()
    barrier()
    for _ in range(args.steps):           # kernel-level timing pass (events on the stream)
        step.run(timed=True)
    kl_ms = step.kern_ms[0] / args.steps
    tv_ms = step.kern_ms[1] / args.steps

    e0, e1 = t.cuda.Event(enable_timing=True), t.cuda.Event(enable_timing=True)
    step.launches = 0
    with ClockSampler(local) as clocks:   # whole-step timing: the reported value
        barrier()
        e0.record(stream)
        for _ in range(args.steps):
            step.run()
        e1.record(stream)
        barrier()
    launches = step.launches
    el_ms = max_over_ranks(e0.elapsed_time(e1))
    value = 2 * rows * ws * args.steps / (el_ms / 1e3)
    flags_kl = step.out_kl[rows:].view(t.int32).cpu().numpy()

    # ------------------------------------------------ e2e via the public API
    e2e = None
    if ws == 1:
        host = np.empty((rows, k))
        for a in range(0, rows, 16384):
            b = min(rows, a + 16384)
            host[a:b] = P_dev[a:b, :k].cpu().numpy()
        pk = pf.PoissonKernel(host, np.array([], np.int64), 0.0, 0.0)
        dev.register(host, dk)
        kl, tv = pf.builtin_f("kl"), pf.builtin_f("tv")
        # warm-up identical to the timed loop (results held across iterations, so the
        # pinned result pool reaches its steady size before timing)
        for _ in range(args.warmup):
            fkl = pf.dv_field(pk, kl, target)
            ftv = pf.dv_field(pk, tv, target)
        barrier()
        per = []
        w0 = time.perf_counter()
        for _ in range(args.steps):
            p0 = time.perf_counter()
            fkl = pf.dv_field(pk, kl, target)
            ftv = pf.dv_field(pk, tv, target)
            per.append(time.perf_counter() - p0)
        barrier()
        e2e_s = time.perf_counter() - w0
        assert np.array_equal(fkl.values, step.out_kl[:rows].cpu().numpy())
        assert np.array_equal(ftv.values, step.out_tv[:rows].cpu().numpy())
        e2e = {"value": 2 * rows * args.steps / e2e_s, "unit": "evals/s",
               "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 2 * (rows + 2) * 8,
               "ms_per_step": 1e3 * e2e_s / args.steps,
               "step_ms_min_median_max": [1e3 * min(per), 1e3 * statistics.median(per),
                                          1e3 * max(per)],
               "note": "wall clock of dv_field(pk, kl, t) + dv_field(pk, tv, t) per step through "
                       "the public API: P resident in HBM (per-PoissonKernel device cache, as "
                       "DomainContext keeps P resident); the target index is a kernel argument; "
                       "each n-vector field + flags is copied D2H into a fresh numpy array and "
                       "returned as a read-only ScalarField"}
        # cold: a PoissonKernel the device has not seen (first query of a DomainContext),
        # so P itself crosses PCIe inside the timed region
        cold_steps = max(1, min(3, args.steps))
        dev.evict(pk)
        t.cuda.empty_cache()
        per = []
        for _ in range(cold_steps):
            barrier()
            p0 = time.perf_counter()
            fkl = pf.dv_field(pk, kl, target)
            ftv = pf.dv_field(pk, tv, target)
            per.append(time.perf_counter() - p0)
            assert np.array_equal(fkl.values, step.out_kl[:rows].cpu().numpy())
            dev.evict(pk)
            t.cuda.empty_cache()
        cold_s = statistics.median(per)
        e2e["cold"] = {"value": 2 * rows / cold_s, "unit": "evals/s",
                       "h2d_bytes_per_step": rows * k * 8 + rows,
                       "d2h_bytes_per_step": 2 * (rows + 2) * 8,
                       "ms_per_step": 1e3 * cold_s, "steps": cold_steps,
                       "h2d_gbs_lower_bound": rows * k * 8 / cold_s / 1e9,
                       "note": "dv_field(kl) + dv_field(tv) on a PoissonKernel with no device "
                               "mirror: pinned staged upload of the host P (_hostpool."
                               "upload_rows), K1 negentropy, K2, K3, D2H of both fields"}
        del host, pk
    else:
        # N > 1: the sharded public API (parallel.ShardedField.field: NCCL broadcast of
        # the target row + slab kernels), each rank's field slab copied back to host
        from paper_1708_02845_b200 import _hostpool
        kl, tv = pf.builtin_f("kl"), pf.builtin_f("tv")

        def e2e_step():
            a = sharded.field(kl, target)
            ha = _hostpool.to_host(t, a, stream)
            b = sharded.field(tv, target)
            hb = _hostpool.to_host(t, b, stream)
            return ha, hb

        for _ in range(args.warmup):
            keep = e2e_step()
        barrier()
        w0 = time.perf_counter()
        for _ in range(args.steps):
            keep = e2e_step()
        barrier()
        e2e_s = max_over_ranks(time.perf_counter() - w0)
        del keep
        e2e = {"value": 2 * rows * ws * args.steps / e2e_s, "unit": "evals/s",
               "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 2 * rows * 8 * ws,
               "ms_per_step": 1e3 * e2e_s / args.steps,
               "note": "wall clock (max over ranks) of ShardedField.field(kl|tv, t) per step: "
                       "NCCL broadcast of the target row from its owner, the slab kernels, "
                       "and each rank's field slab copied to host memory"}

    # ------------------------------------------------ CPU baseline (rank 0, N=1)
    cpu = None
    if rank == 0 and ws == 1 and not args.no_cpu:
        threads = os.cpu_count() or 1
        ref = CpuReference(k, args.cpu_budget, threads)
        v, el = ref.step()
        cpu = {"value": v, "unit": "evals/s", "cores": threads, "kind": "port",
               "sample": ref.sample + f" ({el:.1f} s); oracle/divergence.py restating "
                                      "pathfield divergence.py:137-187 (numpy)",
               "host": host_info()}

    peak, peak_kind = peaks()
    bytes_kl = rows * (8 * k + 16) + 8 * k
    bytes_tv = rows * (8 * k + 8) + 8 * k
    traffic = None
    prof = ROOT / "profiles" / "ncu_summary.json"
    if prof.exists():
        try:
            traffic = json.loads(prof.read_text()).get(args.workload, {}).get("dense_kl_dram_bytes")
        except Exception:
            traffic = None
    roof = _roof(bytes_kl, kl_ms, peak)
    roof.update({"traffic": traffic, "kernel": "pf::dense_kl_kernel (guarded rows re-evaluated in place)",
                 "peak_kind": ("measured (MEASURED_PEAKS.json hbm_gbs, copy)"
                               if peak_kind == "measured" else "fallback 6.65 TB/s")})

    extras = {}
    want = set(args.extras.split(","))
    if ws == 1 and not args.no_extras:
        if "f32" in want:
            try:
                extras["c2_f32"] = extra_f32(t, nat, dev, pf, dk, target, args.steps, peak)
            except Exception as exc:
                extras["c2_f32"] = {"error": f"{type(exc).__name__}: {exc}"}
        del step, dk, P_dev
        t.cuda.empty_cache()
        for name, key, fn in (
                ("c3_csr", "c3", lambda: extra_c3(t, nat, dev, pf, device, args.steps, peak)),
                ("c4_c5", "c4c5", lambda: extra_c4_and_c5(t, nat, dev, pf, device, args.steps,
                                                          peak)),
                ("c5_tracer", "tracer", lambda: extra_tracer(t, nat, dev, pf, device)),
                ("poisson", "poisson", lambda: extra_poisson(
                    t, nat, dev, device,
                    ((extras.get("c5_batched_kl") or {}).get("fp64_dmma_path") or {}).get(
                        "dfma_peak_tflops"))),
                ("wire", "wire", lambda: extra_wire(t, dev, pf, device))):
            if key not in want:
                continue
            try:
                r = fn()
                if name == "c4_c5":
                    extras["c4_dense"], extras["c5_batched_kl"] = r
                else:
                    extras[name] = r
            except Exception as exc:  # an extra must never hide the headline number
                extras[name] = {"error": f"{type(exc).__name__}: {exc}"}
            t.cuda.empty_cache()

    line = {
        "metric": METRIC, "value": value, "unit": "evals/s", "n_gpus": ws,
        "steps": args.steps, "warmup": args.warmup, "ms_per_step": el_ms / args.steps,
        "higher_is_better": True, "scaling": "weak", "vs_baseline": None, "dtype": "f64",
        "data": "synthetic",
        "config": {"workload": desc, "rows_per_gpu": rows, "k": k, "n_total": n_total,
                   "parallelism": f"row-shard x{ws}", "target": target,
                   "l2": "inputs larger than L2 (P slab %.2f GB/GPU vs 126 MB L2)"
                         % (rows * ld * 8 / 1e9)},
        "roofline": roof,
        "roofline_tv": _roof(bytes_tv, tv_ms, peak),
        "kl_guarded_rows": int(flags_kl[1]),
        "cpu_baseline": cpu,
        "e2e": e2e,
        "gpu_launches": launches,
        "clocks": clocks.summary(),
        "extras": extras,
    }
    if rank == 0:
        print(json.dumps(line), flush=True)
    if dist is not None:
        dist.barrier()
        dist.destroy_process_group()
    return 0


NO_CPU = False


def main():
    global NO_CPU
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=50)
    ap.add_argument("--warmup", type=int, default=5)
    ap.add_argument("--impl", default="native", choices=["native", "reference"])
    ap.add_argument("--workload", default="c2", choices=sorted(WORKLOADS))
    ap.add_argument("--cpu-budget", type=float, default=10.0)
    ap.add_argument("--no-cpu", action="store_true")
    ap.add_argument("--no-extras", action="store_true",
                    help="skip the C3/C4/C5/tracer side measurements (N=1 only)")
    ap.add_argument("--extras", default="f32,c3,c4c5,tracer,wire,poisson",
                    help="comma list of side measurements to run "
                         "(f32, c3, c4c5, tracer, wire, poisson)")
    args = ap.parse_args()
    NO_CPU = bool(args.no_cpu)
    if args.warmup < 3:
        args.warmup = 3
    if args.impl == "reference":
        return run_reference_arm(args)
    return run_native(args)


if __name__ == "__main__":
    sys.exit(main())
