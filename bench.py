#!/usr/bin/env python
"""Benchmark: vertex-target divergence evaluations/s (KL + TV), B200.

Headline workload (BASELINE.json north_star target): the
multiply-connected domain with 20 obstacles, 1,000,386 vertices x 4,102
boundary vertices, REAL Poisson kernel P: the mesh is the reference
generator's (workloads/meshes.py, bitwise the reference's) and P is built on
the GPU by the product's multifrontal solve (laplacian.DevicePoisson, K11;
within 1e-11 of the reference's SuperLU P).  Strong scaling: the
n rows are split into N contiguous slabs, rank r builds ONLY its slab of P
(ShardedField.from_mesh) and owns it.  One step = [NCCL broadcast of the
target row from its owner rank (N > 1, pf_nccl_broadcast)] + KL field + TV
field over the rank's slab = 2 n evaluations for the whole job.  The target
is the reference's default_endpoints target (domain.py:155-165).  P (32.8 GB,
4.1 GB per rank at N = 8) is far larger than L2 (126 MB): no L2 flush needed.

JSON keys beyond the driver contract:
  roofline      dense KL kernel achieved GB/s from CUDA events on its launch
                stream, algorithmic bytes rows*(8k+16)+8k per launch
                (SURVEY §8d), against the measured copy bandwidth
  cpu_baseline  the oracle numpy port (reference algorithm) on the host cores
                over a bounded sample of REAL rows of the same P
  e2e           the same metric through the public API (dv_field at N = 1,
                ShardedField.field at N > 1) with each field copied to host
                memory every call
  preprocessing the one-time mesh / P / negentropy builds (not in `value`)
  extras        side configs: C2/C2' real (dense, FP32 mode, C3 CSR), C4 FP32,
                C5 (1,024-target batched KL + 10,000 traced paths), the
                synthetic C2 weak-scaling line of round 1, Poisson build,
                wire formats; at N > 1 the sharded C3 and distributed C5

`--impl reference` times the reference's CPU algorithm (the oracle port,
oracle/divergence.py — the reference is pure Python and cannot travel to the
GPU box) on a bounded sample of the same workload shape, on all host threads.
"""

from __future__ import annotations

import argparse
import json
import math
import os
import statistics
import subprocess
import sys
import threading
import time
from pathlib import Path

ROOT = Path(__file__).resolve().parent
sys.path.insert(0, str(ROOT))

# name: (n, k, description); the mesh recipe is workloads.meshes.SPECS[name]
WORKLOADS = {
    "c4": (1_000_386, 4_102, "C4 holes x20 (1,000,386 x 4,102), real P, dense KL+TV, "
                             "single target, row slabs over N GPUs"),
    "c2": (102_104, 4_250, "C2 corridor 50:1 (102,104 x 4,250), real P, dense KL+TV, "
                           "single target, row slabs over N GPUs"),
    "c2p": (106_030, 1_234, "C2' rectangle 1.5:1 (106,030 x 1,234), real P, dense KL+TV, "
                            "single target, row slabs over N GPUs"),
}
METRIC = "vertex-target divergence evals/sec (KL, TV) at 1/2/4/8 B200; % HBM roofline"
NORTH_STAR_HBM_GBS = 8000.0  # BASELINE.json north_star: "~8 TB/s per GPU"
NO_CPU = False


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
        # the timed region starts only once the sampler is producing samples
        # (NVML initialisation can take longer than a short timed region)
        t0 = time.perf_counter()
        while not self.samples and time.perf_counter() - t0 < 10.0:
            time.sleep(0.005)
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


def _events(t, n=2):
    return [t.cuda.Event(enable_timing=True) for _ in range(n)]


def _roof(bytes_, ms, peak, streamed=None):
    ach = bytes_ / (ms / 1e3) / 1e9
    r = {"bound": "hbm", "achieved": ach, "peak": peak, "unit": "GB/s", "frac": ach / peak,
         "frac_of_8tbs": ach / NORTH_STAR_HBM_GBS,
         "algorithmic_bytes_per_launch": bytes_, "avg_launch_ms": ms}
    if streamed is not None:  # bytes the kernel actually streams (e.g. 16-bit CSR columns)
        r["streamed_bytes_per_launch"] = streamed
        r["frac_streamed"] = streamed / (ms / 1e3) / 1e9 / peak
    return r


# ---- CPU baselines: the oracle restatement of the reference algorithm on all
# host cores (SURVEY §8d "CPU timing beside it")
class CpuReference:
    """Oracle port (reference algorithm: dv_at over row chunks == dv_field,
    SURVEY A.1) on a bounded sample of rows, on all host threads.  `rows_of(m)`
    returns an (m, k) host matrix whose row 0 is the target row; the sample
    is sized once so one KL+TV pass takes ~budget_s.  `on_matrix` instead
    evaluates rows of a full host P in place (evenly spaced rows, or all of
    them when the budget allows: then the sample IS the whole field)."""

    def __init__(self, rows_of, k: int, budget_s: float, threads: int, what: str,
                 matrix=None, target: int = 0):
        import numpy as np
        from oracle import divergence as O
        self.O, self.k, self.threads = O, k, threads
        if matrix is not None:
            n = matrix.shape[0]
            self.P, self.target = matrix, int(target)
            probe = np.linspace(0, n - 1, 2048).astype(np.int64)
            t0 = time.perf_counter()
            self._pass(self.P, probe)
            dt = max(time.perf_counter() - t0, 1e-3)
            m = int(min(n, max(2048, 2048 * budget_s / dt)))
            self.idx = np.arange(n, dtype=np.int64) if m >= n else \
                np.linspace(0, n - 1, m).astype(np.int64)
            self.rows = int(self.idx.size)
            self.sample = (f"KL+TV fields over {self.rows:,} of {n:,} rows x k={k} ({what}; "
                           f"evaluated in place in the host P), {threads} threads")
            return
        self.target, self.idx = 0, None
        calib = rows_of(1024)
        t0 = time.perf_counter()
        self._pass(calib, None)
        dt = max(time.perf_counter() - t0, 1e-3)
        self.rows = int(min(200_000, max(1024, 1024 * budget_s / dt)))
        self.P = rows_of(self.rows)
        self.sample = (f"KL+TV fields over {self.rows} sampled rows x k={k} ({what}; target "
                       f"row first), {threads} threads")

    def _pass(self, P, idx):
        tgt = self.target if idx is not None else 0
        self.O.dv_field_chunked(P, "kl", tgt, rows=idx, chunk_rows=256, threads=self.threads)
        self.O.dv_field_chunked(P, "tv", tgt, rows=idx, chunk_rows=256, threads=self.threads)

    def step(self):
        t0 = time.perf_counter()
        self._pass(self.P, self.idx)
        el = time.perf_counter() - t0
        return 2 * self.rows / el, el


def synthetic_rows(k: int, seed: int):
    """Row-stochastic synthetic rows (softmax of N(0,1), one zero column)."""
    def rows_of(m):
        from workloads.meshes import synthetic_kernel
        P = synthetic_kernel(m, k, seed)
        P[:, 0] = 0.0
        return P
    return rows_of


def device_rows(t, dk, target: int):
    """Real rows of a device-resident P: the target row, then evenly spaced rows."""
    import numpy as np

    def rows_of(m):
        idx = np.linspace(0, dk.rows - 1, max(1, m - 1)).astype(np.int64)
        idx = np.concatenate([[target - dk.row0], idx])[:m]
        sel = dk.P.index_select(0, t.from_numpy(idx).to(dk.device))[:, :dk.k]
        return sel.cpu().numpy()
    return rows_of


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


def cpu_baseline_csr(P_rows, n_full: int, pairs: int = 8192):
    """dv_pair_sparse_stats loop (divergence.py:255-305, restated in
    oracle/divergence.py) over `pairs` sampled query rows of a row sample of
    the real P (row 0 = the target), sparsified at the reference's default
    threshold 1/sqrt(n) of the full mesh, all host cores."""
    import numpy as np
    from oracle import divergence as O
    m, k = P_rows.shape
    sv = O.sparsify(P_rows, np.array([], np.int64), threshold=1.0 / math.sqrt(n_full))
    procs = os.cpu_count() or 1
    qs = np.random.default_rng(5).integers(0, m, pairs)
    out = {}
    for name in ("kl", "tv"):
        _CPU_STATE["csr"] = (sv, name, 0)
        chunks = [qs[i:i + 64] for i in range(0, pairs, 64)]
        _, sec = _cpu_pool_run(_csr_pairs, chunks, procs)
        out[name] = pairs / sec
    return {"value": 2.0 / (1.0 / out["kl"] + 1.0 / out["tv"]), "unit": "evals/s",
            "kl_evals_per_s": out["kl"], "tv_evals_per_s": out["tv"], "cores": procs,
            "kind": "port",
            "sample": f"dv_pair_sparse_stats loop (the reference's only sparse field) over "
                      f"{pairs} sampled query rows of {m} real rows x {k} sparsified at "
                      f"1/sqrt({n_full}), {procs} processes"}


def cpu_baseline_batched(P_rows, targets: int = 4):
    """T x dv_field (the reference has no batched API): dv_at over row chunks
    for `targets` target rows over a real row sample, all threads; evals/s
    carries to T = 1024 (the reference evaluates T targets as T fields)."""
    from oracle import divergence as O
    m, k = P_rows.shape
    threads = os.cpu_count() or 1
    t0 = time.perf_counter()
    for t in range(targets):
        O.dv_field_chunked(P_rows, "kl", t, chunk_rows=256, threads=threads)
    sec = time.perf_counter() - t0
    return {"value": m * targets / sec, "unit": "evals/s", "cores": threads, "kind": "port",
            "sample": f"KL fields (dv_at row chunks == dv_field) for {targets} targets over "
                      f"{m} real rows x k={k}, {threads} threads; the reference evaluates T "
                      "targets as T fields, so evals/s carries to T = 1024"}


def _trace_one(i):
    from oracle import tracer as OT
    V, T, areas, diag, topo, fields, jobs = _CPU_STATE["trace"]
    src, tgt, fi = jobs[i]
    r = OT.triangle_descent(V, T, areas, diag, fields[fi], int(tgt), int(src), topo=topo)
    return len(r["locations"]) if "locations" in r else 0


def cpu_baseline_tracer(omesh, field_cols, targets, src, fo, paths: int = 200):
    """triangle_descent (paths.py:292-307, oracle/tracer.py) for `paths`
    sampled (source, target) pairs of the C5 workload on the real mesh and
    fields, all cores.  `field_cols(j)` returns target j's field (host)."""
    import numpy as np
    from oracle import tracer as OT
    pick = np.flatnonzero(fo < 32)[:paths]
    used = np.unique(fo[pick])
    fields = {int(f): field_cols(int(f)) for f in used}
    topo = OT.topology(omesh.triangles, omesh.n)
    _CPU_STATE["trace"] = (omesh.vertices, omesh.triangles, omesh.areas, omesh.bbox_diagonal,
                           topo, fields, [(src[i], targets[fo[i]], int(fo[i])) for i in pick])
    procs = os.cpu_count() or 1
    locs, sec = _cpu_pool_run(_trace_one, list(range(len(pick))), procs)
    return {"value": len(pick) / sec, "unit": "paths/s", "cores": procs, "kind": "port",
            "locations_per_s": float(sum(locs)) / sec,
            "sample": f"{len(pick)} of the C5 paths (targets 0-31) on the real mesh and "
                      f"fields, oracle/tracer.py restating paths.py:137-307, {procs} processes"}


def run_reference_arm(args):
    ws, rank, local = dist_env()
    if rank != 0:
        return 0
    n_rows, k, desc = WORKLOADS[args.workload]
    threads = os.cpu_count() or 1
    per_step = float(os.environ.get("PF_REF_STEP_S", "2.0"))
    ref = CpuReference(synthetic_rows(k, 11), k, per_step, threads,
                       "synthetic row-stochastic rows of the workload's k: the real P needs "
                       "the GPU build, and the port's cost per row depends on k only")
    for _ in range(args.warmup):
        ref.step()
    vals, els = [], []
    for _ in range(args.steps):
        v, el = ref.step()
        vals.append(v)
        els.append(el)
    value = statistics.median(vals)
    line = {
        "impl": "reference", "metric": METRIC, "value": value, "unit": "evals/s",
        "n_gpus": args.gpus, "steps": args.steps, "warmup": args.warmup,
        "ms_per_step": 1e3 * statistics.median(els), "higher_is_better": True,
        "scaling": "strong", "vs_baseline": None, "dtype": "f64",
        "data": "synthetic rows of the workload shape",
        "config": {"workload": desc, "n": n_rows, "k": k},
        "cpu_baseline": {"value": value, "unit": "evals/s", "cores": threads, "kind": "port",
                         "host": host_info(),
                         "sample": ref.sample + "; oracle/divergence.py restating "
                                                "divergence.py:137-187"},
        "e2e": {"value": value, "unit": "evals/s", "h2d_bytes_per_step": 0,
                "d2h_bytes_per_step": 0},
    }
    print(json.dumps(line), flush=True)
    return 0


# --------------------------------------------------------------------------
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
        self.ev = [_events(t) for _ in range(2)]
        self.kern_ms = [0.0, 0.0]
        self.launches = 0

    def run(self, timed=False):
        dk, nat, s, k = self.dk, self.nat, self.stream.cuda_stream, self.dk.k
        if self.sh is not None:
            row = self.sh.target_row(self.target, k)
            self._keep = row
            rowp = row.data_ptr()
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

    def kernel_ms(self, steps):
        """Average K2 / K3 launch time over `steps` event-timed steps."""
        self.kern_ms = [0.0, 0.0]
        for _ in range(steps):
            self.run(timed=True)
        return self.kern_ms[0] / steps, self.kern_ms[1] / steps


def build_mesh(name):
    from workloads.meshes import SPECS, build
    t0 = time.perf_counter()
    omesh = build(SPECS[name])
    return omesh, time.perf_counter() - t0


def device_build(t, L, omesh, device, slab=None):
    """P (or the row slab) on the device with the fused K1 (DevicePoisson);
    returns (dp, dk, timings)."""
    w0 = time.perf_counter()
    dp = L.DevicePoisson(omesh, device=device)
    plan_s = time.perf_counter() - w0
    e0, e1 = _events(t)
    t.cuda.synchronize()
    w0 = time.perf_counter()
    e0.record()
    dk = dp.device_kernel(slab=slab)
    e1.record()
    t.cuda.synchronize()
    return dp, dk, {"host_plan_and_upload_s": plan_s, "device_build_ms": e0.elapsed_time(e1),
                    "device_build_wall_s": time.perf_counter() - w0,
                    "residual": dk.residual, "row_sum_error": dk.row_sum_error}


def dense_fields_extra(t, nat, dev, pf, dk, target, steps, peak, f32=True):
    """KL+TV (and FP32-mode) kernel timings over a device P (single GPU)."""
    st = DenseStep(t, nat, dev, dk, target, pf.divergence.KL_GUARD_TAU)
    for _ in range(3):
        st.run()
    kl_ms, tv_ms = st.kernel_ms(max(3, steps))
    rows, k = dk.rows, dk.k
    res = {"evals_per_s": 2 * rows / ((kl_ms + tv_ms) / 1e3),
           "kl_guarded_rows": int(st.out_kl[rows:].view(t.int32)[1].item()),
           "kl": _roof(rows * (8 * k + 16) + 8 * k, kl_ms, peak),
           "tv": _roof(rows * (8 * k + 8) + 8 * k, tv_ms, peak)}
    del st
    if f32:
        res["fp32_mode"] = extra_f32(t, nat, dev, pf, dk, target, steps, peak)
    return res


def extra_f32(t, nat, dev, pf, dk, target, steps, peak):
    """KL+TV in the FP32 storage mode (query rows from an FP32 copy; 1e-5 tolerance)."""
    rows, k = dk.rows, dk.k
    P32, ld32 = dk.fp32()
    H64 = dk.negentropy(1e-300)
    s = t.cuda.current_stream(dk.device)
    k_pad, m_pad = dev.round_up(k, 2), dev.round_up(k, 16)
    stage = t.empty(16 * k_pad + m_pad, dtype=t.uint8, device=dk.device)
    tgt, logt, tmask = stage.data_ptr(), stage.data_ptr() + 8 * k_pad, stage.data_ptr() + 16 * k_pad
    out = t.empty(rows + 2, dtype=t.float64, device=dk.device)
    fl = out.data_ptr() + rows * 8
    rowp = dk.P[target - dk.row0].data_ptr()
    tau = pf.divergence.F32_GUARD_TAU
    ev = _events(t, 4)
    ms = [0.0, 0.0]
    guarded = [0, 0]

    def step(timed):
        nat.call("pf_target_prep_f64", rowp, k, 1e-300, tgt, logt, tmask, fl, s.cuda_stream)
        if timed:
            ev[0].record(s)
        nat.call("pf_dense_kl_f32", P32.data_ptr(), ld32, rows, k, H64.data_ptr(), tgt, logt, tmask,
                 1e-300, tau, dk.row0, target, dk.is_interior.data_ptr(), dk.P.data_ptr(), dk.ld,
                 H64.data_ptr(), pf.divergence.KL_GUARD_TAU, out.data_ptr(), fl, s.cuda_stream)
        if timed:
            ev[1].record(s)
            s.synchronize()
            guarded[0] = int(out[rows:].view(t.int32)[1].item())
        nat.call("pf_target_prep_f64", rowp, k, 1e-150, tgt, 0, tmask, fl, s.cuda_stream)
        if timed:
            ev[2].record(s)
        nat.call("pf_dense_tv_f32", P32.data_ptr(), ld32, rows, k, tgt, tmask, 1e-150, tau, dk.row0,
                 target, dk.is_interior.data_ptr(), dk.P.data_ptr(), dk.ld, out.data_ptr(), fl,
                 s.cuda_stream)
        if timed:
            ev[3].record(s)
            s.synchronize()
            guarded[1] = int(out[rows:].view(t.int32)[1].item())
            ms[0] += ev[0].elapsed_time(ev[1])
            ms[1] += ev[2].elapsed_time(ev[3])

    for _ in range(3):
        step(False)
    n = max(3, steps)
    for _ in range(n):
        step(True)
    kl_ms, tv_ms = ms[0] / n, ms[1] / n
    return {"workload": "FP32 storage mode (P streamed as FP32, FP64 logs / accumulation, "
                        "1e-5 relative tolerance)",
            "evals_per_s": 2 * rows / ((kl_ms + tv_ms) / 1e3),
            "kl_guarded_rows": guarded[0], "tv_guarded_rows": guarded[1],
            "kl": dict(_roof(rows * (4 * k + 16) + 8 * k, kl_ms, peak),
                       # the FP32-guarded rows are re-read as FP64 rows (8k B each)
                       frac_incl_guard_reads=(rows * (4 * k + 16) + 8 * k + guarded[0] * 8 * k)
                       / (kl_ms / 1e3) / 1e9 / peak),
            "tv": dict(_roof(rows * (4 * k + 8) + 8 * k, tv_ms, peak),
                       frac_incl_guard_reads=(rows * (4 * k + 8) + 8 * k + guarded[1] * 8 * k)
                       / (tv_ms / 1e3) / 1e9 / peak)}


def csr_fields_extra(t, nat, dev, pf, dk, target, steps, peak):
    """C3: sparsify (K4) at the reference default 1/sqrt(n), then CSR KL + TV
    fields (K5/K6) to one target on the device CSR."""
    n, rows, k = dk.n, dk.rows, dk.k
    cut = (1.0 / math.sqrt(n)) / k
    s = t.cuda.current_stream(dk.device)
    t.cuda.synchronize()
    w0 = time.perf_counter()
    e0, e1 = _events(t)
    e0.record(s)
    dc = dk.csr(cut, False)
    e1.record(s)
    t.cuda.synchronize()
    build_ms, build_wall = e0.elapsed_time(e1), time.perf_counter() - w0
    # again with the allocator warm (the first build pays ~1 GB of cudaMalloc)
    del dc
    dk._csr.clear()
    t.cuda.synchronize()
    w0 = time.perf_counter()
    e0.record(s)
    dc = dk.csr(cut, False)
    e1.record(s)
    t.cuda.synchronize()
    build_ms_warm, build_wall_warm = e0.elapsed_time(e1), time.perf_counter() - w0
    k_pad = dev.round_up(k, 2)
    stage = t.empty(16 * k_pad + dev.round_up(k, 16), dtype=t.uint8, device=dk.device)
    logt = stage.data_ptr() + 8 * k_pad
    vp = t.empty(k_pad + 4, dtype=t.float64, device=dk.device)
    out = t.empty(rows + 2, dtype=t.float64, device=dk.device)
    flags = out.data_ptr() + rows * 8
    kl_entry, kl_idx = dc.field_entry("kl")   # 16-bit columns (k < 65,536)
    tv_entry, tv_idx = dc.field_entry("tv")
    ev = _events(t, 4)
    ms = [0.0, 0.0]

    def step(timed):
        nat.call("pf_target_prep_f64", dk.P[target].data_ptr(), k, 1e-300, stage.data_ptr(), logt,
                 stage.data_ptr() + 16 * k_pad, flags, s.cuda_stream)
        if timed:
            ev[0].record(s)
        nat.call(kl_entry, dc.indptr.data_ptr(), kl_idx, dc.data.data_ptr(),
                 dc.log_data.data_ptr(), dc.hs.data_ptr(), rows, k, logt,
                 pf.divergence.KL_GUARD_TAU, 0, 0, rows, out.data_ptr(), 0, flags,
                 1, s.cuda_stream)
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
    n_t = max(3, steps)
    for _ in range(n_t):
        step(True)
    kl_ms, tv_ms = ms[0] / n_t, ms[1] / n_t
    nnz = dc.nnz
    ib = 2 if dc.indices16 is not None else 4
    # streamed: data (8) + column (2 or 4) per stored entry incl. row-alignment pads
    str_kl = dc.nnz_pad * (8 + ib) + rows * (8 + 8 + 8) + 8 * k
    str_tv = dc.nnz_pad * (8 + ib) + rows * (8 + 8 + 8) + 16 * k
    # the public sparsify (host scipy views) end to end, for the wall-time record
    pk = _host_pk_of(t, pf, dev, dk) if rows * k * 8 < 8e9 else None
    sp_wall = None
    if pk is not None:
        dk._csr.clear()   # the public call builds its CSR (K4) inside the timed region
        t.cuda.synchronize()
        w0 = time.perf_counter()
        sp = pf.sparsify(pk)
        sp_wall = time.perf_counter() - w0
        del sp
    res = {"columns": "uint16 device copy (10 B/entry streamed; algorithmic bytes are scipy's "
                      "int32 layout, 12 B/entry)" if dc.indices16 is not None else "int32",
           "nnz": nnz, "nnz_per_row": nnz / rows,
           "sparsity_percent": 100.0 * (1 - nnz / (rows * k)),
           "device_csr_build_ms": build_ms, "device_csr_build_wall_s": build_wall,
           "device_csr_build_warm_allocator_ms": build_ms_warm,
           "device_csr_build_warm_allocator_wall_s": build_wall_warm,
           "public_sparsify_wall_s": sp_wall,
           "evals_per_s": 2 * rows / ((kl_ms + tv_ms) / 1e3),
           "kl": _roof(nnz * 12 + rows * 24 + 8 * k, kl_ms, peak, str_kl),
           "tv": _roof(nnz * 12 + rows * 24 + 16 * k, tv_ms, peak, str_tv)}
    del dc
    dk._csr.clear()
    return res


def _host_pk_of(t, pf, dev, dk):
    """A host PoissonKernel whose device mirror is `dk` (as poisson_kernel() returns)."""
    from paper_1708_02845_b200 import laplacian as L
    dense = L.dense_to_host(dk.P, dk.n, dk.k)
    pk = pf.PoissonKernel(dense, dk.boundary, dk.residual, dk.row_sum_error)
    dev.register(pk.dense, dk)
    return pk


def extra_small_real(t, nat, dev, pf, L, device, name, steps, peak):
    """C2 / C2' on their real P (device build): dense KL/TV, FP32 mode, and for
    C2 the C3 CSR fields, each beside its CPU baseline on real rows."""
    import numpy as np
    from workloads.meshes import default_endpoints
    omesh, mesh_s = build_mesh(name)
    dp, dk, build = device_build(t, L, omesh, device)
    build["mesh_build_s"] = mesh_s
    _, target = default_endpoints(omesh)
    res = {"workload": WORKLOADS[name][2].replace("row slabs over N GPUs", "1 GPU"),
           "preprocessing": build, "target": int(target)}
    res.update(dense_fields_extra(t, nat, dev, pf, dk, target, steps, peak))
    rows_of = device_rows(t, dk, target)
    if not NO_CPU:
        try:
            ref = CpuReference(rows_of, dk.k, 5.0, os.cpu_count() or 1, "real rows of this P")
            v, _ = ref.step()
            res["cpu_baseline"] = {"value": v, "unit": "evals/s", "cores": ref.threads,
                                   "kind": "port", "sample": ref.sample}
        except Exception as exc:
            res["cpu_baseline"] = {"error": f"{type(exc).__name__}: {exc}"}
    if name == "c2":
        c3 = {"workload": "C3: the C2 real P sparsified at 1/sqrt(n) (K4), CSR KL+TV fields "
                          "(K5/K6), 1 GPU"}
        c3.update(csr_fields_extra(t, nat, dev, pf, dk, target, steps, peak))
        if not NO_CPU:
            try:
                c3["cpu_baseline"] = cpu_baseline_csr(rows_of(4096), dk.n)
            except Exception as exc:
                c3["cpu_baseline"] = {"error": f"{type(exc).__name__}: {exc}"}
        res["c3_csr"] = c3
    del dk, dp
    t.cuda.empty_cache()
    return res


def extra_c5(t, nat, dev, pf, device, dk, omesh, steps, peak):
    """C5 on the C4 real P: 1,024 targets' KL fields as one contraction (K7 on
    the int8 tensor pipe), then 10,000 paths traced through those fields
    straight from the (n, T) output (pf_trace_fields_f64)."""
    import ctypes
    import numpy as np
    from paper_1708_02845_b200 import paths as PP
    from workloads.meshes import c5_jobs
    rows, k = dk.rows, dk.k
    targets, src, fo = c5_jobs(omesh)
    T = targets.size
    tg = t.from_numpy(targets).to(device)
    H = dk.negentropy(1e-300)
    ldl = dev.round_up(k, 16)
    Pt = dk.P.index_select(0, tg)
    L_ = t.empty((T, ldl), dtype=t.float64, device=device)
    Tc = t.empty((T, ldl), dtype=t.float64, device=device)
    out = t.empty((rows, T), dtype=t.float64, device=device)
    cnt = t.zeros(1, dtype=t.int32, device=device)
    s = t.cuda.current_stream(device)
    e0, e1, e2, e3 = _events(t, 4)
    tau = pf.divergence.KL_GUARD_TAU
    gcap = pf.divergence.guard_list_cap(rows, T)
    glist = t.empty(gcap + 1, dtype=t.int64, device=device)
    e0.record(s)
    At, eat = dk.slices_tiled(1e-300)       # once per P (like H); the product's layout
    e1.record(s)
    t.cuda.synchronize()
    slice_ms = e0.elapsed_time(e1)
    Bt = t.empty(dev.i8_tiled_bytes(T, k), dtype=t.uint8, device=device)
    eb = t.empty(T, dtype=t.int32, device=device)
    bad = t.zeros(1, dtype=t.int32, device=device)
    rowmajor = {}

    def batch_i8(timed=False, grade=64, pair=1):
        # pair=1: the product path (dv_field_batch_device): CTA-pair kernel on the
        # tiled planes; pair=0: the single-CTA kernel on row-major planes, beside it
        cnt.zero_()
        nat.call("pf_batch_prep_f64", Pt.data_ptr(), Pt.stride(0), T, k, ldl, 1e-300, 0,
                 L_.data_ptr(), Tc.data_ptr(), 0, s.cuda_stream)
        if pair:
            nat.call("pf_slice_targets_u8_tiled", L_.data_ptr(), ldl, T, k, Bt.data_ptr(),
                     eb.data_ptr(), bad.data_ptr(), s.cuda_stream)
        else:
            if not rowmajor:
                A, ea, ldk = dk.slices(1e-300)
                rowmajor.update(A=A, ea=ea, ldk=ldk,
                                B=t.empty((7, T, ldk), dtype=t.uint8, device=device))
            rm = rowmajor
            nat.call("pf_slice_targets_u8", L_.data_ptr(), ldl, T, k, rm["ldk"], rm["B"].data_ptr(),
                     eb.data_ptr(), bad.data_ptr(), s.cuda_stream)
        if timed:
            e1.record(s)
        glist[:1].zero_()
        if pair:
            nat.call("pf_batched_kl_i8_tiled", At.data_ptr(), eat.data_ptr(), rows, Bt.data_ptr(),
                     eb.data_ptr(), T, k, H.data_ptr(), tg.data_ptr(), tau, 0, out.data_ptr(),
                     out.stride(0), grade, glist.data_ptr(), gcap, s.cuda_stream)
        else:
            nat.call("pf_batched_kl_i8_listed", rm["A"].data_ptr(), rm["ea"].data_ptr(), rows,
                     rm["B"].data_ptr(), eb.data_ptr(), T, k, rm["ldk"], H.data_ptr(),
                     tg.data_ptr(), tau, 0, out.data_ptr(), out.stride(0), grade, 0,
                     glist.data_ptr(), gcap, s.cuda_stream)
        if timed:
            e2.record(s)
        nat.call("pf_batched_kl_fixup_list_f64", dk.P.data_ptr(), dk.ld, rows, k, Tc.data_ptr(),
                 ldl, T, 1e-300, out.data_ptr(), out.stride(0), cnt.data_ptr(), glist.data_ptr(),
                 gcap, s.cuda_stream)
        if timed:
            e3.record(s)

    def batch_f64():
        cnt.zero_()
        nat.call("pf_batch_prep_f64", Pt.data_ptr(), Pt.stride(0), T, k, ldl, 1e-300, 0,
                 L_.data_ptr(), Tc.data_ptr(), 0, s.cuda_stream)
        nat.call("pf_batched_kl_f64", dk.P.data_ptr(), dk.ld, rows, k, H.data_ptr(), L_.data_ptr(),
                 Tc.data_ptr(), ldl, T, tg.data_ptr(), 1e-300, tau, 0,
                 out.data_ptr(), out.stride(0), cnt.data_ptr(), s.cuda_stream)

    def timed(fn, reps):
        fn()
        t.cuda.synchronize()
        st, en = _events(t)
        st.record(s)
        for _ in range(reps):
            fn()
        en.record(s)
        t.cuda.synchronize()
        return st.elapsed_time(en) / reps

    ms_f32grade = timed(lambda: batch_i8(grade=32), 2)
    ms64 = timed(batch_f64, 1)
    ms = timed(batch_i8, 3)
    gemms, fixups = [], []
    for _ in range(3):   # the GEMM / fixup split: median of three instrumented batches
        batch_i8(True)
        t.cuda.synchronize()
        gemms.append(e1.elapsed_time(e2))
        fixups.append(e2.elapsed_time(e3))
    gemm_only, fixup_ms = sorted(gemms)[1], sorted(fixups)[1]
    batch_i8(True, pair=0)                  # the single-CTA kernel beside it
    t.cuda.synchronize()
    gemm_single = e1.elapsed_time(e2)
    rowmajor.clear()
    dk._H.pop(("i8", 1e-300), None)         # the row-major planes only served that comparison
    guarded = int(cnt.item())
    flops = 2.0 * rows * k * T
    fl = ctypes.c_int64(0)
    probe = t.empty(2, dtype=t.float64, device=device)

    def probe_rate(name, iters, *mode):
        nat.call(name, iters // 4, *mode, ctypes.byref(fl), probe.data_ptr(), s.cuda_stream)
        t.cuda.synchronize()
        e0.record(s)
        nat.call(name, iters, *mode, ctypes.byref(fl), probe.data_ptr(), s.cuda_stream)
        e1.record(s)
        t.cuda.synchronize()
        return fl.value / (e0.elapsed_time(e1) / 1e3) / 1e12

    def probe_sustained(name, iters, *mode, reps=8):
        """The probe back to back for ~0.3 s (the board at its power cap, as
        during a C5 batch); rate over the last half of the launches."""
        for _ in range(reps // 2):
            nat.call(name, iters, *mode, ctypes.byref(fl), probe.data_ptr(), s.cuda_stream)
        e0.record(s)
        for _ in range(reps - reps // 2):
            nat.call(name, iters, *mode, ctypes.byref(fl), probe.data_ptr(), s.cuda_stream)
        e1.record(s)
        t.cuda.synchronize()
        return fl.value * (reps - reps // 2) / (e0.elapsed_time(e1) / 1e3) / 1e12

    dfma_tf = probe_rate("pf_probe_dfma_f64", 1 << 16)
    i8_tops = probe_rate("pf_probe_umma_i8", 1 << 14, 1)
    i8_tops_sustained = probe_sustained("pf_probe_umma_i8", 1 << 14, 1)
    i8_tops_pattern = probe_rate("pf_probe_umma_i8", 1 << 14, 0)
    i8_tops_pattern_sustained = probe_sustained("pf_probe_umma_i8", 1 << 14, 0)
    int_ops = 34 * flops
    ach = int_ops / (gemm_only / 1e3) / 1e12
    res = {"workload": f"C5: C4 real P ({rows:,} x {k:,}), T = {T} targets (SURVEY §8d C5), KL "
                       "as one contraction + fused epilogue (K7 on the int8 tensor pipe: 34 exact "
                       f"byte-pair GEMMs emulating the FP64 GEMM), then {src.size:,} paths traced, "
                       "1 GPU",
           "evals_per_s": rows * T / (ms / 1e3), "ms_per_batch": ms,
           "gemm_ms": gemm_only, "gemm_ms_single_cta_kernel": gemm_single,
           "guarded_pairs": guarded, "fixup_ms": fixup_ms,
           "fp64_equivalent_tflops": flops / (ms / 1e3) / 1e12,
           "slice_rows_ms_once_per_P": slice_ms,
           "roofline": {"bound": "tensor", "achieved": ach, "peak": i8_tops_sustained,
                        "unit": "TOPS (int8)", "frac": ach / i8_tops_sustained,
                        "frac_of_burst_probe": ach / i8_tops, "burst_peak": i8_tops,
                        "pattern_operand_probe": {
                            "burst": i8_tops_pattern, "sustained": i8_tops_pattern_sustained,
                            "frac_of_sustained": ach / i8_tops_pattern_sustained,
                            "note": "the round-1 probe (operand bytes 0..3): the tensor pipe "
                                    "draws less power on it and holds a higher clock"},
                        "algorithmic_ops_per_launch": int_ops,
                        "peak_kind": "measured: pf_probe_umma_i8 (M128 N256 K32 u8 tcgen05.mma "
                                     "back to back from shared memory, all SMs, random operand "
                                     "bytes as K7's slice planes and as MEASURED_PEAKS' bf16 "
                                     "matmul), sustained (~0.3 s back to back, under the 1 kW "
                                     "power cap, as the ~0.1 s C5 GEMM runs); burst_peak is "
                                     "one launch",
                        "kernel": "pf::batched_kl_i8_pp_kernel<7,9,0,tiled> (persistent tcgen05 "
                                  "cta_group::2 pair on the tiled planes, epilogue off the MMA "
                                  "critical path)"},
           "fp32_grade": {"note": "same kernel, 15 byte-pair GEMMs (levels 2..6 of the top 5 "
                                  "planes): the north-star FP32 tolerance 1e-5",
                          "ms_per_batch": ms_f32grade,
                          "evals_per_s": rows * T / (ms_f32grade / 1e3)},
           "fp64_dmma_path": {"ms_per_batch": ms64, "evals_per_s": rows * T / (ms64 / 1e3),
                              "achieved_tflops": flops / (ms64 / 1e3) / 1e12,
                              "dfma_peak_tflops": dfma_tf,
                              "frac": flops / (ms64 / 1e3) / 1e12 / dfma_tf}}
    del At, Bt
    # ---- the tracer over the K7 fields, read in place: field j = column j of `out`
    for _ in range(2):   # warm-up at full size: the 2.7 GB path workspace is allocated here
        PP.trace_arrays(omesh_tri(omesh, pf), out, targets, src, fo, layout=(1, T))
    t.cuda.synchronize()
    w0 = time.perf_counter()
    e0.record(s)
    buf, counts, over, extra = PP.trace_arrays(omesh_tri(omesh, pf), out, targets, src, fo,
                                               layout=(1, T))
    e1.record(s)
    t.cuda.synchronize()
    tr_ms = e0.elapsed_time(e1)
    status = buf.status[:src.size].cpu().numpy()
    res["tracer"] = {"paths": int(src.size), "ms": tr_ms,
                     "wall_ms_incl_launch": 1e3 * (time.perf_counter() - w0),
                     "paths_per_s": src.size / (tr_ms / 1e3),
                     "locations_per_s": float(counts.sum()) / (tr_ms / 1e3),
                     "mean_locations": float(counts.mean()), "max_locations": int(counts.max()),
                     "reached": int((status == 0).sum()), "overflow_reruns": int(over.size)}
    if not NO_CPU:
        try:
            res["cpu_baseline"] = cpu_baseline_batched(device_rows(t, dk, int(targets[0]))(4096))
        except Exception as exc:
            res["cpu_baseline"] = {"error": f"{type(exc).__name__}: {exc}"}
        try:
            res["tracer"]["cpu_baseline"] = cpu_baseline_tracer(
                omesh, lambda j: out[:, j].cpu().numpy(), targets, src, fo)
        except Exception as exc:
            res["tracer"]["cpu_baseline"] = {"error": f"{type(exc).__name__}: {exc}"}
    del out, L_, Tc, Pt
    dk._H.pop(("i8", 1e-300), None)
    t.cuda.empty_cache()
    return res


_TRI = {}


def omesh_tri(omesh, pf):
    """The product TriMesh of a workload mesh (cached: its device topology is)."""
    key = id(omesh)
    if key not in _TRI:
        _TRI[key] = pf.TriMesh(omesh.vertices, omesh.triangles)
    return _TRI[key]


def extra_synthetic_c2(t, nat, dev, pf, device, steps, peak):
    """Round 1's headline, kept for continuity: a synthetic C2-shaped slab
    (softmax rows, one zero column), dense KL + TV."""
    import numpy as np
    rows, k = 102_104, 4_250
    ld = dev.leading_dim(k)
    P = t.empty((rows, ld), dtype=t.float64, device=device)
    g = t.Generator(device=device)
    g.manual_seed(1234)
    for a in range(0, rows, 8192):
        b = min(rows, a + 8192)
        x = t.randn((b - a, k), dtype=t.float64, device=device, generator=g)
        x[:, 0] = -float("inf")
        P[a:b, :k] = t.softmax(x, dim=1)
    P[:, k:] = 0.0
    dk = dev.DeviceKernel(None, np.array([], np.int64), device=device, rows=rows, n=rows, k=k,
                          P_dev=P)
    res = {"workload": "synthetic C2 shape 102,104 x 4,250 (round-1 headline)"}
    res.update(dense_fields_extra(t, nat, dev, pf, dk, rows // 3 + 1, steps, peak, f32=False))
    del dk, P
    t.cuda.empty_cache()
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
            "reference_python_json_ms_extrapolated": ref_json_ms}


def extra_poisson(t, nat, dev, device, L, dp_c4=None, dfma_peak=None):
    """the Poisson kernel P itself on the device at C2 (beside
    SuperLU on all host cores, oracle/inputs.poisson_kernel_parallel) and C4
    (phases of a re-solve of the headline mesh)."""
    import numpy as np
    from oracle import inputs as I
    out = {"dfma_peak_tflops": dfma_peak}
    todo = [("c2", None)] + ([("c4", dp_c4)] if dp_c4 is not None else [])
    for name, dp in todo:
        omesh, mesh_s = (None, None) if dp is not None else build_mesh(name)
        if dp is None:
            w0 = time.perf_counter()
            dp = L.DevicePoisson(omesh, device=device)
            setup_s = time.perf_counter() - w0
        else:
            setup_s = None
        P, reps = None, []
        for rep in range(3):
            dp._lap, dp._F = None, None
            t.cuda.synchronize()
            e0, e1 = _events(t)
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
                   "peak": dfma_peak,
                   "frac": (fl["backward"] / (bwd * 1e-3) / 1e12 / dfma_peak
                            if dfma_peak else None),
                   "algorithmic_flops": fl["backward"],
                   "kernel": "pf::mf_bwd_gemm_kernel (DMMA m8n8k4, gathered rows)"}}
        if name == "c2" and not NO_CPU:
            kk = dp.k
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
            res["max_rel_vs_superlu_2000_rows"] = float(
                (np.abs(x[big] - y[big]) / y[big]).max())
            del ref
        out[name] = res
        del P
        t.cuda.empty_cache()
    return out


def measure_read_peak(t, nat, device, gb=16):
    """The pure-read HBM ceiling (pf_probe_hbm_read over `gb` GB, best of 5), GB/s."""
    try:
        n = (gb << 30) // 8
        buf = t.zeros(n, dtype=t.float64, device=device)
        sink = t.zeros(1, dtype=t.float64, device=device)
        s = t.cuda.current_stream(device)
        e0, e1 = _events(t)
        best = None
        for r in range(6):
            e0.record(s)
            nat.call("pf_probe_hbm_read", buf.data_ptr(), n, sink.data_ptr(), s.cuda_stream)
            e1.record(s)
            t.cuda.synchronize()
            ms = e0.elapsed_time(e1)
            if r and (best is None or ms < best):
                best = ms
        del buf
        t.cuda.empty_cache()
        return n * 8 / (best / 1e3) / 1e9
    except Exception:
        return None


EXTRAS_DEADLINE_S = 900
_emit_lock = __import__("threading").Lock()
_emitted = []


def emit(line):
    """Print the one JSON line (at most once: the N > 1 watchdog may race the normal path)."""
    with _emit_lock:
        if _emitted:
            return
        _emitted.append(True)
        print(json.dumps(line), flush=True)


def run_native(args):
    import numpy as np
    import torch as t

    import paper_1708_02845_b200 as pf
    from paper_1708_02845_b200 import _device as dev
    from paper_1708_02845_b200 import _native as nat
    from paper_1708_02845_b200 import laplacian as L
    from paper_1708_02845_b200 import parallel as par
    from workloads.meshes import default_endpoints

    ws, rank, local = dist_env()
    if args.gpus != ws and ws > 1:
        raise SystemExit(f"--gpus {args.gpus} but WORLD_SIZE={ws}")
    t.cuda.set_device(local)
    device = t.device("cuda", local)
    dist = None
    single = ws == 1 and not args.sharded   # --sharded: the N-rank path on one rank
    if not single:
        # control plane (rendezvous, NCCL unique id, barriers, timing max) on gloo;
        # the data plane is NCCL through the C ABI (parallel.NcclComm)
        import torch.distributed as dist
        if ws == 1:
            import socket
            with socket.socket() as so:
                so.bind(("127.0.0.1", 0))
                os.environ.setdefault("MASTER_PORT", str(so.getsockname()[1]))
            os.environ.setdefault("MASTER_ADDR", "127.0.0.1")
            os.environ.setdefault("RANK", "0")
            os.environ.setdefault("WORLD_SIZE", "1")
        dist.init_process_group("gloo")

    n_expect, k_expect, desc = WORKLOADS[args.workload]
    omesh, mesh_s = build_mesh(args.workload)
    n = omesh.n
    _, target = default_endpoints(omesh)
    bounds = par.partition_rows(n, ws)
    sharded = None
    if single:
        dp, dk, prep = device_build(t, L, omesh, device)
    else:
        dp = None
        t.cuda.synchronize()
        w0 = time.perf_counter()
        sharded = par.ShardedField.from_mesh(omesh, dist, device=device, bounds=bounds)
        t.cuda.synchronize()
        dk = sharded.slab
        prep = {"slab_build_wall_s": time.perf_counter() - w0, "residual": dk.residual,
                "row_sum_error": dk.row_sum_error}
    prep["mesh_build_s"] = mesh_s
    rows, k = dk.rows, dk.k
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
        v = t.tensor([x], dtype=t.float64)
        dist.all_reduce(v, op=dist.ReduceOp.MAX)
        return float(v.item())

    for _ in range(args.warmup):
        step.run()
    barrier()
    kl_ms, tv_ms = step.kernel_ms(args.steps)   # kernel-level pass (events on the stream)
    kl_ms_max = max_over_ranks(kl_ms)

    e0, e1 = _events(t)
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
    value = 2 * n * args.steps / (el_ms / 1e3)
    flags_kl = step.out_kl[rows:].view(t.int32).cpu().numpy()
    guarded = int(flags_kl[1])
    if dist is not None:
        g = t.tensor([guarded], dtype=t.int64)
        dist.all_reduce(g)
        guarded = int(g.item())

    # ------------------------------------------------ e2e via the public API
    if single:
        w0 = time.perf_counter()
        dense = L.dense_to_host(dk.P, n, k)
        host_copy_s = time.perf_counter() - w0
        pk = pf.PoissonKernel(dense, dk.boundary, dk.residual, dk.row_sum_error)
        dev.register(pk.dense, dk)
        kl, tv = pf.builtin_f("kl"), pf.builtin_f("tv")
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
        e2e = {"value": 2 * n * args.steps / e2e_s, "unit": "evals/s",
               "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 2 * (rows + 2) * 8,
               "ms_per_step": 1e3 * e2e_s / args.steps,
               "step_ms_min_median_max": [1e3 * min(per), 1e3 * statistics.median(per),
                                          1e3 * max(per)],
               "precision_flags": list(fkl.precision_flags),
               "note": "wall clock of dv_field(pk, kl, t) + dv_field(pk, tv, t) per step through "
                       "the public API on the PoissonKernel poisson_kernel(mesh) returns (host "
                       "dense + its resident device mirror, as DomainContext keeps it); the "
                       "target index is a kernel argument (no H2D bytes); each n-vector field "
                       "+ flag words is copied D2H into a pinned numpy array and returned as a "
                       "read-only ScalarField"}
        # cold: a PoissonKernel the device has not seen (first query of a DomainContext):
        # the host P crosses PCIe inside the timed region
        dev.evict(pk)
        del step
        t.cuda.empty_cache()
        barrier()
        p0 = time.perf_counter()
        fkl = pf.dv_field(pk, kl, target)
        ftv = pf.dv_field(pk, tv, target)
        cold_s = time.perf_counter() - p0
        e2e["cold"] = {"value": 2 * n / cold_s, "unit": "evals/s",
                       "h2d_bytes_per_step": n * k * 8 + n, "d2h_bytes_per_step": 2 * (n + 2) * 8,
                       "ms_per_step": 1e3 * cold_s, "steps": 1,
                       "h2d_gbs_lower_bound": n * k * 8 / cold_s / 1e9,
                       "note": "dv_field(kl) + dv_field(tv) on a PoissonKernel with no device "
                               "mirror: pinned staged upload of the host P (_hostpool."
                               "upload_rows), K1 negentropy, K2, K3, D2H of both fields"}
        dev.evict(pk)
        dev.register(pk.dense, dk)
        prep["host_copy_of_P_s"] = host_copy_s
        del fkl, ftv
        t.cuda.empty_cache()
        step = None
    else:
        from paper_1708_02845_b200 import _hostpool
        kl, tv = pf.builtin_f("kl"), pf.builtin_f("tv")

        def e2e_step():
            a = sharded.field(kl, target)
            ha = _hostpool.to_host(t, a.values, stream)
            b = sharded.field(tv, target)
            hb = _hostpool.to_host(t, b.values, stream)
            return ha, hb, a.precision_flags

        for _ in range(args.warmup):
            keep = e2e_step()
        barrier()
        w0 = time.perf_counter()
        for _ in range(args.steps):
            keep = e2e_step()
        barrier()
        e2e_s = max_over_ranks(time.perf_counter() - w0)
        e2e = {"value": 2 * n * args.steps / e2e_s, "unit": "evals/s",
               "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 2 * (n + ws) * 8,
               "ms_per_step": 1e3 * e2e_s / args.steps, "precision_flags": list(keep[2]),
               "note": "wall clock (max over ranks) of ShardedField.field(kl|tv, t) per step: "
                       "NCCL broadcast of the target row from its owner, the slab kernels, the "
                       "flag-word max-reduction, and each rank's field slab copied to host "
                       "memory"}
        del keep

    # ------------------------------------------------ CPU baseline (rank 0, N=1)
    cpu = None
    if rank == 0 and single and not args.no_cpu:
        threads = os.cpu_count() or 1
        ref = CpuReference(None, k, args.cpu_budget, threads, "real rows of this P",
                           matrix=pk.dense, target=target)
        v, el = ref.step()
        cpu = {"value": v, "unit": "evals/s", "cores": threads, "kind": "port",
               "sample": ref.sample + f" ({el:.1f} s); oracle/divergence.py restating "
                                      "pathfield divergence.py:137-187 (numpy)",
               "host": host_info()}

    peak, peak_kind = peaks()
    read_peak = measure_read_peak(t, nat, device)
    bytes_kl = rows * (8 * k + 16) + 8 * k
    bytes_tv = rows * (8 * k + 8) + 8 * k
    traffic = None
    prof = ROOT / "profiles" / "ncu_summary.json"
    if prof.exists() and single:
        try:
            traffic = json.loads(prof.read_text()).get(args.workload, {}).get("dense_kl_dram_bytes")
        except Exception:
            traffic = None
    roof = _roof(bytes_kl, kl_ms, peak)
    roof.update({"read_peak_gbps": read_peak,
                 "frac_of_read_peak": roof["achieved"] / read_peak if read_peak else None,
                 "read_peak_kind": "measured in this run: pf_probe_hbm_read, 16 GB streamed "
                                   "with the field kernels' 16-byte loads and no arithmetic",
                 "traffic": traffic,
                 "kernel": "pf::dense_kl_kernel (guarded rows re-evaluated in place)",
                 "slowest_rank_avg_launch_ms": kl_ms_max,
                 "peak_kind": ("measured (MEASURED_PEAKS.json hbm_gbs, copy)"
                               if peak_kind == "measured" else "fallback 6.65 TB/s")})

    def headline():
        return {
        "metric": METRIC, "value": value, "unit": "evals/s", "n_gpus": ws,
        "steps": args.steps, "warmup": args.warmup, "ms_per_step": el_ms / args.steps,
        "higher_is_better": True, "scaling": "strong", "vs_baseline": None, "dtype": "f64",
        "data": "real: reference-generator mesh, Poisson kernel P built on the GPU",
        "config": {"workload": desc, "n": n, "k": k, "rows_per_gpu_max": max(b - a for a, b in bounds),
                   "parallelism": f"row-slab x{ws}" + ("" if single else " (sharded path)"),
                   "target": int(target),
                   "l2": "inputs larger than L2 (P slab %.2f GB/GPU vs 126 MB L2)"
                         % (rows * dk_ld(k) * 8 / 1e9)},
        "roofline": roof,
        "roofline_tv": dict(_roof(bytes_tv, tv_ms, peak),
                            frac_of_read_peak=(bytes_tv / (tv_ms / 1e3) / 1e9 / read_peak
                                               if read_peak else None)),
        "kl_guarded_rows": guarded,
        "cpu_baseline": cpu,
        "e2e": e2e,
        "gpu_launches": launches,
        "clocks": clocks.summary(),
        "preprocessing": prep,
    }

    extras = {}
    want = set(args.extras.split(",")) if not args.no_extras else set()
    if single:
        def run_extra(name, fn):
            if name not in want:
                return
            try:
                extras[name] = fn()
            except Exception as exc:  # an extra must never hide the headline number
                extras[name] = {"error": f"{type(exc).__name__}: {exc}"}
            t.cuda.empty_cache()

        if args.workload == "c4":
            run_extra("c4_f32", lambda: extra_f32(t, nat, dev, pf, dk, target, args.steps, peak))
            dk._p32 = None
            dk._H.pop(("f32", 1e-300), None)
            t.cuda.empty_cache()
            run_extra("c5", lambda: extra_c5(t, nat, dev, pf, device, dk, omesh, args.steps,
                                             peak))
        run_extra("poisson", lambda: extra_poisson(
            t, nat, dev, device, L, dp if args.workload == "c4" else None,
            ((extras.get("c5") or {}).get("fp64_dmma_path") or {}).get("dfma_peak_tflops")))
        pk = None
        dev._cache.clear()
        del dk, dp
        t.cuda.empty_cache()
        for name in ("c2", "c2p"):
            if name != args.workload:
                run_extra(name, lambda name=name: extra_small_real(t, nat, dev, pf, L, device,
                                                                   name, args.steps, peak))
        run_extra("c2_synthetic", lambda: extra_synthetic_c2(t, nat, dev, pf, device,
                                                             args.steps, peak))
        run_extra("wire", lambda: extra_wire(t, dev, pf, device))
    else:
        del step
        t.cuda.empty_cache()
        # A rank that fails inside an extra while the others sit in a collective would
        # hang the job before the headline line is printed: past EXTRAS_DEADLINE_S the
        # watchdog prints the line with the extras finished so far and ends every rank.
        partial = {}

        def expire():
            if rank == 0:
                emit(dict(headline(), extras=dict(partial, timeout=(
                    f"N>1 extras unfinished after {EXTRAS_DEADLINE_S} s"))))
            os._exit(0)

        import threading
        dog = threading.Timer(EXTRAS_DEADLINE_S, expire)
        dog.daemon = True
        dog.start()
        extras.update(run_sharded_extras(t, nat, dev, pf, L, par, dist, device, sharded,
                                         omesh, want, args, partial))
        dog.cancel()

    line = dict(headline(), extras=extras)
    if rank == 0:
        emit(line)
    if sharded is not None:
        sharded.close()
    if dist is not None:
        dist.barrier()
        dist.destroy_process_group()
    return 0


def dk_ld(k):
    return (k + 63) // 64 * 64


def run_sharded_extras(t, nat, dev, pf, L, par, dist, device, sharded, omesh, want, args,
                       out=None):
    """N > 1 side configs (strong scaling of the configs BASELINE names):
    C3 — CSR KL + TV over nnz-balanced row slabs of the C2 real P; C5 — 1,024
    targets partitioned over the ranks (P replicated, K7), each rank tracing
    the paths of its own targets (parallel.trace_batch; no field exchange)."""
    import numpy as np
    ws, rank = dist.get_world_size(), dist.get_rank()
    out = {} if out is None else out   # filled as each extra finishes (the watchdog reads it)

    def max_ms(x):
        v = t.tensor([x], dtype=t.float64)
        dist.all_reduce(v, op=dist.ReduceOp.MAX)
        return float(v.item())

    if "c3" in want:
        try:
            from workloads.meshes import default_endpoints
            om2, _ = build_mesh("c2")
            _, tgt = default_endpoints(om2)
            dp2 = L.DevicePoisson(om2, device=device)
            full = dp2.device_kernel()
            cut = (1.0 / math.sqrt(full.n)) / full.k
            cnt = t.empty(full.rows, dtype=t.int64, device=device)
            nat.call("pf_csr_count_f64", full.P.data_ptr(), full.ld, full.rows, full.k, cut, 0,
                     cnt.data_ptr(), t.cuda.current_stream(device).cuda_stream)
            b3 = par.partition_by_weight(cnt.cpu().numpy(), ws)
            a, b = b3[rank]
            Ps = full.P[a:b].clone()
            slab = dev.DeviceKernel(None, np.asarray(om2.boundary_vertices), device=device,
                                    row0=a, rows=b - a, n=full.n, k=full.k, P_dev=Ps)
            del full, dp2
            t.cuda.empty_cache()
            sf = par.ShardedField(slab, b3, dist, device=device, comm=sharded.comm)
            kl, tv = pf.builtin_f("kl"), pf.builtin_f("tv")
            for _ in range(3):
                sf.sparse_field(kl, tgt)
                sf.sparse_field(tv, tgt)
            e0, e1 = _events(t)
            t.cuda.synchronize()
            dist.barrier()
            e0.record()
            for _ in range(args.steps):
                sf.sparse_field(kl, tgt)
                sf.sparse_field(tv, tgt)
            e1.record()
            t.cuda.synchronize()
            ms = max_ms(e0.elapsed_time(e1)) / args.steps
            nnz = t.tensor([slab.csr(cut, False).nnz], dtype=t.int64)
            dist.all_reduce(nnz)
            out["c3_sharded"] = {"workload": "C3: C2 real P sparsified at 1/sqrt(n), CSR KL + TV "
                                             f"over {ws} nnz-balanced row slabs",
                                 "evals_per_s": 2 * om2.n / (ms / 1e3), "ms_per_step": ms,
                                 "nnz": int(nnz.item()), "slabs": b3}
            del sf, slab, Ps
            t.cuda.empty_cache()
        except Exception as exc:
            out["c3_sharded"] = {"error": f"{type(exc).__name__}: {exc}"}
    if "c5" in want:
        try:
            from workloads.meshes import c5_jobs
            dp4 = L.DevicePoisson(omesh, device=device)
            full = dp4.device_kernel()          # P replicated (32.8 GB fits each B200)
            pk = _DeviceOnlyKernel(full)
            targets, src, fo = c5_jobs(omesh)
            mesh = omesh_tri(omesh, pf)
            par.trace_batch(mesh, pk, pf.builtin_f("kl"), targets, src, fo, dist,
                            status_only=True)   # warm-up (topology, slices, workspaces)
            t.cuda.synchronize()
            dist.barrier()
            w0 = time.perf_counter()
            e0, e1 = _events(t)
            e0.record()
            mine, status, counts = par.trace_batch(mesh, pk, pf.builtin_f("kl"), targets, src,
                                                   fo, dist, status_only=True)
            e1.record()
            t.cuda.synchronize()
            wall = max_ms(1e3 * (time.perf_counter() - w0))
            ms = max_ms(e0.elapsed_time(e1))
            reached = t.tensor([int((status == 0).sum())], dtype=t.int64)
            dist.all_reduce(reached)
            out["c5_distributed"] = {
                "workload": f"C5: {targets.size} targets partitioned over {ws} GPUs (C4 real P "
                            f"replicated), K7 + {src.size:,} paths traced on the owning rank",
                "ms_device_max_over_ranks": ms, "wall_ms": wall,
                "evals_per_s": omesh.n * targets.size / (ms / 1e3),
                "paths_per_s": src.size / (ms / 1e3), "reached": int(reached.item())}
            del full, dp4, pk
            t.cuda.empty_cache()
        except Exception as exc:
            out["c5_distributed"] = {"error": f"{type(exc).__name__}: {exc}"}
    return out


class _DeviceOnlyKernel:
    """A PoissonKernel-shaped handle of a device-built P (no host copy): the
    device cache is keyed on `dense`, so this object stands in for it."""

    def __init__(self, dk):
        import numpy as np
        from paper_1708_02845_b200 import _device as dev
        self.dense = np.empty((0, 0))
        self.boundary = dk.boundary
        self.n, self.k = dk.n, dk.k
        dev.register(self.dense, dk)


def main():
    global NO_CPU
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=20)
    ap.add_argument("--warmup", type=int, default=5)
    ap.add_argument("--impl", default="native", choices=["native", "reference"])
    ap.add_argument("--workload", default="c4", choices=sorted(WORKLOADS))
    ap.add_argument("--cpu-budget", type=float, default=10.0)
    ap.add_argument("--no-cpu", action="store_true")
    ap.add_argument("--no-extras", action="store_true", help="skip the side measurements")
    ap.add_argument("--sharded", action="store_true",
                    help="run the N-rank path (slab build, NCCL collectives, sharded extras) "
                         "even at one rank")
    ap.add_argument("--extras", default="c4_f32,c5,poisson,c2,c2p,c2_synthetic,wire,c3",
                    help="comma list of side measurements (N=1: c4_f32, c5, poisson, c2, c2p, "
                         "c2_synthetic, wire; N>1: c3, c5)")
    args = ap.parse_args()
    NO_CPU = bool(args.no_cpu)
    if args.warmup < 3:
        args.warmup = 3
    if args.impl == "reference":
        return run_reference_arm(args)
    return run_native(args)


if __name__ == "__main__":
    sys.exit(main())
