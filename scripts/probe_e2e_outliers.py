"""Where do the e2e step outliers come from? Time 300 dv_field(kl)+dv_field(tv)
steps through the public API and log garbage-collector pauses beside them."""
import gc
import statistics
import sys
import time
from pathlib import Path

sys.path.insert(0, str(Path(__file__).resolve().parent.parent))
import numpy as np  # noqa: E402
import torch  # noqa: E402
import paper_1708_02845_b200 as pf  # noqa: E402
from paper_1708_02845_b200 import _device as dev  # noqa: E402
import bench  # noqa: E402

rows, k, _ = bench.WORKLOADS["c2"]
ld = dev.leading_dim(k)
P = bench.make_synthetic_slab(torch, rows, k, ld, 7, torch.device("cuda", 0))
host = P[:, :k].cpu().numpy()
pk = pf.PoissonKernel(host, np.array([], np.int64), 0.0, 0.0)
dk = dev.DeviceKernel(None, np.array([], np.int64), n=rows, k=k, P_dev=P)
dev.register(host, dk)
kl, tv = pf.builtin_f("kl"), pf.builtin_f("tv")
gcs = []
t_gc = [0.0]


def cb(phase, info):
    if phase == "start":
        t_gc[0] = time.perf_counter()
    else:
        gcs.append((info["generation"], 1e3 * (time.perf_counter() - t_gc[0])))


for _ in range(5):
    pf.dv_field(pk, kl, 3)
    pf.dv_field(pk, tv, 3)
gc.callbacks.append(cb)
per = []
for i in range(300):
    p0 = time.perf_counter()
    a = pf.dv_field(pk, kl, 3)
    b = pf.dv_field(pk, tv, 3)
    per.append(1e3 * (time.perf_counter() - p0))
gc.callbacks.remove(cb)
per = np.array(per)
print("steps ms: min %.3f median %.3f mean %.3f max %.3f; >2ms at %s" % (
    per.min(), np.median(per), per.mean(), per.max(), np.flatnonzero(per > 2).tolist()))
print("gc pauses (gen, ms):", [(g, round(ms, 2)) for g, ms in gcs if ms > 0.2][:20],
      "count", len(gcs))
