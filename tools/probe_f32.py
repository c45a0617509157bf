"""FP32 storage mode: dense KL / TV launch time on a synthetic C4-sized P
(1,000,386 x 4,102) for the dense32 kernel variant in PF_F32_VARIANT."""
import json, os, sys
from pathlib import Path
sys.path.insert(0, str(Path(__file__).resolve().parent.parent))
import torch as t
from paper_1708_02845_b200 import _native as nat

rows, k = int(os.environ.get("ROWS", 1000386)), 4102
ld = (k + 15) // 16 * 16
ld32 = (k + 3) // 4 * 4
g = t.Generator(device="cuda"); g.manual_seed(0)
P = t.empty((rows, ld), dtype=t.float64, device="cuda")
for r0 in range(0, rows, 100000):
    x = t.rand((min(100000, rows - r0), k), dtype=t.float64, device="cuda", generator=g) ** 4
    P[r0:r0 + x.shape[0], :k] = x / x.sum(1, keepdim=True)
P32 = t.zeros((rows, ld32), dtype=t.float32, device="cuda")
s = t.cuda.current_stream().cuda_stream
nat.call("pf_convert_f32", P.data_ptr(), ld, rows, k, P32.data_ptr(), ld32, s)
H = t.empty(rows, dtype=t.float64, device="cuda")
H64 = t.empty(rows, dtype=t.float64, device="cuda")
nat.call("pf_row_negentropy_f32", P32.data_ptr(), ld32, rows, k, 1e-300, H.data_ptr(), s)
nat.call("pf_row_negentropy_f64", P.data_ptr(), ld, rows, k, 1e-300, H64.data_ptr(), None, s)
target = 12345
tgt = P[target, :k].contiguous()
logt = t.log(tgt)
tmask = t.ones(k, dtype=t.uint8, device="cuda")
inter = t.ones(rows, dtype=t.uint8, device="cuda")
out = t.empty(rows, dtype=t.float64, device="cuda")
flags = t.zeros(4, dtype=t.int32, device="cuda")
res = {}
for name in ("kl", "tv"):
    def run():
        if name == "kl":
            nat.call("pf_dense_kl_f32", P32.data_ptr(), ld32, rows, k, H64.data_ptr(), tgt.data_ptr(),
                     logt.data_ptr(), tmask.data_ptr(), 1e-300, 1e-2, 0, target, inter.data_ptr(),
                     P.data_ptr(), ld, H64.data_ptr(), 1e-3, out.data_ptr(), flags.data_ptr(), s)
        else:
            nat.call("pf_dense_tv_f32", P32.data_ptr(), ld32, rows, k, tgt.data_ptr(), tmask.data_ptr(),
                     1e-300, 1e-2, 0, target, inter.data_ptr(), P.data_ptr(), ld, out.data_ptr(),
                     flags.data_ptr(), s)
    for _ in range(3):
        run()
    e0, e1 = t.cuda.Event(enable_timing=True), t.cuda.Event(enable_timing=True)
    ms = []
    for _ in range(10):
        e0.record(); run(); e1.record(); t.cuda.synchronize(); ms.append(e0.elapsed_time(e1))
    byts = rows * k * 4.0
    res[name] = {"ms_min": min(ms), "ms_med": sorted(ms)[5], "GBps": byts / (min(ms) / 1e3) / 1e9,
                 "frac_6537": byts / (min(ms) / 1e3) / 1e9 / 6537.3}
print(json.dumps({"variant": os.environ.get("PF_F32_VARIANT", "0"), **res}))
