"""CSR K5 / K6 launch times on the real C3 kernel (C2 P sparsified at 1/sqrt(n))."""
import json, math, sys
from pathlib import Path
sys.path.insert(0, str(Path(__file__).resolve().parent.parent))
import torch as t
import paper_1708_02845_b200 as pf
from paper_1708_02845_b200 import _device as dev, _native as nat, laplacian as L
from workloads.meshes import SPECS, build, default_endpoints

m = build(SPECS["c2"])
dk = L.DevicePoisson(m).device_kernel()
_, tgt = default_endpoints(m)
k, rows = dk.k, dk.rows
cut = (1.0 / math.sqrt(dk.n)) / k
dc = dk.csr(cut, False)
s = t.cuda.current_stream().cuda_stream
kp = dev.round_up(k, 2)
st = pf.divergence._Staging(t, k, dk.device)
vp = t.empty(kp + 4, dtype=t.float64, device=dk.device)
out = t.empty(rows + 2, dtype=t.float64, device=dk.device)
fl = out.data_ptr() + rows * 8
kl_e, kl_i = dc.field_entry("kl")
tv_e, tv_i = dc.field_entry("tv")
res = {}
for name in ("kl", "tv"):
    def run():
        if name == "kl":
            nat.call("pf_target_prep_f64", dk.row_ptr(tgt), k, 1e-300, st.tgt, st.logt, st.tmask, fl, s)
            nat.call(kl_e, dc.indptr.data_ptr(), kl_i, dc.data.data_ptr(), dc.log_data.data_ptr(),
                     dc.hs.data_ptr(), rows, k, st.logt, 1e-3, 0, 0, rows, out.data_ptr(), 0, fl, 1, s)
        else:
            nat.call("pf_csr_target_prep_f64", dc.indptr.data_ptr(), dc.indices.data_ptr(), dc.data.data_ptr(),
                     dc.dropped.data_ptr(), tgt, k, vp.data_ptr(), vp.data_ptr() + kp * 8, s)
            nat.call(tv_e, dc.indptr.data_ptr(), tv_i, dc.data.data_ptr(), dc.dropped.data_ptr(), rows, k,
                     vp.data_ptr(), vp.data_ptr() + kp * 8, 0, 0, rows, out.data_ptr(), 0, s)
    for _ in range(3):
        run()
    e0, e1 = t.cuda.Event(enable_timing=True), t.cuda.Event(enable_timing=True)
    ms = []
    for _ in range(15):
        t.cuda.synchronize(); e0.record(); run(); e1.record(); t.cuda.synchronize()
        ms.append(e0.elapsed_time(e1))
    streamed = dc.nnz_pad * 10 + rows * 24
    run(); t.cuda.synchronize()
    import hashlib
    digest = hashlib.sha1(out[:rows].cpu().numpy().tobytes()).hexdigest()[:16]
    res[name] = {"ms_min": min(ms), "ms_med": sorted(ms)[7], "streamed_GBs": streamed / (min(ms) / 1e3) / 1e9,
                 "sha1": digest}
res["nnz"] = dc.nnz
print(json.dumps(res))
