"""Guarded-row cost probe: dense KL launch time on real P (C2, C2') with
tau = 0 (no guarded rows) / 1e-3, with and without the guard workspace."""
import json, sys, time
from pathlib import Path
ROOT = Path(__file__).resolve().parent.parent
sys.path.insert(0, str(ROOT))
import torch as t
import paper_1708_02845_b200 as pf
from paper_1708_02845_b200 import _device as dev, _native as nat, laplacian as L
from workloads.meshes import SPECS, build, default_endpoints

out = {}
for name in sys.argv[1:] or ["c2", "c2p"]:
    m = build(SPECS[name])
    dk = L.DevicePoisson(m).device_kernel()
    _, tgt = default_endpoints(m)
    k, rows = dk.k, dk.rows
    s = t.cuda.current_stream()
    st = pf.divergence._Staging(t, k, dk.device)
    o = t.empty(rows + 2, dtype=t.float64, device="cuda")
    fl = o.data_ptr() + rows * 8
    H = dk.negentropy(1e-300)
    ws = (0, 0)
    res = {}
    for tau in (0.0, 1e-30, 1e-3):
        for use_ws in (False,):
            def run():
                nat.call("pf_target_prep_f64", dk.row_ptr(tgt), k, 1e-300, st.tgt, st.logt, st.tmask, fl, s.cuda_stream)
                nat.call("pf_dense_kl_f64", dk.P.data_ptr(), dk.ld, rows, k, H.data_ptr(), st.tgt, st.logt,
                         st.tmask, 1e-300, tau, 0, tgt, dk.is_interior.data_ptr(), o.data_ptr(), fl,
                         s.cuda_stream)
            for _ in range(3):
                run()
            e0, e1 = t.cuda.Event(enable_timing=True), t.cuda.Event(enable_timing=True)
            ms = []
            for _ in range(10):
                nat.call("pf_target_prep_f64", dk.row_ptr(tgt), k, 1e-300, st.tgt, st.logt, st.tmask, fl, s.cuda_stream)
                e0.record()
                nat.call("pf_dense_kl_f64", dk.P.data_ptr(), dk.ld, rows, k, H.data_ptr(), st.tgt, st.logt,
                         st.tmask, 1e-300, tau, 0, tgt, dk.is_interior.data_ptr(), o.data_ptr(), fl,
                         s.cuda_stream)
                e1.record()
                t.cuda.synchronize()
                ms.append(e0.elapsed_time(e1))
            g = int(o[rows:].view(t.int32)[1].item())
            res[f"tau={tau} ws={use_ws}"] = {"ms_min": min(ms), "ms_med": sorted(ms)[5], "guarded": g}
    out[name] = res
    del dk
    t.cuda.empty_cache()
print(json.dumps(out, indent=1))
