"""Small driver for ncu captures of the CSR and batched kernels (not a benchmark)."""
import math
import sys

import numpy as np
import torch as t

sys.path.insert(0, ".")
import bench  # noqa: E402
import paper_1708_02845_b200 as pf  # noqa: E402
from paper_1708_02845_b200 import _device as dev  # noqa: E402
from paper_1708_02845_b200 import _native as nat  # noqa: E402

device = t.device("cuda", 0)
peak = 6552.0
which = sys.argv[1] if len(sys.argv) > 1 else "csr"
if which == "csr":
    r = bench.extra_c3(t, nat, dev, pf, device, 3, peak)
    print({k: v for k, v in r.items()})
elif which == "tracer":
    print(bench.extra_tracer(t, nat, dev, pf, device))
elif which == "f32":
    rows, k = 102104, 4250
    ld = dev.leading_dim(k)
    P = bench.make_synthetic_slab(t, rows, k, ld, 0, device)
    dk = dev.DeviceKernel(None, np.array([], np.int64), device=device, rows=rows, n=rows, k=k,
                          P_dev=P)
    print(bench.extra_f32(t, nat, dev, pf, dk, rows // 3 + 1, 5, peak))
elif which == "hausdorff":
    sys.path.insert(0, "tests")
    from tests.conftest import case
    c = case("disk40")
    pairs = [(c[f"path/kl/{pi}/points"], c[f"path/tv/{pi}/points"]) for pi in range(24)]
    for _ in range(2):
        print(pf.path_hausdorff_batch(pairs)[:3])
else:
    rows, k, T = 131072, 4102, 1024
    ld = dev.leading_dim(k)
    P = bench.make_synthetic_slab(t, rows, k, ld, 7, device)
    dk = dev.DeviceKernel(None, np.array([], np.int64), device=device, rows=rows, n=rows, k=k,
                          P_dev=P)
    pk = pf.PoissonKernel(np.empty((0, 0)), np.array([], np.int64), 0.0, 0.0)
    H = dk.negentropy(1e-300)
    ldl = dev.round_up(k, 16)
    tg = t.arange(0, rows, rows // T, device=device)[:T].contiguous()
    Pt = dk.P.index_select(0, tg)
    L = t.empty((T, ldl), dtype=t.float64, device=device)
    Tc = t.empty((T, ldl), dtype=t.float64, device=device)
    out = t.empty((rows, T), dtype=t.float64, device=device)
    s = t.cuda.current_stream().cuda_stream
    A, ea, ldk = dk.slices(1e-300)
    B = t.empty((7, T, ldk), dtype=t.uint8, device=device)
    eb = t.empty(T, dtype=t.int32, device=device)
    for _ in range(3):
        nat.call("pf_batch_prep_f64", Pt.data_ptr(), Pt.stride(0), T, k, ldl, 1e-300, 0,
                 L.data_ptr(), Tc.data_ptr(), 0, s)
        if which == "gemm_i8":
            nat.call("pf_slice_targets_u8", L.data_ptr(), ldl, T, k, ldk, B.data_ptr(),
                     eb.data_ptr(), 0, s)
            nat.call("pf_batched_kl_i8", A.data_ptr(), ea.data_ptr(), rows, B.data_ptr(),
                     eb.data_ptr(), T, k, ldk, H.data_ptr(), tg.data_ptr(), 1e-3, 0,
                     out.data_ptr(), T, 64, s)
        else:
            nat.call("pf_batched_kl_f64", dk.P.data_ptr(), dk.ld, rows, k, H.data_ptr(),
                     L.data_ptr(), Tc.data_ptr(), ldl, T, tg.data_ptr(), 1e-300, 1e-3, 0,
                     out.data_ptr(), T, 0, s)
    t.cuda.synchronize()
    print("ok")
