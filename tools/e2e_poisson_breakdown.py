"""Where the end-to-end poisson_kernel(mesh) time goes (host prep, device, D2H)."""
import sys
import time
from pathlib import Path

sys.path.insert(0, str(Path(__file__).resolve().parent.parent))
import torch  # noqa: E402
from oracle import inputs as I  # noqa: E402
import paper_1708_02845_b200.laplacian as L  # noqa: E402
sys.path.insert(0, str(Path(__file__).resolve().parent))
from bench_poisson import SPECS  # noqa: E402

name = sys.argv[1] if len(sys.argv) > 1 else "c2"
mesh = I.build(SPECS[name])
for rep in range(2):
    torch.cuda.synchronize()
    t0 = time.perf_counter()
    dp = L.DevicePoisson(mesh)
    t1 = time.perf_counter()
    dk = dp.device_kernel()
    torch.cuda.synchronize()
    t2 = time.perf_counter()
    dense = L.dense_to_host(dk.P, dk.n, dk.k)
    t3 = time.perf_counter()
    print(f"{name} rep{rep}: init(topology+plan+upload) {t1 - t0:.3f} s, device {t2 - t1:.3f} s, "
          f"host copy {t3 - t2:.3f} s ({dense.nbytes / (t3 - t2) / 1e9:.1f} GB/s)", flush=True)
    del dk, dense, dp
    torch.cuda.empty_cache()
