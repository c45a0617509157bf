"""Persistent K7 pair kernel: per-tile phase timeline of cluster 0
in SM clocks (PF_K7_DIAG=4; 6: no epilogue math, 7: + no loads); tiled
operands unless --row-major."""
import json, os, sys
from pathlib import Path
sys.path.insert(0, str(Path(__file__).resolve().parent.parent))
sys.argv.append("--scan")
import numpy as np
src = open(Path(__file__).parent / "probe_k7pair.py").read().split("ONCE = ")[0]
ns = {"__file__": str(Path(__file__).parent / "probe_k7pair.py"), "__name__": "pk"}
exec(compile(src, "probe_k7pair.py", "exec"), ns)
c = ns["setup"](131072, 4102, 1024, seed=5)
LAYOUT = 1 if "--row-major" in sys.argv else 2
ns["run"](c, LAYOUT)
out = ns["run"](c, LAYOUT)
ntiles = 512 * 8
kmax = (ntiles + 73) // 74
st = out.view(-1)[: kmax * 16].view(kmax, 16).cpu().numpy()[:, :10]
st = st[st[:, 0] > 0]
d = lambda a, b: float(np.median(st[1:, b] - st[1:, a]))
res = {"diag": os.environ.get("PF_K7_DIAG"), "tiles": int(len(st)),
       "free_wait": d(0, 1), "pass1_issue": d(1, 2), "drained_wait": d(2, 3),
       "pass2_issue": d(3, 4), "tile": float(np.median(np.diff(st[:, 1]))),
       "ideal_tile": 129 * (640 + 1536),
       "epi_pass1_seen_after_issue": d(2, 5), "epi_drain1": d(5, 6),
       "epi_pass2_seen_after_issue": d(4, 7), "epi_drain2": d(7, 8),
       "epi_compute_store": d(8, 9) if int(os.environ.get("PF_K7_DIAG", "0")) & 4 else None}
print(json.dumps(res, indent=1))
