"""Persistent K7 pair kernel: per-tile phase timeline of cluster 0
(PF_K7_DIAG=6: no epilogue stores, 7: + no loads)."""
import json, os, sys
from pathlib import Path
sys.path.insert(0, str(Path(__file__).resolve().parent.parent))
sys.argv.append("--scan")
import numpy as np
src = open(Path(__file__).parent / "probe_k7pair.py").read().split("ONCE = ")[0]
ns = {"__file__": str(Path(__file__).parent / "probe_k7pair.py"), "__name__": "pk"}
exec(compile(src, "probe_k7pair.py", "exec"), ns)
c = ns["setup"](131072, 4102, 1024, seed=5)
ns["run"](c, 1)
out = ns["run"](c, 1)
ntiles = 512 * 8
kmax = (ntiles + 73) // 74
st = out.view(-1)[: kmax * 16].view(kmax, 16).cpu().numpy()[:, :10]
st = st[st[:, 0] > 0]
d = lambda a, b: np.median(st[1:, b] - st[1:, a]) / 1e3
res = {"diag": os.environ.get("PF_K7_DIAG"), "tiles": int(len(st)),
       "free_wait_us": d(0, 1), "pass1_issue_us": d(1, 2), "drained_wait_us": d(2, 3),
       "pass2_issue_us": d(3, 4), "tile_us": float(np.median(np.diff(st[:, 1])) / 1e3),
       "epi_pass1_seen_after_issue_us": d(2, 5), "epi_drain1_us": d(5, 6),
       "epi_pass2_seen_after_issue_us": d(4, 7), "epi_drain2_us": d(7, 8),
       "epi_compute_store_us": d(8, 9) if os.environ.get("PF_K7_DIAG") in ("4", "68", "132", "324") else None}
print(json.dumps(res, indent=1))
