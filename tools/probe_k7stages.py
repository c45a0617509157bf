"""K7 pair kernel on tiled operands (PF_K7_DIAG=10: no epilogue math, stage timeline): for the
first 2,048 ring stages of cluster 0's leader, the time from the TMA issue of
a stage to the MMA thread seeing it full, and the MMA-side gaps, in SM clocks."""
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
tl = out.view(-1)[65536: 65536 + 8192].view(4096, 2).cpu().numpy()[:2048]
issue, full = tl[:, 0], tl[:, 1]
lat = full - issue          # SM clocks
gap = np.diff(full)
nkb = (4102 + 31) // 32
p1 = np.array([(i // nkb) % 2 == 0 for i in range(len(lat))])
res = {"issue_to_full_clk": {"p1_med": float(np.median(lat[p1])), "p2_med": float(np.median(lat[~p1])),
                            "p90": float(np.percentile(lat, 90)), "max": float(lat.max())},
       "mma_gap_clk": {"p1_med": float(np.median(gap[p1[1:]])), "p2_med": float(np.median(gap[~p1[1:]])),
                       "p1_mean": float(np.mean(gap[p1[1:]])), "p2_mean": float(np.mean(gap[~p1[1:]]))},
       "ideal_stage_clk": {"p1": 640, "p2": 1536}}
print(json.dumps(res, indent=1))
