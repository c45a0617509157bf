"""K7 pair kernel phase timeline (PF_K7_DIAG=4 or 7 builds stamps into out):
per-CTA setup / pass 1 / drain wait / pass 2 / epilogue / teardown and the
gap between consecutive CTAs on one SM."""
import json, os, sys
from pathlib import Path
sys.path.insert(0, str(Path(__file__).resolve().parent.parent))
sys.argv.append("--scan")   # keep probe_k7pair's module-level runs off
import numpy as np
import torch as t
import importlib.util
spec = importlib.util.spec_from_file_location("pk", str(Path(__file__).parent / "probe_k7pair.py"))
src = open(spec.origin).read().split("ONCE = ")[0]
ns = {"__file__": spec.origin, "__name__": "pk"}
exec(compile(src, spec.origin, "exec"), ns)
c = ns["setup"](131072, 4102, 1024, seed=5)
ns["run"](c, 1)
out = ns["run"](c, 1)
gx, gy = 2 * 8, 512
st = out.view(-1)[: gx * gy * 8].view(gx * gy, 8).cpu().numpy()
st[:, :7] -= st[:, 0].min()
ph = {"setup": st[:, 1] - st[:, 0], "pass1_issue": st[:, 2] - st[:, 1], "drain_wait": st[:, 3] - st[:, 2],
      "pass2": st[:, 4] - st[:, 3], "epilogue": st[:, 5] - st[:, 4], "teardown": st[:, 6] - st[:, 5],
      "total": st[:, 6] - st[:, 0]}
lead = np.arange(gx * gy) % 2 == 0
res = {k: {"med_us": float(np.median(v[lead]) / 1e3), "p90_us": float(np.percentile(v[lead], 90) / 1e3)}
       for k, v in ph.items()}
gaps = []
for sm in np.unique(st[:, 7]):
    r = st[st[:, 7] == sm]
    r = r[np.argsort(r[:, 0])]
    gaps += list(r[1:, 0] - r[:-1, 6])
res["gap_between_ctas_us"] = {"med": float(np.median(gaps) / 1e3), "p90": float(np.percentile(gaps, 90) / 1e3)}
res["span_ms"] = float(st[:, 6].max() / 1e6)
print(json.dumps({"diag": os.environ.get("PF_K7_DIAG"), **res}, indent=1))
if int(os.environ.get("PF_K7_DIAG", "0")) & 8:   # CTA (0,0)'s MMA-thread stage timeline
    nkb = (4102 + 31) // 32
    tl = out.view(-1)[gx * gy * 8: gx * gy * 8 + 4 * nkb].view(2 * nkb, 2).cpu().numpy()
    wait = tl[:, 1] - tl[:, 0]
    step = np.diff(tl[:, 1])
    print(json.dumps({"pass1_wait_clk_med": float(np.median(wait[1:nkb])),
                      "pass1_step_clk_med": float(np.median(step[: nkb - 1])),
                      "pass2_wait_clk_med": float(np.median(wait[nkb + 1:])),
                      "pass2_step_clk_med": float(np.median(step[nkb:])),
                      "pass1_step_clk_p10_p90": [float(np.percentile(step[: nkb - 1], 10)), float(np.percentile(step[: nkb - 1], 90))],
                      "first_steps": step[:12].tolist()}))
