import sys; sys.path.insert(0, '.')
import numpy as np, torch as t
from paper_1708_02845_b200 import fileio as F, _native as nat
from tests.test_wire_gpu import edge_values
v = edge_values()
import os
if os.environ.get("STACK"):
    from cuda.bindings import runtime as rt
    t.zeros(1, device='cuda')
    print("set stack", rt.cudaDeviceSetLimit(rt.cudaLimit.cudaLimitStackSize, int(os.environ["STACK"])))
    print("get", rt.cudaDeviceGetLimit(rt.cudaLimit.cudaLimitStackSize))
else:
    from cuda.bindings import runtime as rt
    t.zeros(1, device='cuda')
    print("default stack", rt.cudaDeviceGetLimit(rt.cudaLimit.cudaLimitStackSize))
dv = t.from_numpy(v).cuda()
n = len(v)
for kind in (5, 4):
    slots = t.zeros(n * 64, dtype=t.uint8, device='cuda'); lens = t.zeros(n, dtype=t.int32, device='cuda')
    nat.call("pf_format_lines", dv.data_ptr(), n, kind, 0, slots.data_ptr(), lens.data_ptr(), 0, t.cuda.current_stream().cuda_stream)
    t.cuda.synchronize()
    sl = slots.view(n, 64).cpu().numpy(); ln = lens.cpu().numpy()
    bad = 0
    for i in range(n):
        got = sl[i, :ln[i]].tobytes().decode('ascii', 'replace')
        ref = f"{v[i]:.17g}" if kind == 5 else repr(float(v[i]))
        if got != ref:
            bad += 1
            if bad < 8: print(kind, i, repr(v[i]), ln[i], repr(got), ref)
    print("kind", kind, "bad", bad, "of", n)
