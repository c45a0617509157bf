"""Summarise an ncu --metrics gpu__time_duration.sum CSV: per-kernel totals."""
import collections
import csv
import sys

rows = [l for l in open(sys.argv[1]) if l.startswith('"')]
agg = collections.OrderedDict()
seq = []
for r in csv.DictReader(rows):
    if r.get("Metric Name") != "gpu__time_duration.sum":
        continue
    name = r["Kernel Name"].split("(")[0].replace("pf::<unnamed>::", "")
    v = float(r["Metric Value"].replace(",", ""))
    v *= {"ns": 1e-3, "nsecond": 1e-3, "us": 1.0, "usecond": 1.0, "ms": 1e3, "msecond": 1e3}[r["Metric Unit"]]
    a = agg.setdefault(name, [0, 0.0])
    a[0] += 1
    a[1] += v
    seq.append((name, r["Grid Size"], v))
tot = sum(t for _, t in agg.values())
for k, (n, t) in sorted(agg.items(), key=lambda x: -x[1][1]):
    print(f"{t:11.1f} us {100 * t / tot:5.1f}%  x{n:<4d} {k}")
if "-v" in sys.argv:
    for name, g, v in seq:
        print(f"{v:10.1f} {g:>16s} {name}")
