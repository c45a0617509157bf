"""Per-kernel summary of an ncu launch list (--metrics gpu__time_duration.sum --csv
--log-file <csv>): launches, total / average ns, share of the total kernel time.

    python tools/launch_summary.py gpurun_out/launches_<tag>.csv > profiles/<tag>_launches_summary.csv
"""
import csv
import sys
from collections import defaultdict
from io import StringIO

rows = [ln for ln in open(sys.argv[1]) if ln.startswith('"')]
r = list(csv.reader(StringIO("".join(rows))))
h = r[0]
iK, iM, iV, iU = h.index("Kernel Name"), h.index("Metric Name"), h.index("Metric Value"), h.index("Metric Unit")
tot = defaultdict(float)
cnt = defaultdict(int)
scale = {"nsecond": 1.0, "usecond": 1e3, "msecond": 1e6, "second": 1e9}
for row in r[1:]:
    if row[iM] != "gpu__time_duration.sum":
        continue
    name = row[iK].split("(")[0].strip()
    tot[name] += float(row[iV].replace(",", "")) * scale.get(row[iU], 1.0)
    cnt[name] += 1
total = sum(tot.values())
w = csv.writer(sys.stdout)
w.writerow(["kernel", "launches", "total_ns", "avg_ns", "share_of_total"])
for name in sorted(tot, key=lambda n: -tot[n]):
    w.writerow([name, cnt[name], int(tot[name]), int(tot[name] / cnt[name]), round(tot[name] / total, 4)])
