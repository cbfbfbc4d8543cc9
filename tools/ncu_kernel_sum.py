"""Sum gpu__time_duration per kernel name from an ncu --csv launch list:
    python tools/ncu_kernel_sum.py launches.csv"""
import csv
import sys
from collections import defaultdict

rows = list(csv.reader(open(sys.argv[1])))
i = next(k for k, r in enumerate(rows) if "Kernel Name" in r)
hdr = rows[i]
tot = defaultdict(float)
cnt = defaultdict(int)
for r in rows[i + 1:]:
    if len(r) != len(hdr):
        continue
    d = dict(zip(hdr, r))
    if d.get("Metric Name") != "gpu__time_duration.sum":
        continue
    name = d["Kernel Name"].split("(")[0]
    v = float(d["Metric Value"].replace(",", ""))
    unit = d.get("Metric Unit", "")
    ms = v * {"ns": 1e-6, "usecond": 1e-3, "us": 1e-3, "msecond": 1.0, "ms": 1.0, "nsecond": 1e-6}.get(unit, 1e-6)
    tot[name] += ms
    cnt[name] += 1
for name, ms in sorted(tot.items(), key=lambda kv: -kv[1]):
    print(f"{ms:10.3f} ms  {cnt[name]:5d}  {name}")
print(f"{sum(tot.values()):10.3f} ms  total")
