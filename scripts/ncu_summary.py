"""Summarise an ncu --csv launch list (gpu__time_duration.sum) per kernel name.

python scripts/ncu_summary.py launches.csv [top]
"""
import csv
import sys
from collections import defaultdict

path = sys.argv[1]
top = int(sys.argv[2]) if len(sys.argv) > 2 else 30
rows = []
with open(path) as f:
    lines = [l for l in f if l.startswith('"')]
rd = csv.DictReader(lines)
tot = defaultdict(float)
cnt = defaultdict(int)
for r in rd:
    if r.get("Metric Name") != "gpu__time_duration.sum":
        continue
    kn = r["Kernel Name"].replace("(anonymous namespace)::", "").replace("void ", "").replace("aj::", "")
    name = kn.split("(")[0]
    v = float(r["Metric Value"].replace(",", ""))
    unit = r.get("Metric Unit", "nsecond")
    scale = {"nsecond": 1e-6, "usecond": 1e-3, "msecond": 1.0, "second": 1e3}.get(unit, 1e-6)
    tot[name] += v * scale
    cnt[name] += 1
T = sum(tot.values())
print(f"total {T:.2f} ms over {sum(cnt.values())} launches")
for k in sorted(tot, key=tot.get, reverse=True)[:top]:
    print(f"{tot[k]:10.2f} ms {100 * tot[k] / T:5.1f} %  {cnt[k]:6d}  {k}")
