"""Aggregate an ncu --csv launch list (gpu__time_duration.sum) by kernel name."""
import csv
import sys
from collections import defaultdict

lines = [ln for ln in open(sys.argv[1]) if ln.startswith('"')]
rows = list(csv.DictReader(lines))
agg = defaultdict(lambda: [0, 0.0])
total = 0.0
for r in rows:
    if r.get("Metric Name") != "gpu__time_duration.sum":
        continue
    name = r["Kernel Name"].split("(")[0][:60]
    v = float(r["Metric Value"].replace(",", ""))
    unit = r.get("Metric Unit", "nsecond")
    v = v * {"nsecond": 1e-3, "ns": 1e-3, "usecond": 1.0, "us": 1.0, "msecond": 1e3, "ms": 1e3}.get(unit, 1e-3)
    agg[name][0] += 1
    agg[name][1] += v
    total += v
cycles = int(sys.argv[2]) if len(sys.argv) > 2 else 1
print(f"total {total:.1f} us over {cycles} cycle(s) = {total / cycles:.1f} us/cycle")
for k, (n, t) in sorted(agg.items(), key=lambda x: -x[1][1]):
    print(f"{t / cycles:10.1f} us/cycle {100 * t / total:5.1f}%  n={n // cycles:5d}  avg {t / n:8.2f} us  {k}")
