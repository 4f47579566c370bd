"""Summarise an `ncu --metrics gpu__time_duration.sum --csv --log-file` launch list."""
import csv, io, sys
from collections import defaultdict
txt = open(sys.argv[1]).read().splitlines()
start = next(i for i, l in enumerate(txt) if l.startswith('"ID"'))
rows = list(csv.DictReader(io.StringIO("\n".join(txt[start:]))))
agg = defaultdict(lambda: [0, 0.0])
for r in rows:
    if r.get("Metric Name") != "gpu__time_duration.sum":
        continue
    v = float(r["Metric Value"].replace(",", ""))
    unit = r.get("Metric Unit", "")
    v = v * {"nsecond": 1e-3, "ns": 1e-3, "usecond": 1.0, "us": 1.0, "msecond": 1e3, "ms": 1e3}.get(unit, 1.0)
    name = r["Kernel Name"].split("(")[0][:70]
    agg[name][0] += 1
    agg[name][1] += v
tot = sum(v for _, v in agg.values())
print(f"{'launches':>8} {'total_us':>10} {'avg_us':>9} {'share':>6}  kernel")
for k, (c, v) in sorted(agg.items(), key=lambda x: -x[1][1]):
    print(f"{c:8d} {v:10.1f} {v/c:9.1f} {100*v/tot:5.1f}%  {k}")
