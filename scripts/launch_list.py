"""ncu --metrics gpu__time_duration.sum --csv launch list -> profiles/launches_*.json."""
import csv
import json
import sys
from collections import defaultdict

src, cmd = sys.argv[1], sys.argv[2]
lines = [l for l in open(src) if l.startswith('"')]
rows = list(csv.DictReader(lines))
agg = defaultdict(lambda: [0, 0.0])
for r in rows:
    if r["Metric Name"] != "gpu__time_duration.sum":
        continue
    name = r["Kernel Name"].split("(")[0]
    v = float(r["Metric Value"].replace(",", ""))
    scale = {"ns": 1e-3, "us": 1.0, "ms": 1e3}[r["Metric Unit"]]
    agg[name][0] += 1
    agg[name][1] += v * scale
total = sum(t for _, t in agg.values())
out = {"command": cmd,
       "note": "cold-cache, serialised per-launch times: compare shares, not absolutes",
       "kernels": {k: {"launches": n, "total_us": round(t, 1), "share": round(t / total, 4)}
                   for k, (n, t) in sorted(agg.items(), key=lambda kv: -kv[1][1])}}
print(json.dumps(out, indent=1))
