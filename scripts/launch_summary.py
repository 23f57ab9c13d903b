"""Summarise an ncu launch list (gpu__time_duration.sum per launch) by kernel name."""
import csv
import json
import sys
from collections import defaultdict

rows = list(csv.DictReader([l for l in open(sys.argv[1]) if not l.startswith("==")]))
tot = defaultdict(float)
cnt = defaultdict(int)
for r in rows:
    if r.get("Metric Name") != "gpu__time_duration.sum":
        continue
    k = r["Kernel Name"].split("(")[0]
    v = float(r["Metric Value"].replace(",", ""))
    if r.get("Metric Unit") == "us":
        v *= 1e3
    tot[k] += v
    cnt[k] += 1
allns = sum(tot.values())
out = {k: {"launches": cnt[k], "total_us": tot[k] / 1e3, "share": tot[k] / allns} for k in sorted(tot, key=lambda x: -tot[x])}
print(json.dumps(out, indent=1))
