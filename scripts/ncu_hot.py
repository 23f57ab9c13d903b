"""Top SASS instructions by warp-stall samples from an ncu source-page CSV.

  ncu -i rep.ncu-rep --page source --csv --print-source sass --kernel-name regex:flow --launch-skip K \
      --launch-count 1 > src.csv ; python scripts/ncu_hot.py src.csv [N]
"""
import csv
import sys

rows = list(csv.reader(open(sys.argv[1])))
n = int(sys.argv[2]) if len(sys.argv) > 2 else 60
# find header row
hi = next(i for i, r in enumerate(rows) if any("Source" == c or "Address" in c for c in r))
hdr = rows[hi]
body = rows[hi + 1:]
cols = {c: i for i, c in enumerate(hdr)}
samp_col = next((c for c in hdr if c.startswith("Warp Stall Sampling (All")), None)
print("columns:", [c for c in hdr][:40])
if samp_col is None:
    sys.exit(0)
tot = 0.0
data = []
for r in body:
    try:
        v = float(r[cols[samp_col]] or 0)
    except Exception:
        continue
    tot += v
    data.append((v, r))
data.sort(key=lambda x: -x[0])
src = cols.get("Source", 1)
stall_cols = [c for c in hdr if c.startswith("stall_") or "Stall" in c][:12]
for v, r in data[:n]:
    print(f"{100 * v / max(tot, 1):5.1f}%  {r[src][:90]}")
