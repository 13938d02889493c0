"""Per-kernel share of device time from an ncu --metrics gpu__time_duration.sum CSV launch list.
Only the LAST occurrence window is used: launches after the final `--skip` count are summed."""
import csv
import re
import sys
from collections import defaultdict

path = sys.argv[1]
rows = []
with open(path) as f:
    lines = [l for l in f if not l.startswith("==")]
rd = csv.DictReader(lines)
for r in rd:
    if r.get("Metric Name") != "gpu__time_duration.sum":
        continue
    name = r["Kernel Name"]
    v = float(r["Metric Value"].replace(",", ""))
    unit = r.get("Metric Unit", "")
    if unit in ("nsecond", "ns"):
        v /= 1000.0
    elif unit in ("msecond", "ms"):
        v *= 1000.0
    rows.append((int(r["ID"]), name, v))
rows.sort()
ours = [r for r in rows if "nimble" in r[1]]
agg = defaultdict(lambda: [0, 0.0])
for _, n, v in ours:
    key = re.sub(r"\(.*", "", n)
    key = re.sub(r"<unnamed>::|nimble::", "", key)
    agg[key][0] += 1
    agg[key][1] += v
tot = sum(v for _, v in agg.values())
print(f"libnimble kernels: {len(ours)} launches, {tot:.1f} us total (ncu: serialised, cold-cache)")
for k, (c, v) in sorted(agg.items(), key=lambda x: -x[1][1]):
    print(f"  {100 * v / tot:5.1f}%  {v:10.1f} us  {c:5d} x  avg {v / c:8.2f} us  {k}")
