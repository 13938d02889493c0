"""Top CUDA source lines with their dominant stall reasons."""
import csv
import io
import subprocess
import sys

rep = sys.argv[1]
n = int(sys.argv[2]) if len(sys.argv) > 2 else 20
out = subprocess.run(["ncu", "-i", rep, "--page", "source", "--csv", "--print-source", "cuda,sass"],
                     capture_output=True, text=True).stdout
rows = list(csv.reader(io.StringIO(out)))
fname, hdr, agg = None, None, []
for r in rows:
    if not r:
        continue
    if r[0] == "File Path":
        fname = r[1].split("/")[-1]; continue
    if r[0] == "Line No":
        hdr = r; continue
    if hdr is None or r[0] == "Function Name" or len(r) < len(hdr) or r[2] != "-":
        continue
    S = int(r[4] or 0)
    if not S:
        continue
    reasons = {}
    for k, v in zip(hdr, r):
        if k.startswith("stall_") and "Not Issued" not in k and v not in ("", "0"):
            reasons[k[6:]] = int(v)
    top = sorted(reasons.items(), key=lambda x: -x[1])[:4]
    agg.append((S, int(r[7] or 0), f"{fname}:{r[0]}", r[1].strip()[:70], top))
tot = sum(a[0] for a in agg)
print("total", tot)
for S, ie, loc, src, top in sorted(agg, key=lambda x: -x[0])[:n]:
    print(f"{S:>6} {ie:>9} {loc:<16} {src:<70} {' '.join(f'{k}={v}' for k, v in top)}")
