"""Aggregate ncu warp-stall samples + instructions by CUDA source line (needs -lineinfo)."""
import csv
import io
import subprocess
import sys

rep = sys.argv[1]
n = int(sys.argv[2]) if len(sys.argv) > 2 else 25
out = subprocess.run(["ncu", "-i", rep, "--page", "source", "--csv", "--print-source", "cuda,sass"],
                     capture_output=True, text=True).stdout
rows = list(csv.reader(io.StringIO(out)))
fname, agg, tot = None, [], 0
hdr = None
for r in rows:
    if not r:
        continue
    if r[0] == "File Path":
        fname = r[1].split("/")[-1]
        continue
    if r[0] == "Line No":
        hdr = r
        continue
    if hdr is None or r[0] == "Function Name" or len(r) < len(hdr):
        continue
    if r[2] != "-":
        continue    # sass sub-rows
    S = int(r[4] or 0)
    ie = int(r[7] or 0)
    if S or ie:
        agg.append((S, ie, f"{fname}:{r[0]}", r[1].strip()))
        tot += S
print("total samples", tot)
for S, ie, loc, src in sorted(agg, key=lambda x: -x[0])[:n]:
    print(f"{S:>6} {ie:>10}  {loc:<18} {src[:100]}")
