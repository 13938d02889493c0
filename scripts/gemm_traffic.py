"""DRAM traffic per launch of the dominant kernel (dense GEMM) from an ncu --set full report:
dram__bytes_read.sum + dram__bytes_write.sum averaged over the captured launches (one
layer's QKV, O, FFN1, FFN2 at the bench configuration).  Output JSON for bench.py."""
import csv
import io
import json
import subprocess
import sys

SCALE = {"byte": 1, "Kbyte": 1e3, "Mbyte": 1e6, "Gbyte": 1e9}
rep = sys.argv[1]
raw = list(csv.reader(io.StringIO(subprocess.run(["ncu", "-i", rep, "--page", "raw", "--csv"],
                                                 capture_output=True, text=True).stdout)))
hdr, units = raw[0], raw[1]
u = dict(zip(hdr, units))
per = []
for row in raw[2:]:
    d = dict(zip(hdr, row))
    rd = float(d["dram__bytes_read.sum"]) * SCALE[u["dram__bytes_read.sum"]]
    wr = float(d["dram__bytes_write.sum"]) * SCALE[u["dram__bytes_write.sum"]]
    per.append({"kernel": d["Kernel Name"][:80], "grid": d["Grid Size"], "dram_read": rd, "dram_write": wr,
                "duration_us": float(d["gpu__time_duration.sum"])})
out = {"source": rep, "launches": per,
       "traffic_bytes_per_launch": sum(p["dram_read"] + p["dram_write"] for p in per) / max(len(per), 1)}
print(json.dumps(out, indent=1))
