set -u
mkdir -p gpurun_out; O=gpurun_out; F=$O/kd1_ab.jsonl; rm -f $F
for i in 1 2; do
  timeout 300 python scripts/exp/pair_medium.py kd2_$i 256,512,1024,2048 >> $F 2>/dev/null
  NIMBLE_KD=1 timeout 300 python scripts/exp/pair_medium.py kd1_$i 256,512,1024,2048 >> $F 2>/dev/null
done
python - <<'PY'
import json,collections,statistics
t=collections.defaultdict(lambda: collections.defaultdict(list))
for l in open("gpurun_out/kd1_ab.jsonl"):
    r=json.loads(l); t[(r["N"],r["K"],r["M"],r["family"])][r["tag"][:3]].append(r["us"])
rs=[]
for k in sorted(t):
    a=min(t[k]["kd2"]); b=min(t[k]["kd1"]); rs.append(a/b); print(k, a, b, f"x{a/b:.3f}")
print("geomean kd2/kd1", statistics.geometric_mean(rs))
PY
