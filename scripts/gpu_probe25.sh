set -u
mkdir -p gpurun_out; O=gpurun_out; F=$O/kd_ab_r2f.jsonl; rm -f $F
for i in 1 2; do
  for kd in 0 2 3; do
    NIMBLE_EXP_KD=$kd timeout 600 python scripts/gemm_sweep.py --Ms 512,1024,2048,4096,17448 --tag "kd$kd.$i" --out $F > /dev/null 2>&1
  done
done
python - <<'PY'
import json,collections
t=collections.defaultdict(lambda: collections.defaultdict(list))
for l in open("gpurun_out/kd_ab_r2f.jsonl"):
    r=json.loads(l)
    if r.get("op")!="dense": continue
    t[(r["N"],r["K"],r["M"])][r["tag"].split(".")[0]].append(r["us"])
for k in sorted(t):
    print(k, {a: round(min(v),2) for a,v in t[k].items()})
PY
