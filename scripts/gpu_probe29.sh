set -u
mkdir -p gpurun_out; O=gpurun_out; F=$O/c3_ab.txt; rm -f $F
L=$PWD/paper_2006_03031_b200
for i in 1 2; do
  for v in r2d mw cur; do
    if [ $v = cur ]; then lib=$L/libnimble.so; else lib=$L/libnimble_$v.so; fi
    echo -n "$v " >> $F; NIMBLE_LIB=$lib timeout 300 python scripts/exp/c3_time.py >> $F 2>&1
  done
done
cat $F
G=$O/c3_gemm_ab.jsonl; rm -f $G
for v in r2d cur; do
  if [ $v = cur ]; then lib=$L/libnimble.so; else lib=$L/libnimble_$v.so; fi
  NIMBLE_LIB=$lib timeout 600 python scripts/gemm_sweep.py --shapes base --Ms 1,64,128 --tag $v --out $G > /dev/null 2>&1
done
python - <<'PY'
import json,collections
t=collections.defaultdict(dict)
for l in open("gpurun_out/c3_gemm_ab.jsonl"):
    d=json.loads(l); t[(d.get("op"),d["N"],d["K"],d["M"])][d["tag"]]=round(d["us"],2)
for k in sorted(t): print(k, t[k])
PY
