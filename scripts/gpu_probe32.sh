set -u
mkdir -p gpurun_out; O=gpurun_out
timeout 900 python -m pytest tests/test_gpu_parity_r2.py tests/test_gpu_dense_ln.py tests/test_gpu_bench_config.py tests/test_gpu_dense_bmm.py -q -x -p no:cacheprovider > $O/pytest_t240.txt 2>&1; tail -3 $O/pytest_t240.txt
F=$O/t240_ab.jsonl; rm -f $F
for i in 1 2; do
  timeout 600 python scripts/gemm_sweep.py --Ms 4096,8192,17448 --tag t240.$i --out $F > /dev/null 2>&1
  NIMBLE_EXP_T3=256 timeout 600 python scripts/gemm_sweep.py --Ms 4096,8192,17448 --tag t256.$i --out $F > /dev/null 2>&1
done
python - <<'PY'
import json,collections
t=collections.defaultdict(lambda: collections.defaultdict(list))
for l in open("gpurun_out/t240_ab.jsonl"):
    r=json.loads(l)
    if r.get("op")!="dense": continue
    t[(r["N"],r["K"],r["M"])][r["tag"].split(".")[0]].append(round(r["us"],2))
for k in sorted(t): print(k, dict(t[k]))
PY
for i in 1 2; do
  timeout 600 python bench.py --steps 20 --warmup 3 > $O/b240.json 2>/dev/null; python -c "
import json; d=json.loads(open('$O/b240.json').read().strip().splitlines()[-1]); print('t240 bench', round(d['value'],1), d['roofline']['frac'], d['clocks']['sm_mhz'])"
  NIMBLE_EXP_T3=256 timeout 600 python bench.py --steps 20 --warmup 3 > $O/b256.json 2>/dev/null; python -c "
import json; d=json.loads(open('$O/b256.json').read().strip().splitlines()[-1]); print('t256 bench', round(d['value'],1), d['roofline']['frac'], d['clocks']['sm_mhz'])"
done
