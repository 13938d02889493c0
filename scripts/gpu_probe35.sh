set -u
mkdir -p gpurun_out; O=gpurun_out; L=$PWD/paper_2006_03031_b200
F=$O/tw_ab.jsonl; rm -f $F
for i in 1 2; do
  timeout 300 python scripts/exp/pair_medium.py base$i 512,1024,2048 >> $F 2>/dev/null
  NIMBLE_LIB=$L/libnimble_tw.so timeout 300 python scripts/exp/pair_medium.py tw$i 512,1024,2048 >> $F 2>/dev/null
done
G=$O/tw_big.jsonl; rm -f $G
for i in 1 2; do
  timeout 600 python scripts/gemm_sweep.py --Ms 17448 --tag base$i --out $G > /dev/null 2>&1
  NIMBLE_LIB=$L/libnimble_tw.so timeout 600 python scripts/gemm_sweep.py --Ms 17448 --tag tw$i --out $G > /dev/null 2>&1
done
python - <<'PY'
import json,collections
for f in ("gpurun_out/tw_ab.jsonl","gpurun_out/tw_big.jsonl"):
    t=collections.defaultdict(lambda: collections.defaultdict(list))
    for l in open(f):
        r=json.loads(l)
        if r.get("op","dense")!="dense": continue
        t[(r["N"],r["K"],r["M"])][r["tag"][:-1]].append(r["us"])
    for k in sorted(t):
        b=min(t[k]["base"]); w=min(t[k]["tw"]); print(k, round(b,2), round(w,2), f"x{b/w:.3f}")
PY
for i in 1 2; do
  timeout 600 python bench.py --steps 20 --warmup 3 > $O/bb.json 2>/dev/null; python -c "
import json; d=json.loads(open('$O/bb.json').read().strip().splitlines()[-1]); print('base bench', round(d['value'],1), d['roofline']['frac'], d['clocks']['sm_mhz'])"
  NIMBLE_LIB=$L/libnimble_tw.so timeout 600 python bench.py --steps 20 --warmup 3 > $O/bt.json 2>/dev/null; python -c "
import json; d=json.loads(open('$O/bt.json').read().strip().splitlines()[-1]); print('tw bench', round(d['value'],1), d['roofline']['frac'], d['clocks']['sm_mhz'])"
done
NIMBLE_LIB=$L/libnimble_tw.so timeout 900 python -m pytest tests/test_gpu_parity_r2.py tests/test_gpu_dense_bmm.py tests/test_gpu_dense_ln.py tests/test_gpu_devdispatch.py -q -x -p no:cacheprovider > $O/pytest_tw.txt 2>&1; tail -1 $O/pytest_tw.txt
