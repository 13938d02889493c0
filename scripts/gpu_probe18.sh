set -u
mkdir -p gpurun_out; O=gpurun_out
timeout 1500 python -m pytest tests -m gpu -q -x -p no:cacheprovider > $O/pytest_gpu_r2d.txt 2>&1; tail -3 $O/pytest_gpu_r2d.txt
rm -f $O/sweep_kd_default.jsonl
for i in 1 2; do
  timeout 600 python scripts/gemm_sweep.py --Ms 1,16,64,128,256,512,1024,2048,4096,17448 --tag "kddef$i" --out $O/sweep_kd_default.jsonl > /dev/null 2>&1
done
timeout 900 python bench.py > $O/bench_r2d.json 2> $O/bench_r2d.err; python -c "
import json; d=json.loads(open('$O/bench_r2d.json').read().strip().splitlines()[-1]); print('bench', d['value'], d['roofline']['frac'], d.get('batch1',{}).get('value'), d['e2e']['value'], d['clocks'])"
