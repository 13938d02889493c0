set -u
mkdir -p gpurun_out; O=gpurun_out
rm -f $O/sweep_kd3.jsonl
for kd in 2 3 2 3; do
  NIMBLE_EXP_KD=$kd timeout 600 python scripts/gemm_sweep.py --Ms 256,512,1024,2048,4096,17448 --tag "kd$kd" --out $O/sweep_kd3.jsonl > /dev/null 2>&1
done
NIMBLE_EXP_KD=3 timeout 600 python -m pytest tests/test_gpu_parity_r2.py tests/test_gpu_dense_ln.py -q -x -p no:cacheprovider 2>&1 | tail -2
NIMBLE_EXP_KD=3 timeout 900 python bench.py --no-static > $O/bench_kd3.json 2> $O/bench_kd3.err; python -c "
import json; d=json.loads(open('$O/bench_kd3.json').read().strip().splitlines()[-1]); print('bench kd3', d['value'], d['roofline']['frac'], d['batch1']['value'])"
timeout 900 python bench.py --no-static > $O/bench_kd2.json 2> $O/bench_kd2.err; python -c "
import json; d=json.loads(open('$O/bench_kd2.json').read().strip().splitlines()[-1]); print('bench kd2', d['value'], d['roofline']['frac'], d['batch1']['value'])"
