set -u
mkdir -p gpurun_out; O=gpurun_out
python scripts/trace_stages.py 17448x3072x1024,17448x4096x1024 2>&1 | grep -v '^$'
rm -f $O/sweep_roles.jsonl
timeout 600 python scripts/gemm_sweep.py --Ms 2048,4096,17448 --tag roles --out $O/sweep_roles.jsonl > /dev/null 2>&1; echo "sweep rc=$?"
timeout 900 python bench.py --no-static > $O/bench_roles.json 2> $O/bench_roles.err; python -c "
import json; d=json.loads(open('$O/bench_roles.json').read().strip().splitlines()[-1]); print('bench', d['value'], d['e2e']['value'], d['roofline']['frac'], d['clocks'])"
timeout 600 python -m pytest tests/test_gpu_parity_r2.py tests/test_gpu_dense_ln.py -x -q -p no:cacheprovider 2>&1 | tail -2
